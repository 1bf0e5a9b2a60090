for v in peer_exact peer_fast; do echo "== $v"; SDR_LIB_PATH=variants/$v.so timeout 200 python tools/time_peer.py; done
