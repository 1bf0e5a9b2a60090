for v in peer_mb1 peer_mb4 peer_mb5; do echo "== $v"; SDR_LIB_PATH=variants/$v.so timeout 200 python tools/time_peer.py 2>&1 | head -2; done
