for v in pj96 pj8 pj96 pj8; do echo "== $v"; SDR_LIB_PATH=variants/$v.so timeout 200 python tools/time_peer_conc.py 2>&1; done
