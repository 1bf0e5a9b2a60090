for v in r_base r_mb6 r_mb6p r_base r_mb6 r_mb6p; do echo "== $v"; SDR_LIB_PATH=variants/$v.so timeout 200 python tools/time_peer.py 2>&1 | head -2; done
