for v in r_base r_t8 r_t8p r_t8p_mb4 r_t16p r_t8_mb6 r_t8p_mb6; do echo "== $v"; SDR_LIB_PATH=variants/$v.so timeout 200 python tools/time_peer.py 2>&1 | head -2; done
