for v in peer_nopdl peer_pdl_notrig peer_pdl; do echo "== $v"; SDR_LIB_PATH=variants/$v.so timeout 200 python tools/time_peer_conc.py 2>&1; done
SDR_LIB_PATH=variants/peer_pdl.so timeout 300 python -m pytest tests/test_peer_gpu.py -q -x 2>&1 | tail -2
for v in peer_nopdl peer_pdl; do echo "== pack $v"; SDR_LIB_PATH=variants/$v.so timeout 200 python tools/time_pack.py 2>&1; done
