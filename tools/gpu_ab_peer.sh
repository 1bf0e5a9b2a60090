timeout 200 python tools/time_peer.py 2>&1 | head -2
timeout 200 python tools/time_peer_conc.py 2>&1
timeout 600 python -m pytest tests/test_peer_gpu.py tests/test_redistribute_gloo.py -q -x -m gpu -k "peer or concurrent or local" 2>&1 | tail -2
