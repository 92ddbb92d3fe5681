timeout 300 python -m pytest tests/test_peer_reduce_gpu.py -q -x 2>&1 | tail -2
timeout 300 python tools/e2e_probe.py 2>&1 | tail -24
nvidia-smi topo -m 2>&1 | head -5
