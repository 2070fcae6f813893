timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q -k "pinned" 2>&1 | tail -2
python tools/e2e_probe.py
