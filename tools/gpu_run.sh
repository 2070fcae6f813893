timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q -k "timing" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
