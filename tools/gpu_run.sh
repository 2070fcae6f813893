set -x
timeout 1200 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-sweep --cpu-seconds 1 > gpurun_out/bench_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:simt_gemm -s 2 -c 1 -o gpurun_out/prof_sel_2048 python tools/run_config.py --mkn 2048,2048,2048 --cfg 8,8,4,16,8 --iters 3 > gpurun_out/ncu_sel.log 2>&1
timeout 1500 python -m paper_2003_06795_b200 sweep --shapes networks+squares --family f32 --trans nt --out gpurun_out/b200_f32_nt_train.csv --sidecar gpurun_out/b200_f32_nt_train.sidecar.json > gpurun_out/sweep_nt.log 2>&1
tail -2 gpurun_out/sweep_nt.log
