timeout 600 ncu --set full --clock-control none --import-source on -k regex:simt_gemm -s 2 -c 1 -o gpurun_out/prof_sel2_2048 python tools/run_config.py --mkn 2048,2048,2048 --cfg 2,4,8,16,8 --iters 3 > gpurun_out/ncu_sel.log 2>&1
tail -1 gpurun_out/ncu_sel.log
