for spec in "1,1,4,8,8" "4,2,8,16,16" "4,1,8,16,16"; do
  timeout 300 ncu --set full --clock-control none -k regex:tc_gemm -s 2 -c 1 -o gpurun_out/prof_bf16_2048_${spec//,/} python tools/run_config.py --family bf16 --mkn 2048,2048,2048 --cfg $spec --iters 3 > gpurun_out/ncu_tc.log 2>&1
  python tools/run_config.py --family bf16 --mkn 2048,2048,2048 --cfg $spec --iters 3
done
