timeout 900 python -m pytest tests/test_tc_gpu.py -x -q 2>&1 | tail -3
for fam in bf16 tf32; do for cfg in 1,1,4,8,8 4,1,8,16,16 2,1,2,8,8; do for s in 512 1024 2048; do
python tools/run_config.py --family $fam --mkn $s,$s,$s --cfg $cfg --iters 3 --schedule 0
python tools/run_config.py --family $fam --mkn $s,$s,$s --cfg $cfg --iters 3 --schedule 1
done; done; done
