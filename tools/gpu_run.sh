set -x
timeout 900 python tools/k1_ab.py --tag pol --sizes 2048,4096 --layouts nn,nt,tn,tt --cfgs "1,8,8,32,8;2,8,4,16,8;4,8,4,16,16;4,8,8,32,8;4,8,8,16,16;2,8,8,16,16;8,8,8,16,16;2,4,8,16,16" --schedules 0,1 > gpurun_out/ab_pol.jsonl 2>gpurun_out/ab_pol.err
tail -3 gpurun_out/ab_pol.err
timeout 1200 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -5
