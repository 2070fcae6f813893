CF="1,8,8,32,8;2,8,4,16,8;4,8,4,16,16;4,8,8,32,8;4,8,8,16,16;2,8,8,16,16;8,8,8,16,16;8,8,4,16,8;8,8,4,16,16"
timeout 900 python tools/k1_ab.py --tag base --sizes 1024,2048,4096 --cfgs "$CF" > gpurun_out/ab_base.jsonl 2>&1
KP_LIB_PATH=paper_2003_06795_b200/libkp_mb1.so timeout 900 python tools/k1_ab.py --tag mb1 --sizes 1024,2048,4096 --cfgs "$CF" > gpurun_out/ab_mb1.jsonl 2>&1
