CF="1,8,8,32,8;2,8,4,16,8;4,8,4,16,16;4,8,8,32,8;8,8,4,16,8;8,8,4,16,16;4,4,4,16,8;2,4,4,16,8;4,2,2,8,8;8,8,2,8,16"
KP_STAGE_OCC=0 timeout 900 python tools/k1_ab.py --tag old --sizes 512,1024,2048,4096 --cfgs "$CF" > gpurun_out/ab_st_old.jsonl 2>&1
timeout 900 python tools/k1_ab.py --tag new --sizes 512,1024,2048,4096 --cfgs "$CF" > gpurun_out/ab_st_new.jsonl 2>&1
