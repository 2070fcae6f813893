for fam in bf16 tf32; do
 for mode in 0 1; do
  for cfg in 4,1,4,8,8 2,1,2,8,8 4,1,8,8,8 8,1,4,16,16; do
   python tools/run_config.py --family $fam --trans nt --mkn 392,4608,512 --cfg $cfg --tc-split $mode --iters 2 | sed "s/^/split=$mode /"
  done
 done
done
