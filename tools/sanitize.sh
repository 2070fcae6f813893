#!/bin/sh
# compute-sanitizer sweep over odd shapes for every family (race
# detection / memcheck). Run on the GPU box:  sh tools/sanitize.sh > gpurun_out/sanitize.log
set -u
CS=${CS:-compute-sanitizer}
run() { echo "== $*"; timeout 300 $CS "$@" 2>&1 | grep -E "ERROR SUMMARY|error|TFLOP|launched" | head -5; }
for tool in memcheck racecheck; do
  for t in nn nt tn tt; do
    run --tool $tool python tools/run_config.py --family f32 --trans $t --cfg 8,8,8,16,16 --mkn 17,27,2049 --iters 1 --no-time
    run --tool $tool python tools/run_config.py --family f32 --trans $t --cfg 1,1,2,128,1 --mkn 129,15,33 --iters 1 --no-time
  done
done
# ordered stream-K hand-off (forced) and the transposed B staging (m >= 2048)
for tool in memcheck racecheck; do
  run --tool $tool python tools/run_config.py --family f32 --trans nn --cfg 8,8,8,16,16 --mkn 300,77,200 --schedule 2 --iters 2 --no-time
  run --tool $tool python tools/run_config.py --family f32 --trans tn --cfg 4,4,4,8,8 --mkn 130,64,70 --schedule 2 --iters 2 --no-time
  run --tool $tool python tools/run_config.py --family f32 --trans nt --cfg 4,8,8,16,16 --mkn 2053,45,37 --iters 1 --no-time
  run --tool $tool python tools/run_config.py --family f32 --trans tt --cfg 1,1,2,128,1 --mkn 2053,45,37 --iters 1 --no-time
done
for fam in tf32 bf16; do
  for t in nn tt; do
    run --tool memcheck python tools/run_config.py --family $fam --trans $t --cfg 2,1,2,8,8 --mkn 200,136,264 --iters 1 --no-time
  done
done
# persistent 1-CTA (NBUF = 2, double-buffered TMEM accumulator) and CTA-pair
# kernels with several tiles per CTA / pair (round-2 parity gap)
for tool in memcheck racecheck; do
  for fam in tf32 bf16; do
    run --tool $tool python tools/run_config.py --family $fam --trans nn --cfg 1,1,1,16,16 --mkn 1536,136,1536 --iters 1 --no-time
    run --tool $tool python tools/run_config.py --family $fam --trans tn --cfg 4,1,4,16,16 --mkn 2200,72,2112 --iters 1 --no-time
    run --tool $tool python tools/run_config.py --family $fam --trans nt --cfg 2,2,4,16,16 --mkn 4096,128,2048 --iters 1 --no-time
    run --tool $tool python tools/run_config.py --family $fam --trans tt --cfg 4,2,8,16,16 --mkn 4096,96,4352 --iters 1 --no-time
  done
done
# small-M path (K6): B normal / transposed, vector and scalar (unaligned)
# kernels, split-K last-CTA finish, fp32 and bf16 (round 2)
for tool in memcheck racecheck; do
  for fam in f32 bf16; do
    for t in nn nt tn tt; do
      run --tool $tool python tools/run_config.py --family $fam --trans $t --cfg 0,0,0,0,0 --mkn 5,3000,520 --iters 2 --no-time
    done
    run --tool $tool python tools/run_config.py --family $fam --trans nn --cfg 0,0,0,0,0 --mkn 16,4096,1000 --iters 2 --no-time
    run --tool $tool python tools/run_config.py --family $fam --trans nt --cfg 0,0,0,0,0 --mkn 1,25088,512 --iters 2 --no-time
    run --tool $tool python tools/run_config.py --family $fam --trans nn --cfg 0,0,0,0,0 --mkn 3,777,333 --iters 2 --no-time
  done
done
# tcgen05 TMA-store epilogue and split-K partials through TMA (round 2)
for tool in memcheck racecheck; do
  run --tool $tool python tools/run_config.py --family bf16 --trans nn --cfg 1,1,4,8,8 --mkn 1000,520,1000 --iters 2 --no-time
  run --tool $tool python tools/run_config.py --family tf32 --trans tt --cfg 2,1,4,8,8 --mkn 392,4608,512 --iters 2 --no-time
done
