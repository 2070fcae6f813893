#!/bin/sh
# compute-sanitizer sweep over odd shapes for every family (race
# detection / memcheck). Run on the GPU box:  sh tools/sanitize.sh > gpurun_out/sanitize.log
set -u
CS=${CS:-compute-sanitizer}
run() { echo "== $*"; timeout 300 $CS "$@" 2>&1 | grep -E "ERROR SUMMARY|error|TFLOP" | head -5; }
for tool in memcheck racecheck; do
  for t in nn nt tn tt; do
    run --tool $tool python tools/run_config.py --family f32 --trans $t --cfg 8,8,8,16,16 --mkn 17,27,2049 --iters 1
    run --tool $tool python tools/run_config.py --family f32 --trans $t --cfg 1,1,2,128,1 --mkn 129,15,33 --iters 1
  done
done
for fam in tf32 bf16; do
  for t in nn tt; do
    run --tool memcheck python tools/run_config.py --family $fam --trans $t --cfg 2,1,2,8,8 --mkn 200,136,264 --iters 1
  done
done
