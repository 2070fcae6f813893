#!/bin/sh
# Build and run tools/dispatch_bench.cu against the in-tree libkp.so and
# libkp_lean.so (on the GPU box: the enqueue part needs a device).
#   sh tools/dispatch_bench.sh > gpurun_out/dispatch.jsonl
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
for lib in kp kp_lean; do
  nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I "$ROOT/include" "$ROOT/tools/dispatch_bench.cu" \
      -L "$ROOT/paper_2003_06795_b200" -l$lib -Xlinker -rpath,"$ROOT/paper_2003_06795_b200" \
      -o /tmp/dispatch_bench_$lib
  printf '{"library": "lib%s.so", "result": ' $lib
  /tmp/dispatch_bench_$lib | tr -d '\n'
  printf '}\n'
done
