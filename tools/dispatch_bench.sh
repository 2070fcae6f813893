#!/bin/sh
# Build and run tools/dispatch_bench.cpp against the in-tree libkp.so and
# libkp_lean.so (on the GPU box: the enqueue part needs a device).
#   sh tools/dispatch_bench.sh > gpurun_out/dispatch.jsonl
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
for lib in kp kp_lean; do
  g++ -O2 -std=c++17 -I "$ROOT/include" "$ROOT/tools/dispatch_bench.cpp" \
      -L "$ROOT/paper_2003_06795_b200" -l$lib -Wl,-rpath,"$ROOT/paper_2003_06795_b200" \
      -I /usr/local/cuda/include -L /usr/local/cuda/lib64 -lcudart -o /tmp/dispatch_bench_$lib
  printf '{"library": "lib%s.so", "result": ' $lib
  /tmp/dispatch_bench_$lib | tr -d '\n'
  printf '}\n'
done
