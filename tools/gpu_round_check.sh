#!/bin/sh
# Round-end style check on one B200 (run through gpurun from the repo root):
#   gpurun --timeout 1800 -- 'mkdir -p gpurun_out; sh tools/gpu_round_check.sh'
# GPU test suite, smoke(), the default bench line, the reference arm and the
# ncu launch list of a short bench run, all into gpurun_out/.
set -u
timeout 1200 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-sweep \
    --cpu-seconds 1 > gpurun_out/bench_ncu.log 2>&1
tail -c 400 gpurun_out/bench.json
