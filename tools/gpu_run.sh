set -x
timeout 1200 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -3
for t in nn nt tn tt; do
  timeout 1500 python -m paper_2003_06795_b200 sweep --shapes networks+squares --family f32 --trans $t --out gpurun_out/b200_f32_${t}_train.csv --sidecar gpurun_out/b200_f32_${t}_train.sidecar.json > gpurun_out/sweep_$t.log 2>&1
  tail -1 gpurun_out/sweep_$t.log
done
