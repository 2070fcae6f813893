for t in nn nt; do
  timeout 1800 python -m paper_2003_06795_b200 sweep --shapes networks-unseen --family f32 --trans $t --out gpurun_out/b200_f32_${t}_unseen.csv --sidecar gpurun_out/b200_f32_${t}_unseen.sidecar.json > gpurun_out/sweep_u_$t.log 2>&1
  tail -1 gpurun_out/sweep_u_$t.log
done
