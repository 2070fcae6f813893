for fam in tf32 bf16; do for t in nn nt tn tt; do
  timeout 900 python -m paper_2003_06795_b200 sweep --shapes networks-unseen --family $fam --trans $t --out gpurun_out/b200_${fam}_${t}_unseen.csv --sidecar gpurun_out/b200_${fam}_${t}_unseen.sidecar.json 2>&1 | tail -1
done; done
for t in tn tt; do
  timeout 2400 python -m paper_2003_06795_b200 sweep --shapes networks-unseen --family f32 --trans $t --out gpurun_out/b200_f32_${t}_unseen.csv --sidecar gpurun_out/b200_f32_${t}_unseen.sidecar.json 2>&1 | tail -1
done
