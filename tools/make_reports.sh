#!/bin/sh
# Regenerate reports/<variant>/{counts,curves,variance,classifiers}.csv for
# all 12 family x layout variants from the committed datasets (CPU only; the
# reference's report functions, report.py:42-93, restated in the package).
#   sh tools/make_reports.sh            (all variants, in parallel)
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
cd "$ROOT"
TMP=$(mktemp -d)
for fam in f32 tf32 bf16; do for t in nn nt tn tt; do
  gzip -dc data/b200_${fam}_${t}_train.csv.gz > $TMP/${fam}_${t}.csv
  ( python -m paper_2003_06795_b200 report --data $TMP/${fam}_${t}.csv \
      --out-dir reports/${fam}_${t} --budgets 2,4,6,8,10,12 \
      --kinds decision-tree,random-forest,knn1,knn3,linear-svm --epochs 20 --trees 20 \
      > /tmp/report_${fam}_${t}.log 2>&1; echo "${fam}_${t} rc=$?" ) &
done; wait; done
