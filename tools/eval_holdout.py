"""Generalisation of the compiled FP32 selectors to network shapes they never
saw: the batch-32/64 VGG16 / ResNet-50 / MobileNetV2 GEMMs (shapes.py
"networks-unseen"), swept with every config on the B200.

    python tools/eval_holdout.py data/b200_f32_nn_unseen.csv.gz:nn ... --out profiles/x.json

For each dataset: the committed selector (selectors/f32_<trans>/model.json,
the tree compiled into libkp.so) scored with the reference's own
evaluate_model (geomean over problems of selected / oracle-best GFLOP/s),
the ceiling of its pruned kernel set (evaluate_selection), and the rows.
"""

from __future__ import annotations

import argparse
import json
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2003_06795_b200 import pruning, selector_models  # noqa: E402
from paper_2003_06795_b200.pipeline import load_matrix  # noqa: E402


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("datasets", nargs="+", help="path:trans or path:family_trans")
    ap.add_argument("--out")
    args = ap.parse_args()
    doc = {"generator": "tools/eval_holdout.py", "variants": {}}
    for spec in args.datasets:
        path, variant = spec.rsplit(":", 1)
        variant = variant if "_" in variant else f"f32_{variant}"
        matrix = load_matrix(path)
        sel_dir = ROOT / "selectors" / variant
        model = selector_models.load_model(sel_dir / "model.json")
        selection = pruning.load_selection(sel_dir / "selection.json", matrix.configs)
        score = selector_models.evaluate_model(model, matrix)
        ceiling = pruning.evaluate_selection(selection, matrix)
        rows = []
        for i, prob in enumerate(matrix.problems):
            cfg = selector_models.predict(model, prob)
            j = matrix.configs.index(cfg)
            rows.append({"mkn": list(prob.as_tuple()), "selected": list(cfg.as_tuple()),
                         "pct_of_best": 100.0 * float(matrix.values[i][j])})
        worst = sorted(rows, key=lambda r: r["pct_of_best"])[:5]
        doc["variants"][variant] = {
            "dataset": path, "problems": len(matrix.problems),
            "selector_pct_oracle_best": score.percent, "pruned_set_ceiling_pct": ceiling.percent,
            "geomean_check": 100.0 * math.exp(sum(math.log(r["pct_of_best"] / 100.0)
                                                  for r in rows) / len(rows)),
            "worst": worst, "rows": rows}
        print(f"{variant}: {len(rows)} unseen problems, selector {score.percent:.2f} % of "
              f"oracle-best (pruned-set ceiling {ceiling.percent:.2f} %)")
    if args.out:
        Path(args.out).write_text(json.dumps(doc, indent=1) + "\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())
