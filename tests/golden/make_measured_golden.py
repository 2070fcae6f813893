"""Regenerate tests/golden/measured_golden.json: the REFERENCE package's
selections / models / headers on the measured B200 datasets in data/.

    python tests/golden/make_measured_golden.py     (needs /root/reference)

north_star: "selector decisions plus pruned kernel sets must be bit-exact given
the same timing dataset" -- tests/test_measured_golden.py replays this on any
machine with this repository's host pipeline.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import reference_pkg  # noqa: E402
from paper_2003_06795_b200.pipeline import materialize  # noqa: E402  (gunzip helper only)

OUT = Path(__file__).resolve().parent / "measured_golden.json"
METHODS = ("top-count", "kmeans", "pca-kmeans", "decision-tree")
BUDGETS = (4, 6, 8)


def sha(text: str) -> str:
    return hashlib.sha256(text.encode()).hexdigest()


def main() -> int:
    ref = reference_pkg.load()
    if ref is None:
        print("reference not available", file=sys.stderr)
        return 1
    ds, pr, sm, cg, rp = ref.dataset, ref.pruning, ref.selector_models, ref.codegen, ref.report
    doc = {"generator": "tests/golden/make_measured_golden.py (reference kernelprune)",
           "datasets": {}}
    for path in sorted((ROOT / "data").glob("b200_*.csv.gz")):
        csv_path = materialize(path)
        matrix = ds.normalize(ds.build_matrix(ds.load_records(csv_path)))
        part = ds.split(matrix, 0.2, 42)
        opts = rp.default_prune_options(part.train)
        entry = {"csv_sha256": sha(csv_path.read_text()), "cases": {}}
        for method in METHODS:
            for budget in BUDGETS:
                if budget > len(matrix.configs):
                    continue
                sel = pr.prune(method, part.train, budget, 42, opts)
                model = sm.train_model("decision-tree", sm.make_labels(part.train, sel), 42)
                tree = cg.export_tree(model)
                entry["cases"][f"{method}/{budget}"] = {
                    "indices": list(sel.config_indices),
                    "ceiling_hex": pr.evaluate_selection(sel, part.test)
                    .geomean_relative_performance.hex(),
                    "model_sha256": sha(sm.model_to_json(model)),
                    "header_sha256": sha(cg.emit_selector_source(tree, "select_kernel")),
                    "score_hex": sm.evaluate_model(model, part.test)
                    .geomean_relative_performance.hex(),
                }
        doc["datasets"][path.name] = entry
        print(f"{path.name}: {len(entry['cases'])} cases")
    OUT.write_text(json.dumps(doc, indent=1) + "\n")
    print(f"wrote {OUT}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
