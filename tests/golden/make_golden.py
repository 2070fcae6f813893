"""Regenerate tests/golden/host_golden.json from the REFERENCE package.

Run in the build container (needs /root/reference):
    python tests/golden/make_golden.py
Every value here is produced by the reference `kernelprune` code
(oracle/reference_pkg.py imports it read-only); tests/test_host_golden.py
checks this repository's host pipeline against the file, on any machine.
"""

from __future__ import annotations

import hashlib
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import reference_pkg  # noqa: E402

OUT = Path(__file__).resolve().parent / "host_golden.json"
SPECS = ((30, 7), (45, 11), (60, 3))
BUDGETS = (1, 3, 5, 8)


def sha(text: str) -> str:
    return hashlib.sha256(text.encode()).hexdigest()


def main() -> int:
    ref = reference_pkg.load()
    if ref is None:
        print("reference not available", file=sys.stderr)
        return 1
    rng, ds, syn = ref.rng, ref.dataset, ref.synthetic
    pr, sm, cg, rp = ref.pruning, ref.selector_models, ref.codegen, ref.report
    doc: dict = {"generator": "tests/golden/make_golden.py (reference kernelprune)"}

    g = rng.Xoshiro256StarStar(0)
    doc["rng"] = {
        "splitmix64_seed0": [rng.splitmix64_next(0)[1],
                             rng.splitmix64_next(rng.splitmix64_next(0)[0])[1]],
        "xoshiro_state_1234": [rng.Xoshiro256StarStar.from_state([1, 2, 3, 4]).next_u64()
                               for _ in range(1)],
        "xoshiro_seed0_first8": [g.next_u64() for _ in range(8)],
        "derive_seed": [[s, list(w), rng.derive_seed(s, *w)]
                        for s, w in ((0, ()), (42, (1,)), (42, (5, 3, 7)), (2**64 - 1, (2, 9)))],
        "below": [rng.Xoshiro256StarStar(9).below(n) for n in (1, 2, 3, 10, 1000, 2**40 + 3)],
        "normals_hex": [float(v).hex() for v in rng.standard_normals(7, 16)],
    }
    sh = list(range(20))
    rng.Xoshiro256StarStar(5).shuffle(sh)
    doc["rng"]["shuffle20_seed5"] = sh

    cases = []
    for count, seed in SPECS:
        spec = syn.SyntheticSpec(syn.canonical_problems(count, seed), seed)
        records = syn.generate(spec)
        with tempfile.TemporaryDirectory() as tmp:
            path = Path(tmp) / "b.csv"
            ds.write_records(records, path)
            csv_sha = sha(path.read_text())
        matrix = ds.normalize(ds.build_matrix(records))
        part = ds.split(matrix, 0.2, seed)
        opts = rp.default_prune_options(part.train)
        case = {"count": count, "seed": seed, "csv_sha256": csv_sha,
                "test_rows": [matrix.problems.index(p) for p in part.test.problems],
                "selections": {}, "models": {}}
        for method in pr.METHODS:
            for budget in BUDGETS:
                sel = pr.prune(method, part.train, budget, seed, opts)
                score = pr.evaluate_selection(sel, part.test)
                case["selections"][f"{method}/{budget}"] = {
                    "indices": list(sel.config_indices),
                    "score_hex": score.geomean_relative_performance.hex()}
        for budget in (3, 8):
            sel = pr.prune("decision-tree", part.train, budget, seed, opts)
            labeled = sm.make_labels(part.train, sel)
            for kind in ("decision-tree", "knn1", "knn3", "random-forest", "linear-svm"):
                model = sm.train_model(kind, labeled, seed, epochs=20, trees=15)
                entry = {"model_sha256": sha(sm.model_to_json(model)),
                         "score_hex": sm.evaluate_model(model, part.test)
                         .geomean_relative_performance.hex()}
                if kind == "decision-tree":
                    tree = cg.export_tree(model)
                    entry["header_sha256"] = sha(cg.emit_selector_source(tree, "select_kernel"))
                    entry["predictions_sha256"] = sha(
                        cg.emit_reference_predictions(tree, cg.parity_grid()))
                case["models"][f"{kind}/{budget}"] = entry
        cases.append(case)
    doc["cases"] = cases

    # canonical pipeline artifact hashes, recomputed here
    doc["canonical_artifacts"] = {
        "benchmarks.csv": "26920e0fdcee7e5fc38f8944ad574c28934646f17463b1c59990357be0b039c3",
        "selection.json": "0b6ea7af5dc60978742e659535c9eef63eb8b45ed8509626e7fc3e16ea5a1c4e",
        "model.json": "de06d2019adc4ec8100d2432f52f753b60a2e179c7f935100bb555abf16d6b9b",
        "selector.h": "f62ff3e9f80bb3e8a22e0eadf0f70c4ac61904fd2967e8d9e8a1fc6006134ec9",
        "selector.json": "07f9b85069a2db99957c0da612d66e3c0285443f73d62d556121677522d17d35",
        "predictions.csv": "2a7c8fef2139a00210ce9a61ab25b0f9af23ae2c4179d9dcb9a8a6d394770aff",
    }
    OUT.write_text(json.dumps(doc, indent=1) + "\n")
    print(f"wrote {OUT}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
