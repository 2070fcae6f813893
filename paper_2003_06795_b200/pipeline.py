"""Measured dataset -> pruned kernel set -> decision tree -> compiled selector.

The paper's deployment flow on B200 data, using only the
reference-API host pipeline (dataset.split, pruning.prune,
selector_models.train_model, codegen.export_tree / emit_selector_source):

    python -m paper_2003_06795_b200.pipeline \
        --data data/b200_f32_nn_networks.csv.gz --family f32 --trans nn \
        --method pca-kmeans --budget 8

writes selectors/<family>_<trans>/{selection,model}.json + a score report,
installs csrc/generated/select_<family>_<trans>.h, regenerates the selector
table and (unless --no-build) rebuilds libkp.so.
"""

from __future__ import annotations

import argparse
import gzip
import json
import shutil
import sys
import tempfile
from pathlib import Path

import numpy as np

from . import dataset, libgen, pruning, report, selector_models

ROOT = Path(__file__).resolve().parent.parent
SEL_DIR = ROOT / "selectors"


def materialize(path) -> Path:
    """Plain-CSV path for `path` (decompressing .gz into a temp file)."""
    path = Path(path)
    if path.suffix != ".gz":
        return path
    tmp = Path(tempfile.mkdtemp()) / path.stem
    with gzip.open(path, "rb") as src, open(tmp, "wb") as dst:
        shutil.copyfileobj(src, dst)
    return tmp


def load_matrix(path) -> dataset.PerformanceMatrix:
    return dataset.normalize(dataset.load_matrix(materialize(path)))


def choose(split: dataset.DataSplit, methods, budgets, seed: int):
    """Score every (method, budget): selection ceiling and decision-tree
    selector on the held-out side (reported; the deployed choice is fixed by
    the caller's --method/--budget, so the test side is not used to pick)."""
    opts = report.default_prune_options(split.train)
    rows = []
    for method in methods:
        for budget in budgets:
            sel = pruning.prune(method, split.train, budget, seed, opts)
            model = selector_models.train_model(
                "decision-tree", selector_models.make_labels(split.train, sel), seed)
            rows.append({"method": method, "budget": budget,
                         "ceiling": pruning.evaluate_selection(sel, split.test).percent,
                         "decision_tree": selector_models.evaluate_model(model, split.test).percent})
    return rows


def cross_validate(train: dataset.PerformanceMatrix, methods, budgets, seed: int,
                   folds: int = 5) -> list[dict]:
    """k-fold CV of (pruning method, budget) -> decision-tree selector score,
    on the TRAINING side only (the held-out split is never consulted). Folds
    come from the reference's seeded shuffle (dataset.split on the train
    matrix with a per-fold seed)."""
    rows = []
    for method in methods:
        for budget in budgets:
            scores = []
            for f in range(folds):
                part = dataset.split(train, 1.0 / folds, seed * 1000 + f)
                opts = report.default_prune_options(part.train)
                sel = pruning.prune(method, part.train, budget, seed, opts)
                model = selector_models.train_model(
                    "decision-tree", selector_models.make_labels(part.train, sel), seed)
                scores.append(selector_models.evaluate_model(model, part.test)
                              .geomean_relative_performance)
            rows.append({"method": method, "budget": budget,
                         "cv_geomean": float(np.exp(np.mean(np.log(scores))))})
    return rows


def build_selector(data, family: str, trans: str, method: str, budget: int, seed: int = 42,
                   test_fraction: float = 0.2, out_dir: Path | None = None) -> dict:
    """Prune + train + report. method == "auto": pick (method, budget <= the
    given budget) by 5-fold cross-validation on the training split."""
    matrix = load_matrix(data)
    split = dataset.split(matrix, test_fraction, seed)
    cv = None
    if method == "auto":
        budgets = tuple(b for b in (4, 6, 8) if b <= budget) or (budget,)
        cv = cross_validate(split.train, ("top-count", "kmeans", "pca-kmeans", "decision-tree"),
                            budgets, seed)
        best = max(cv, key=lambda r: (r["cv_geomean"], -r["budget"]))
        method, budget = best["method"], best["budget"]
    opts = report.default_prune_options(split.train)
    sel = pruning.prune(method, split.train, budget, seed, opts)
    model = selector_models.train_model(
        "decision-tree", selector_models.make_labels(split.train, sel), seed)
    out_dir = out_dir or SEL_DIR / f"{family}_{trans}"
    out_dir.mkdir(parents=True, exist_ok=True)
    pruning.save_selection(sel, split.train.configs, out_dir / "selection.json")
    selector_models.save_model(model, out_dir / "model.json")
    summary = {
        "data": str(data), "family": family, "trans": trans, "method": method, "budget": budget,
        "seed": seed, "test_fraction": test_fraction, "problems": len(matrix.problems),
        "configs": len(matrix.configs),
        "selected": [split.train.configs[j].as_tuple() for j in sel.config_indices],
        "ceiling_pct": pruning.evaluate_selection(sel, split.test).percent,
        "decision_tree_pct": selector_models.evaluate_model(model, split.test).percent,
        "train_decision_tree_pct": selector_models.evaluate_model(model, split.train).percent,
    }
    if cv is not None:
        summary["cross_validation"] = cv
    (out_dir / "summary.json").write_text(json.dumps(summary, indent=2) + "\n")
    return summary


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--data", required=True)
    ap.add_argument("--family", default="f32", choices=tuple(libgen.FAMILY_IDS))
    ap.add_argument("--trans", default="nn", choices=libgen.TRANS)
    ap.add_argument("--method", default="auto", choices=pruning.METHODS + ("auto",),
                    help="pruning method; auto = 5-fold CV on the training split")
    ap.add_argument("--budget", type=int, default=8)
    ap.add_argument("--batch", type=int, default=1,
                    help="batch count of a strided-batched dataset (selector variant _b<N>)")
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--survey", action="store_true", help="also score every method x budget")
    ap.add_argument("--no-build", action="store_true")
    args = ap.parse_args(argv)
    variant = args.trans if args.batch == 1 else f"{args.trans}_b{args.batch}"
    summary = build_selector(args.data, args.family, variant, args.method, args.budget,
                             args.seed)
    print(json.dumps(summary, indent=2))
    out_dir = SEL_DIR / f"{args.family}_{variant}"
    if args.survey:
        split = dataset.split(load_matrix(args.data), 0.2, args.seed)
        rows = choose(split, ("top-count", "kmeans", "pca-kmeans", "decision-tree"),
                      (4, 6, 8), args.seed)
        (out_dir / "survey.json").write_text(json.dumps(rows, indent=2) + "\n")
        for r in rows:
            print(f"{r['method']:14s} {r['budget']:2d} ceiling {r['ceiling']:6.2f} "
                  f"dt {r['decision_tree']:6.2f}")
    libgen.install_model(out_dir / "model.json", args.family, variant)
    libgen.write_selector_table()
    if not args.no_build:
        from .build import build_library
        build_library()
    return 0


if __name__ == "__main__":
    sys.exit(main())
