"""Bit-exact selections / selector models / headers on the MEASURED B200 timing
datasets, against the reference package's outputs on the same CSVs
(tests/golden/make_measured_golden.py)."""

import hashlib
import json
from pathlib import Path

import pytest

from paper_2003_06795_b200 import codegen, dataset, pruning, report, selector_models
from paper_2003_06795_b200.pipeline import materialize

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = json.loads((Path(__file__).parent / "golden" / "measured_golden.json").read_text())


def sha(text: str) -> str:
    return hashlib.sha256(text.encode()).hexdigest()


@pytest.mark.parametrize("name", sorted(GOLDEN["datasets"]))
def test_measured_dataset_pipeline_bit_exact(name):
    want = GOLDEN["datasets"][name]
    path = materialize(ROOT / "data" / name)
    assert sha(path.read_text()) == want["csv_sha256"], "dataset changed: rerun make_measured_golden"
    matrix = dataset.normalize(dataset.build_matrix(dataset.load_records(path)))
    part = dataset.split(matrix, 0.2, 42)
    opts = report.default_prune_options(part.train)
    for key, case in want["cases"].items():
        method, budget = key.split("/")
        sel = pruning.prune(method, part.train, int(budget), 42, opts)
        assert list(sel.config_indices) == case["indices"], key
        assert pruning.evaluate_selection(sel, part.test).geomean_relative_performance.hex() == \
            case["ceiling_hex"], key
        model = selector_models.train_model(
            "decision-tree", selector_models.make_labels(part.train, sel), 42)
        assert sha(selector_models.model_to_json(model)) == case["model_sha256"], key
        tree = codegen.export_tree(model)
        assert sha(codegen.emit_selector_source(tree, "select_kernel")) == case["header_sha256"]
        assert selector_models.evaluate_model(model, part.test).geomean_relative_performance \
            .hex() == case["score_hex"], key


def test_compiled_selector_matches_committed_model():
    """The header compiled into libkp.so is the codegen output of the
    committed selectors/<variant>/model.json (parity harness pattern,
    reference harness/parity_main.cpp)."""
    from paper_2003_06795_b200 import gemm, libgen
    for family, trans in libgen.installed():
        model = selector_models.load_model(ROOT / "selectors" / f"{family}_{trans}" / "model.json")
        doc = codegen.export_tree(model)
        header = (libgen.GEN_DIR / f"{libgen.symbol_for(family, trans)}.h").read_text()
        assert header == codegen.emit_selector_source(doc, libgen.symbol_for(family, trans))
        for p in codegen.parity_grid()[::97]:
            got = gemm.select(p.m, p.k, p.n, family=family, trans_a=trans[0] == "t",
                              trans_b=trans[1] == "t", batch=libgen.variant_batch(trans))
            assert got == codegen.traverse_document(doc, p.m, p.k, p.n), p


@pytest.mark.parametrize("variant", [f"{f}_{t}" for f in ("f32", "tf32", "bf16")
                                     for t in ("nn", "nt", "tn", "tt")])
def test_compiled_selector_generalises_to_unseen_batches(variant):
    """Each committed selector (trained on batch 1-16 network shapes +
    squares) on the batch-32/64 network shapes it never saw, measured on the
    B200 (data/b200_<variant>_unseen.csv.gz, tools/eval_holdout.py):
    north_star's >= 90 % geomean of the per-size oracle-best."""
    from paper_2003_06795_b200.pipeline import load_matrix
    matrix = load_matrix(ROOT / "data" / f"b200_{variant}_unseen.csv.gz")
    model = selector_models.load_model(ROOT / "selectors" / variant / "model.json")
    train = {p.as_tuple() for p in load_matrix(
        ROOT / "data" / f"b200_{variant}_train.csv.gz").problems}
    assert not train & {p.as_tuple() for p in matrix.problems}
    score = selector_models.evaluate_model(model, matrix).percent
    profile = json.loads((ROOT / "profiles" / "selector_unseen_r02.json").read_text())
    assert abs(score - profile["variants"][variant]["selector_pct_oracle_best"]) < 1e-9
    # out-of-sample generalisation (not a training target): every variant
    # within 15 % of its oracle-best; the cross-variant geomean is pinned
    # >= 90 below.  Round 2 tf32_tn reads 88.69 %.
    assert score >= 85.0, score


def test_unseen_geomean_over_variants():
    import math
    profile = json.loads((ROOT / "profiles" / "selector_unseen_r02.json").read_text())
    scores = [v["selector_pct_oracle_best"] for v in profile["variants"].values()]
    assert len(scores) == 12
    assert math.exp(sum(math.log(s) for s in scores) / len(scores)) >= 90.0
