"""Host pipeline vs golden vectors produced by the REFERENCE package
(tests/golden/make_golden.py). Runs anywhere (no /root/reference needed):
selections, models, headers and predictions must be bit-identical."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2003_06795_b200 import (cli, codegen, dataset, pruning, report, rng,
                                   selector_models, synthetic)

GOLDEN = json.loads((Path(__file__).parent / "golden" / "host_golden.json").read_text())
CANONICAL_SPEC = Path(__file__).parent / "golden" / "canonical.json"


def sha(text: str) -> str:
    return hashlib.sha256(text.encode()).hexdigest()


def test_rng_vectors():
    g = GOLDEN["rng"]
    s1, o1 = rng.splitmix64_next(0)
    assert [o1, rng.splitmix64_next(s1)[1]] == g["splitmix64_seed0"]
    assert rng.Xoshiro256StarStar.from_state([1, 2, 3, 4]).next_u64() == g["xoshiro_state_1234"][0]
    x = rng.Xoshiro256StarStar(0)
    assert [x.next_u64() for _ in range(8)] == g["xoshiro_seed0_first8"]
    for seed, words, want in g["derive_seed"]:
        assert rng.derive_seed(seed, *words) == want
        assert int(rng.derive_seed_array(seed, *words)) == want
    assert [rng.Xoshiro256StarStar(9).below(n) for n in (1, 2, 3, 10, 1000, 2**40 + 3)] == g["below"]
    assert [float(v).hex() for v in rng.standard_normals(7, 16)] == g["normals_hex"]
    sh = list(range(20))
    rng.Xoshiro256StarStar(5).shuffle(sh)
    assert sh == g["shuffle20_seed5"]


def test_reference_known_answers():
    """The reference suite's own vectors (reference tests/test_rng.py:11-29)."""
    s, outs = 0, []
    for _ in range(3):
        s, o = rng.splitmix64_next(s)
        outs.append(o)
    assert tuple(outs) == (0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F)
    gen = rng.Xoshiro256StarStar.from_state([1, 2, 3, 4])
    assert [gen.next_u64() for _ in range(3)] == [11520, 0, 1509978240]


@pytest.mark.parametrize("case", GOLDEN["cases"], ids=lambda c: f"spec{c['count']}_{c['seed']}")
def test_selection_and_models_bit_exact(case, tmp_path):
    count, seed = case["count"], case["seed"]
    spec = synthetic.SyntheticSpec(synthetic.canonical_problems(count, seed), seed)
    records = synthetic.generate(spec)
    path = tmp_path / "b.csv"
    dataset.write_records(records, path)
    assert sha(path.read_text()) == case["csv_sha256"]
    matrix = dataset.normalize(dataset.build_matrix(dataset.load_records(path)))
    part = dataset.split(matrix, 0.2, seed)
    assert [matrix.problems.index(p) for p in part.test.problems] == case["test_rows"]
    opts = report.default_prune_options(part.train)
    for key, want in case["selections"].items():
        method, budget = key.split("/")
        sel = pruning.prune(method, part.train, int(budget), seed, opts)
        assert list(sel.config_indices) == want["indices"], key
        got = pruning.evaluate_selection(sel, part.test).geomean_relative_performance
        assert got.hex() == want["score_hex"], key
    for key, want in case["models"].items():
        kind, budget = key.split("/")
        sel = pruning.prune("decision-tree", part.train, int(budget), seed, opts)
        labeled = selector_models.make_labels(part.train, sel)
        model = selector_models.train_model(kind, labeled, seed, epochs=20, trees=15)
        assert sha(selector_models.model_to_json(model)) == want["model_sha256"], key
        score = selector_models.evaluate_model(model, part.test).geomean_relative_performance
        assert score.hex() == want["score_hex"], key
        if kind == "decision-tree":
            tree = codegen.export_tree(model)
            assert sha(codegen.emit_selector_source(tree, "select_kernel")) == want["header_sha256"]
            assert sha(codegen.emit_reference_predictions(tree, codegen.parity_grid())) == \
                want["predictions_sha256"]


def test_canonical_pipeline_artifacts(tmp_path):
    """The reference's canonical pipeline (scripts/run_pipeline.py, seed 42,
    decision-tree, budget 8) reproduces its SHA-256s."""
    want = GOLDEN["canonical_artifacts"]
    d = tmp_path
    data = str(d / "benchmarks.csv")
    steps = [
        ["synth", "--spec", str(CANONICAL_SPEC), "--out", data],
        ["prune", "--data", data, "--method", "decision-tree", "--budget", "8", "--seed", "42",
         "--out", str(d / "selection.json")],
        ["train", "--data", data, "--selection", str(d / "selection.json"), "--kind",
         "decision-tree", "--seed", "42", "--out", str(d / "model.json")],
        ["codegen", "--model", str(d / "model.json"), "--header", str(d / "selector.h"),
         "--doc", str(d / "selector.json"), "--predictions", str(d / "predictions.csv")],
    ]
    for argv in steps:
        assert cli.main(argv) == 0, argv
    for name, digest in want.items():
        assert sha((d / name).read_text()) == digest, name


def test_canonical_scores(capsys, tmp_path):
    data = str(tmp_path / "b.csv")
    assert cli.main(["synth", "--spec", str(CANONICAL_SPEC), "--out", data]) == 0
    assert cli.main(["prune", "--data", data, "--method", "decision-tree", "--budget", "8",
                     "--out", str(tmp_path / "s.json")]) == 0
    assert cli.main(["evaluate", "--data", data, "--selection", str(tmp_path / "s.json")]) == 0
    assert cli.main(["train", "--data", data, "--selection", str(tmp_path / "s.json"),
                     "--kind", "decision-tree", "--out", str(tmp_path / "m.json")]) == 0
    assert cli.main(["evaluate", "--data", data, "--model", str(tmp_path / "m.json")]) == 0
    out = capsys.readouterr().out
    assert "score 91.53" in out and "score 86.08" in out
