"""bench.py contract on CPU: the committed bench lines carry every key the
driver and the judge read, and the host-side helpers (clock sampling, the
e2e row blocking) behave as documented -- no GPU needed."""

import json
import sys
import types
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
        "gpu_launches", "clocks", "roofline", "cpu_baseline")


BENCH = ROOT / "profiles" / "bench_r02.json"
BENCH_REF = ROOT / "profiles" / "bench_ref_r02.json"


def test_committed_bench_line_has_contract_keys():
    line = json.loads(BENCH.read_text())
    for k in KEYS:
        assert k in line, k
    assert line["warmup"] >= 3 and line["gpu_launches"] > 0
    assert set(line["e2e"]) >= {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"}
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0
    roof = line["roofline"]
    assert set(roof) >= {"bound", "achieved", "peak", "unit", "frac", "traffic"}
    assert abs(roof["frac"] - roof["achieved"] / roof["peak"]) < 1e-9
    assert set(line["cpu_baseline"]) >= {"value", "unit", "cores", "kind", "sample"}
    assert line["clocks"]["samples"] >= 1 and line["clocks"]["sm_mhz"]
    assert "workload" in line["config"] and "l2" in line["config"]


def test_reference_arm_line():
    line = json.loads(BENCH_REF.read_text())
    assert line["impl"] == "reference"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["cpu_baseline"]["value"] == line["value"]
    assert line["cpu_baseline"]["kind"] == "port"   # the oracle restatement


def test_both_arms_share_config_and_metric():
    ours, ref = json.loads(BENCH.read_text()), json.loads(BENCH_REF.read_text())
    assert ours["config"] == ref["config"]
    for k in ("metric", "unit", "higher_is_better", "steps", "warmup", "n_gpus"):
        assert ours[k] == ref[k], k
    import bench
    assert bench.bench_config(1) == ours["config"]


def test_roofline_blocks_follow_from_their_numbers():
    import math
    line = json.loads(BENCH.read_text())
    roof = line["roofline"]
    # FP32 headline against the nominal FMA-pipe peak, the >= 12 ms probe beside it
    assert abs(roof["peak"] - line["peaks"]["fp32_nominal"]) < 1e-9
    assert abs(roof["frac_of_measured"] - roof["achieved"] / roof["peak_measured"]) < 1e-9
    cpu = line["cpu_baseline"]
    assert cpu["kind"] == "port" and cpu["one_core"]["cores"] == 1 and cpu["cores"] >= 1
    large = line["large_sizes"]
    assert large["clocks"]["samples"] >= 1
    assert not set(large["clocks"]["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown",
                                                  "sw_thermal_slowdown"}
    for row in large["rows"]:
        peak = large["summary"][row["family"]]["peak"]
        assert abs(row["selected_frac"] - row["selected_tflops"] / peak) < 1e-9
        assert row["best_tflops"] >= row["selected_tflops"]
    for fam, blk in line["network_roofline"].items():
        fr = [r["frac"] for r in blk["rows"]]
        assert abs(blk["geomean_frac"] - math.exp(sum(map(math.log, fr)) / len(fr))) < 1e-9
        assert all(r["mkn"][0] * r["mkn"][1] * r["mkn"][2] * 2 >= 1e9 for r in blk["rows"])
    for fam, blk in line["held_out"].items():
        for part in ("held_out_split", "unseen_batch32_64"):
            assert 0 < blk[part]["pct_oracle_best"] <= 100.0
    for fam, blk in line["small_m"].items():
        assert all(r["mkn"][0] <= 16 for r in blk["rows"])


def test_clock_sampler_keeps_samples_inside_the_region(tmp_path):
    import bench
    cs = bench.ClockSampler()
    cs.path = str(tmp_path / "clk.csv")
    rows = []
    for i, mhz in enumerate((1000, 1965, 1965, 1965, 1200)):
        rows.append(f"2026/10/17 12:00:00.{100 * i + 50:03d}, 0, {mhz}, 1965, 900.0, 0x0, "
                    f"Not Active, Not Active, Not Active, {'Active' if i == 2 else 'Not Active'}")
    Path(cs.path).write_text("\n".join(rows) + "\n")
    import datetime
    t0 = datetime.datetime(2026, 10, 17, 12, 0, 0).timestamp()
    cs.proc = types.SimpleNamespace(terminate=lambda: None, wait=lambda: None)
    cs.begin, cs.end = t0 + 0.1, t0 + 0.36
    rec = cs.stop(0)
    assert rec["samples"] == 3 and rec["sm_mhz"] == 1965 and rec["reasons"] == ["sw_power_cap"]
    # a region shorter than the sampling period keeps the bracketing samples
    Path(cs.path).write_text("\n".join(rows) + "\n")
    cs.begin, cs.end = t0 + 0.16, t0 + 0.17
    rec = cs.stop(0)
    assert rec["samples"] == 2 and "bracketing" in rec["sampling"]


@pytest.mark.parametrize("m,k,want", [(2048, 2048, 4), (2100, 700, 2), (512, 512, 1), (300, 27, 1),
                                      (100000, 64, 7)])
def test_pinned_pipeline_row_blocks(m, k, want):
    torch = pytest.importorskip("torch")
    from paper_2003_06795_b200.gemm import PinnedPipeline
    fake = types.SimpleNamespace(family="f32", CHUNK_BYTES=PinnedPipeline.CHUNK_BYTES,
                                 MIN_ROWS=PinnedPipeline.MIN_ROWS)
    blocks = PinnedPipeline._blocks(fake, torch.empty((m, k)))
    assert blocks[0][0] == 0 and blocks[-1][1] == m
    assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
    assert len(blocks) == want


def test_cpu_port_baseline_runs_on_cpu(monkeypatch):
    """The CPU arm times the oracle restatement (kind "port") at all host
    threads and at one thread, with numpy/OpenBLAS only as context; on a
    tiny square set it runs here."""
    import bench
    monkeypatch.setattr(bench, "SIZES", (16, 32))
    line = bench.cpu_baseline(0.05)
    assert line["kind"] == "port" and line["unit"] == "TFLOP/s"
    assert line["value"] > 0 and line["one_core"]["value"] > 0 and line["one_core"]["cores"] == 1
    assert line["cpu_blas"]["value"] > 0
    assert "oracle/gemm_ref.c" in line["sample"]


def test_reference_arm_runs_on_cpu(monkeypatch, capsys):
    import bench
    monkeypatch.setattr(bench, "SIZES", (16, 32))
    monkeypatch.delenv("RANK", raising=False)
    args = bench.parse_args(["--impl", "reference", "--steps", "2", "--warmup", "3"])
    assert bench.run_reference(args) == 0
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["config"] == bench.bench_config(1)
    assert line["e2e"]["value"] == line["value"] and line["cpu_baseline"]["kind"] == "port"
