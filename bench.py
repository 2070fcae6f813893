#!/usr/bin/env python
"""Headline benchmark: runtime-selected kernel TFLOP/s on the square size set,
with the full config sweep that defines the per-size oracle-best.

Workload (BASELINE.json configs[1], "full configuration sweep over a small
square-size set (64-2048) on 1 B200"):
  1. sweep: every config of the FP32 SIMT family (640) on every square size
     (64..2048) through the C++ timing loop (kp_sweep_problem) -> the per-size
     oracle-best and the sweep rate (configs*sizes/s);
  2. step (timed K times after W warm-ups): one pass over the square sizes,
     each GEMM dispatched by the compiled decision-tree selector
     (kp_gemm_auto -> csrc/generated/select_f32_nn.h), L2 flushed (256 MiB
     write) before every kernel, each kernel timed with CUDA events on the
     launching stream.
value = whole-job selected-kernel TFLOP/s (sum of flops / device time, max
over ranks); e2e = the same metric through the public host-buffer API
(gemm.matmul_pinned: pinned H2D, kernel, D2H inside the timed region).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
Multi-GPU (torchrun): each rank runs its own replica of the step (weak
scaling) and sweeps an interleaved 1/N of the configs (no data-path
collective; timings are gathered on the host).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = ("selected-kernel TFLOP/s (geomean % of oracle-best, % of roofline); "
          "sweep configs·sizes/s")
SIZES = (64, 128, 256, 512, 1024, 2048)
FLUSH_BYTES = 256 << 20


def parse_args(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--family", default="f32", choices=("f32",))
    ap.add_argument("--sweep-reps", type=int, default=3)
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the held-out / large-size / network roofline blocks")
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="bounded CPU-baseline sample length")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    return args


def flops_of(s: int) -> float:
    return 2.0 * s * s * s


# ----------------------------------------------------------- CPU baselines

def bench_config(world: int) -> dict:
    """The `config` object of both arms' lines (identical by construction)."""
    return {"workload": "BASELINE configs[1]: 640-config FP32 SIMT sweep + runtime-selected "
                        "FP32 GEMM pass over squares 64..2048 (NN, row-major)",
            "sizes": list(SIZES), "layout": "nn", "selector": "csrc/generated/select_f32_nn.h",
            "l2": f"flushed before every timed kernel ({FLUSH_BYTES >> 20} MiB write)",
            "parallelism": f"replicas x{world}"}


def cpu_mats(seed=0):
    import numpy as np
    rng = np.random.default_rng(seed)
    return [(rng.uniform(-1, 1, (s, s)).astype(np.float32),
             rng.uniform(-1, 1, (s, s)).astype(np.float32)) for s in SIZES]


def oracle_pass(mats) -> float:
    """One pass of the CPU restatement of the path (oracle/gemm_ref.c: the
    sequential-k fmaf GEMM K1 matches bit for bit, OpenMP over rows) over the
    square set; returns seconds."""
    from oracle.gemm_oracle import gemm_f32_exact
    t0 = time.perf_counter()
    for a, b in mats:
        s = a.shape[0]
        gemm_f32_exact(a, b, m=s, k=s, n=s)
    return time.perf_counter() - t0


def blas_pass(mats) -> float:
    """numpy float32 a @ b (OpenBLAS) over the square set: context only."""
    t0 = time.perf_counter()
    for a, b in mats:
        a @ b
    return time.perf_counter() - t0


def timed_passes(fn, mats, seconds: float, min_passes: int = 1):
    fn(mats)  # warm-up
    passes, spent = 0, 0.0
    while spent < seconds or passes < min_passes:
        spent += fn(mats)
        passes += 1
    return passes, spent


def cpu_baseline(seconds: float) -> dict:
    """The CPU port of the path (oracle/gemm_ref.c; kind "port": the reference
    ships no GEMM, so its restatement is the oracle) on the
    same squares, all host threads and 1 thread, each a bounded sample; plus
    numpy/OpenBLAS as a tuned-BLAS context figure (not a port)."""
    from oracle.gemm_oracle import set_threads
    mats = cpu_mats()
    work = sum(flops_of(s) for s in SIZES)
    cores = os.cpu_count() or 1
    prev = set_threads(cores)
    n_all, t_all = timed_passes(oracle_pass, mats, seconds)
    set_threads(1)
    n_one, t_one = timed_passes(oracle_pass, mats, seconds / 2)
    set_threads(prev)
    n_blas, t_blas = timed_passes(blas_pass, mats, 2.0, 3)
    return {"value": n_all * work / t_all / 1e12, "unit": "TFLOP/s", "cores": cores,
            "kind": "port",
            "sample": f"{n_all} passes of oracle/gemm_ref.c (sequential-k fmaf restatement, "
                      f"OpenMP, {cores} threads) over squares {list(SIZES)} ({t_all:.1f} s)",
            "one_core": {"value": n_one * work / t_one / 1e12, "unit": "TFLOP/s", "cores": 1,
                         "sample": f"{n_one} passes, 1 thread ({t_one:.1f} s)"},
            "cpu_blas": {"value": n_blas * work / t_blas / 1e12, "unit": "TFLOP/s",
                         "cores": cores, "what": "numpy float32 a@b (OpenBLAS, all threads), "
                         "context only: a tuned BLAS, not a port of the reference"}}


def host_pipeline(cells, configs) -> dict:
    """the reference's own CPU sweep path
    (synthetic.generate, the analytic stand-in for measuring a config) on the
    same configs x sizes cells, and the selection pipeline (prune -> decision
    tree -> C header) on this run's measured sweep -- the reference
    algorithms, restated bit-exactly in this package, timed on one host core."""
    import numpy as np
    from paper_2003_06795_b200 import codegen, dataset, pruning, selector_models, synthetic
    from paper_2003_06795_b200.dataset import ProblemSize
    problems = tuple(ProblemSize(s, s, s) for s in SIZES)
    spec = synthetic.SyntheticSpec(problems, seed=42)
    t0 = time.perf_counter()
    n = 0
    while time.perf_counter() - t0 < 1.0 or n == 0:
        synthetic.generate(spec)
        n += 1
    gen_s = (time.perf_counter() - t0) / n
    grid = np.array([[2.0 * s ** 3 / cells[(i, j)] for j in range(len(configs))]
                     for i, s in enumerate(SIZES)])
    matrix = dataset.normalize(dataset.PerformanceMatrix(problems, tuple(configs), grid))
    t0 = time.perf_counter()
    sel = pruning.prune("top-count", matrix, 4, 42)
    t1 = time.perf_counter()
    model = selector_models.train_model("decision-tree", selector_models.make_labels(matrix, sel), 42)
    t2 = time.perf_counter()
    codegen.emit_selector_source(codegen.export_tree(model), "select_kernel")
    t3 = time.perf_counter()
    return {"synthetic_generate_cells_per_s": len(problems) * len(configs) / gen_s,
            "prune_top_count_ms": 1e3 * (t1 - t0), "train_decision_tree_ms": 1e3 * (t2 - t1),
            "codegen_ms": 1e3 * (t3 - t2), "cores": 1,
            "what": "reference algorithms (bit-exact restatement) on this run's cells: the "
                    "analytic sweep stand-in, and prune/train/codegen on the measured sweep"}


def run_reference(args) -> int:
    """--impl reference: the CPU implementation of the path on the box's host
    cores -- the oracle port (oracle/gemm_ref.c, all host threads; the
    reference itself ships no GEMM to compile) over the same
    workload and config as the GPU arm; rank 0 only."""
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    from oracle.gemm_oracle import set_threads
    cores = os.cpu_count() or 1
    set_threads(cores)
    mats = cpu_mats()
    for _ in range(args.warmup):
        oracle_pass(mats)
    times = [oracle_pass(mats) for _ in range(args.steps)]
    total = sum(times)
    value = args.steps * sum(flops_of(s) for s in SIZES) / total / 1e12
    n_blas, t_blas = timed_passes(blas_pass, mats, 2.0, 3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": bench_config(args.gpus),
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": "port",
                         "sample": f"{args.steps} timed passes (after {args.warmup} warm-up) of "
                                   f"oracle/gemm_ref.c, the sequential-k fmaf restatement of the "
                                   f"GEMM, OpenMP over rows, {cores} threads, over the whole "
                                   f"square set"},
        "cpu_blas": {"value": sum(flops_of(s) for s in SIZES) * n_blas / t_blas / 1e12,
                     "unit": "TFLOP/s", "cores": cores,
                     "what": "numpy float32 a@b (OpenBLAS), context only"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# -------------------------------------------------------------- GPU helpers

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 20 ms. The sampler
    is started before the warm-up steps (nvidia-smi needs ~0.1 s to produce
    its first line) and the timed region is marked with host timestamps;
    samples inside the region are kept. A region shorter than the sampling
    period keeps the samples bracketing it (noted in the record)."""

    QUERY = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self):
        self.proc = None
        self.path = None
        self.begin = self.end = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def mark_begin(self):
        self.begin = time.time()

    def mark_end(self):
        self.end = time.time()

    def _rows(self, gpu_index):
        import datetime
        rows = []
        for line in Path(self.path).read_text().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 10 or f[1] != str(gpu_index):
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                rows.append((ts, float(f[2]), float(f[3]), f[6:10]))
            except ValueError:
                continue
        return rows

    def stop(self, gpu_index: int) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        end = self.end or time.time()
        deadline = time.time() + 2.0
        while time.time() < deadline:  # until a sample after the region exists
            rows = self._rows(gpu_index)
            if rows and rows[-1][0] >= end:
                break
            time.sleep(0.02)
        self.proc.terminate()
        self.proc.wait()
        rows = self._rows(gpu_index)
        os.unlink(self.path)
        begin = self.begin or end
        inside = [r for r in rows if begin <= r[0] <= end]
        note = "samples inside the timed region"
        if not inside and rows:
            before = [r for r in rows if r[0] < begin][-1:]
            after = [r for r in rows if r[0] > end][:1]
            inside = before + after
            note = "region shorter than the 20 ms period: the samples bracketing it"
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = {n for r in inside for n, v in zip(names, r[3]) if v.lower() == "active"}
        mhz = [r[1] for r in inside]
        return {"sm_mhz": statistics.median(mhz) if mhz else None,
                "sm_max_mhz": inside[-1][2] if inside else None,
                "reasons": sorted(reasons), "samples": len(inside), "sampling": note,
                "region_s": round(end - begin, 4)}


def gpu_index() -> int:
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if vis:
        ids = [v for v in vis.split(",") if v.strip()]
        if local < len(ids) and ids[local].strip().isdigit():
            return int(ids[local])
    return local


def traffic_for(cfg, size):
    """dram bytes/launch of this kernel from the committed ncu summary, if any."""
    path = ROOT / "profiles" / "ncu_traffic.json"
    if not path.exists():
        return None
    try:
        doc = json.loads(path.read_text())
    except ValueError:
        return None
    key = f"f32_nn_{size}_{'-'.join(str(v) for v in cfg.as_tuple())}"
    ent = doc.get(key)
    return None if ent is None else ent.get("dram_bytes")


def measured_peaks() -> dict:
    """MEASURED_PEAKS.json (driver-written), else the B200_PROFILING.md fallback."""
    path = ROOT / "MEASURED_PEAKS.json"
    if path.exists():
        doc = json.loads(path.read_text())
        return {"hbm_gbs": float(doc["hbm_gbs"]), "bf16_tflops": float(doc["bf16_tflops"]),
                "source": "MEASURED_PEAKS.json (of measured)"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0,
            "source": "B200_PROFILING.md fallback (of fallback)"}


def fp32_peaks() -> dict:
    """FP32 SIMT denominators: nominal = SMs x 128 FMA lanes x 2 x max SM clock
    (the headline `peak`), and the >= 12 ms FFMA/FFMA2 probe (kp_fp32_peak)
    measured in this process at the run's clocks."""
    import ctypes
    from paper_2003_06795_b200 import _native as nat
    sm, clk, cc = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    import torch
    nat.check(nat.lib().kp_device_info(torch.cuda.current_device(), ctypes.byref(sm),
                                       ctypes.byref(clk), ctypes.byref(cc)), "kp_device_info")
    probe = ctypes.c_double()
    nat.check(nat.lib().kp_fp32_peak(ctypes.byref(probe), None), "kp_fp32_peak")
    nominal = sm.value * 128 * 2 * (clk.value * 1e3) / 1e12
    return {"nominal": nominal, "measured": probe.value,
            "nominal_how": f"{sm.value} SMs x 128 FP32 lanes x 2 x {clk.value / 1e3:.0f} MHz",
            "measured_how": "kp_fp32_peak: full-chip FFMA / FFMA2 chains, >= 12 ms per launch, "
                            "best of 6"}


def tf32_peak_cublas(dev) -> float:
    """Dense TF32 denominator measured here: cuBLAS (torch.matmul, allow_tf32)
    on 8192^3 fp32 operands, best of 10 launches (CUDA events), like
    MEASURED_PEAKS' bf16 burst figure. MEASURED_PEAKS.json has no TF32 entry."""
    import torch
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        n = 8192
        a = torch.randn(n, n, device=dev)
        b = torch.randn(n, n, device=dev)
        c = torch.empty(n, n, device=dev)
        for _ in range(5):
            torch.matmul(a, b, out=c)
        best = float("inf")
        stream = torch.cuda.current_stream()
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            torch.matmul(a, b, out=c)
            e1.record(stream)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        del a, b, c
        return 2.0 * n ** 3 / (best * 1e-3) / 1e12
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def family_peaks(dev) -> dict:
    """{family: (peak TFLOP/s, source)} for the three families."""
    mp = measured_peaks()
    f32 = fp32_peaks()
    tf32 = tf32_peak_cublas(dev)
    return {"f32": (f32["nominal"], "nominal FP32: " + f32["nominal_how"]),
            "tf32": (tf32, "cuBLAS TF32 8192^3 measured in this run (burst, best of 10)"),
            "bf16": (mp["bf16_tflops"], mp["source"] + " bf16_tflops (burst)"),
            "_f32": f32, "_hbm_gbs": mp["hbm_gbs"], "_hbm_source": mp["source"]}


def tensor_peak(family: str, peaks: dict):
    return peaks[family]


def device_operands(m, k, n, family, trans_a, trans_b, dev, seed):
    """U[-1, 1) operands generated on the device in the layout asked for
    (tensor-core families get 16-byte padded row pitches, as the sweep)."""
    import torch
    gen = torch.Generator(device=dev).manual_seed(seed)
    dtype = torch.bfloat16 if family == "bf16" else torch.float32
    align = {"tf32": 4, "bf16": 8}.get(family, 1)

    def alloc(rows, cols):
        inner = -(-cols // align) * align
        full = torch.rand((rows, inner), generator=gen, device=dev) * 2 - 1
        return full.to(dtype)[:, :cols]
    a = alloc(k, m).t() if trans_a else alloc(m, k)
    b = alloc(n, k).t() if trans_b else alloc(k, n)
    return a, b


LARGE_CANDIDATES = {
    "f32": [(4, 8, 8, 32, 8), (4, 8, 8, 16, 16), (8, 8, 8, 16, 16), (2, 8, 8, 16, 16),
            (1, 8, 8, 32, 8), (4, 8, 4, 16, 16)],
    "tf32": [(4, 1, 8, 16, 16), (8, 1, 8, 16, 16), (4, 2, 8, 16, 16), (8, 2, 8, 16, 16),
             (1, 1, 4, 8, 8)],
    "bf16": [(4, 1, 8, 16, 16), (8, 1, 8, 16, 16), (4, 2, 8, 16, 16), (8, 2, 8, 16, 16),
             (1, 1, 4, 8, 8)],
}


def large_sizes_block(dev, peaks, sizes=(4096, 8192)) -> dict:
    """north_star's ">= 70 % of the roofline on large sizes": every family x
    operand layout at 4096^3 / 8192^3, the runtime-selected config (kp_select)
    and the best of a few large-tile configs, timed by the K4 loop (median of
    3 samples; operands >= the 126 MB L2), clock-sampled."""
    import torch
    from paper_2003_06795_b200 import gemm
    clocks = ClockSampler()
    clocks.start()
    time.sleep(0.3)
    clocks.mark_begin()
    rows = []
    for fam in ("f32", "tf32", "bf16"):
        peak = peaks[fam][0]
        for s in sizes:
            for lay in ("nn", "nt", "tn", "tt"):
                ta, tb = lay[0] == "t", lay[1] == "t"
                a, b = device_operands(s, s, s, fam, ta, tb, dev, s)
                c = torch.empty((s, s), device=dev)
                sel = gemm.select(s, s, s, family=fam, trans_a=ta, trans_b=tb).as_tuple()
                cands = [sel] + [x for x in LARGE_CANDIDATES[fam] if x != sel]
                ns = gemm.sweep_problem(a, b, cands, family=fam, out=c, warmup=1, reps=3,
                                        min_sample_ns=0.0, max_cell_ns=0.0, early_exit=False)
                tf = [2.0 * s ** 3 / t / 1e3 for t in ns]
                j = max(range(len(cands)), key=lambda i: tf[i])
                rows.append({"family": fam, "layout": lay, "size": s, "selected": list(sel),
                             "selected_tflops": tf[0], "selected_frac": tf[0] / peak,
                             "best_listed": list(cands[j]), "best_tflops": tf[j],
                             "best_frac": tf[j] / peak})
                del a, b, c
    torch.cuda.synchronize()
    clocks.mark_end()
    clk = clocks.stop(gpu_index())
    torch.cuda.empty_cache()
    summ = {}
    for fam in ("f32", "tf32", "bf16"):
        fr = [r["selected_frac"] for r in rows if r["family"] == fam]
        summ[fam] = {"min_selected_frac": min(fr),
                     "geomean_selected_frac": math.exp(sum(map(math.log, fr)) / len(fr)),
                     "peak": peaks[fam][0], "peak_source": peaks[fam][1]}
    return {"rows": rows, "summary": summ, "clocks": clk,
            "timing": "K4 loop (kp_sweep_problem_ex): 1 warm-up + median of 3 launches per "
                      "config; operands 64-805 MB (>= L2)"}


def _geomean(xs):
    return math.exp(sum(math.log(x) for x in xs) / len(xs)) if xs else None


def network_roofline_block(dev, peaks) -> dict:
    """Roofline on the network-derived set (BASELINE configs[2], VGG16 /
    ResNet-50 / MobileNetV2 im2col + FC, batch 1-64): for each family the
    problems with >= 1 GFLOP and arithmetic intensity >= the family's ridge
    (peak / HBM bandwidth, algorithmic bytes es*(mk + kn) + 4mn), the
    runtime-selected kernel (kp_gemm_auto's choice) timed with the L2 flushed
    before every launch (CUDA events, median of 5)."""
    import torch
    from paper_2003_06795_b200 import gemm
    from paper_2003_06795_b200.shapes import network_problems
    bw = peaks["_hbm_gbs"]
    flush = torch.empty(FLUSH_BYTES // 4, device=dev)
    stream = torch.cuda.current_stream()
    out = {}
    for fam in ("f32", "tf32", "bf16"):
        peak = peaks[fam][0]
        es = 2 if fam == "bf16" else 4
        ridge = peak * 1e12 / (bw * 1e9)
        probs = [p for p in network_problems()
                 if 2.0 * p.m * p.n * p.k >= 1e9
                 and 2.0 * p.m * p.n * p.k / (es * (p.m * p.k + p.k * p.n) + 4 * p.m * p.n) >= ridge]
        rows = []
        for i, p in enumerate(probs):
            a, b = device_operands(p.m, p.k, p.n, fam, False, False, dev, 77 + i)
            c = torch.empty((p.m, p.n), device=dev)
            cfg = gemm.auto_config(p.m, p.k, p.n, family=fam)
            gemm.matmul(a, b, cfg, out=c, family=fam)  # warm-up (first launch)
            ms = []
            for _ in range(5):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                gemm.matmul(a, b, cfg, out=c, family=fam)
                e1.record(stream)
                e1.synchronize()
                ms.append(e0.elapsed_time(e1))
            t = statistics.median(ms)
            tf = 2.0 * p.m * p.n * p.k / (t * 1e-3) / 1e12
            rows.append({"mkn": [p.m, p.k, p.n],
                         "config": cfg if isinstance(cfg, str) else list(cfg.as_tuple()),
                         "tflops": tf, "frac": tf / peak})
            del a, b, c
        fr = [r["frac"] for r in rows]
        out[fam] = {"problems": len(rows), "ridge_flop_per_byte": ridge, "peak": peak,
                    "peak_source": peaks[fam][1], "geomean_frac": _geomean(fr),
                    "min_frac": min(fr) if fr else None, "max_frac": max(fr) if fr else None,
                    "rows": rows}
    del flush
    torch.cuda.empty_cache()
    return out


def _flushed_ms(fn, flush, reps=5, clean=None):
    """Median device time (ms) of fn() with the L2 flushed before each call
    (`clean`: a second buffer read after the flush write, so the timed kernel
    starts on clean L2 lines instead of paying the write-back of the flush
    buffer's dirty ones)."""
    import torch
    stream = torch.cuda.current_stream()
    fn()
    ms = []
    for _ in range(reps):
        flush.zero_()
        if clean is not None:
            clean.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    return statistics.median(ms)


def small_m_block(dev, peaks) -> dict:
    """FC layers at batch 1-16 (m <= 16; VGG16 fc6/fc7/fc8, ResNet-50 fc,
    MobileNetV2 fc): what kp_gemm_auto runs (the small-M B-streaming path)
    against the tile config the decision tree picks, as HBM GB/s of
    algorithmic bytes (es*(mk + kn) + 4mn) and fraction of the HBM peak
    (these shapes sit far below every family's ridge). L2 flushed before
    every launch (a 256 MiB write, then a 256 MiB read so the kernel starts on
    clean lines), CUDA events, median of 5."""
    import torch
    from paper_2003_06795_b200 import gemm
    from paper_2003_06795_b200.shapes import NETWORKS
    bw = peaks["_hbm_gbs"]
    flush = torch.empty(FLUSH_BYTES // 4, device=dev)
    clean = torch.zeros(FLUSH_BYTES // 4, device=dev)
    fcs = {}
    for net, layers in NETWORKS.items():
        for name, hw, k, n in layers:
            if hw == 1:
                fcs.setdefault((k, n), f"{net}.{name}")
    out = {}
    for fam in ("f32", "tf32", "bf16"):
        es = 2 if fam == "bf16" else 4
        rows = []
        for (k, n), name in fcs.items():
            for m in (1, 2, 4, 8, 16):
                a, b = device_operands(m, k, n, fam, False, False, dev, 900 + m)
                c = torch.empty((m, n), device=dev)
                auto = gemm.auto_config(m, k, n, family=fam)
                tile = gemm.select(m, k, n, family=fam)
                t_auto = _flushed_ms(lambda: gemm.matmul(a, b, auto, out=c, family=fam), flush,
                                     clean=clean)
                t_tile = _flushed_ms(lambda: gemm.matmul(a, b, tile, out=c, family=fam), flush,
                                     clean=clean)
                byt = es * (m * k + k * n) + 4 * m * n
                rows.append({"layer": name, "mkn": [m, k, n],
                             "auto": auto if isinstance(auto, str) else list(auto.as_tuple()),
                             "auto_gbs": byt / (t_auto * 1e-3) / 1e9,
                             "auto_frac_hbm": byt / (t_auto * 1e-3) / 1e9 / bw,
                             "tile_config": list(tile.as_tuple()),
                             "tile_gbs": byt / (t_tile * 1e-3) / 1e9,
                             "speedup_vs_tile": t_tile / t_auto})
                del a, b, c
        big = [r for r in rows if r["mkn"][1] * r["mkn"][2] * es >= 16 << 20]
        out[fam] = {"rows": rows, "hbm_gbs_peak": bw,
                    "geomean_frac_hbm_B_ge_16MB": _geomean([r["auto_frac_hbm"] for r in big]),
                    "min_frac_hbm_B_ge_16MB": min(r["auto_frac_hbm"] for r in big)}
    del flush, clean
    torch.cuda.empty_cache()
    return out


HELD_OUT_TOP = 16


def held_out_block(dev, families=("f32", "tf32", "bf16")) -> dict:
    """Out-of-sample selector quality, re-measured live: on the held-out side
    of each NN selector's training split (dataset.split(0.2, seed 42) of the
    committed data/b200_<fam>_nn_train.csv.gz, the rows the tree never saw)
    and on the batch-32/64 network shapes absent from training
    (data/b200_<fam>_nn_unseen.csv.gz), time the runtime-selected config and
    the candidate set -- every config for the 40-config tensor-core families,
    the committed dataset's 16 best for FP32 -- with the K4 loop; % of
    oracle-best = best / selected time, geomean over problems."""
    import torch
    from paper_2003_06795_b200 import dataset, gemm, pipeline
    out = {}
    for fam in families:
        train = pipeline.load_matrix(ROOT / "data" / f"b200_{fam}_nn_train.csv.gz")
        unseen = pipeline.load_matrix(ROOT / "data" / f"b200_{fam}_nn_unseen.csv.gz")
        test = dataset.split(train, 0.2, 42).test
        configs = list(train.configs)
        res = {}
        for name, mat in (("held_out_split", test), ("unseen_batch32_64", unseen)):
            ratios, hits = [], 0
            t0 = time.perf_counter()
            for i, p in enumerate(mat.problems):
                sel = gemm.auto_config(p.m, p.k, p.n, family=fam)
                if fam == "f32":
                    order = sorted(range(len(configs)), key=lambda j: -mat.values[i][j])
                    cands = [configs[j] for j in order[:HELD_OUT_TOP]]
                else:
                    cands = list(configs)
                if sel in cands:
                    hits += 1
                else:
                    cands = [sel] + cands
                a, b = device_operands(p.m, p.k, p.n, fam, False, False, dev, 500 + i)
                c = torch.empty((p.m, p.n), device=dev)
                ns = gemm.sweep_problem(a, b, cands, family=fam, out=c, warmup=2, reps=5,
                                        min_sample_ns=20_000.0, max_cell_ns=5e6,
                                        early_exit=False)
                ratios.append(min(ns) / ns[cands.index(sel)])
                del a, b, c
            res[name] = {"problems": len(ratios), "pct_oracle_best": 100.0 * _geomean(ratios),
                         "min_pct": 100.0 * min(ratios), "selected_in_candidates": hits,
                         "wall_s": time.perf_counter() - t0}
        res["candidates"] = ("all 40 configs" if fam != "f32" else
                             f"the committed dataset's {HELD_OUT_TOP} best configs per problem "
                             "(+ the selected one)")
        out[fam] = res
    torch.cuda.empty_cache()
    return out


class FamilyRun:
    """Sweep + timed selected-kernel steps of one kernel family on the square
    set (one rank's share; gathered / max-reduced by the caller)."""

    def __init__(self, family, args, dev, rank, world, gloo):
        import torch
        from paper_2003_06795_b200 import gemm, measure
        self.family, self.args, self.dev = family, args, dev
        self.rank, self.world, self.gloo = rank, world, gloo
        self.gemm, self.measure, self.torch = gemm, measure, torch
        dt = torch.bfloat16 if family == "bf16" else torch.float32
        gen = torch.Generator(device="cpu").manual_seed(1234 + rank)
        self.probs = []
        for s in SIZES:
            a = (torch.rand((s, s), generator=gen) * 2 - 1).to(dev).to(dt)
            b = (torch.rand((s, s), generator=gen) * 2 - 1).to(dev).to(dt)
            self.probs.append((s, a, b, torch.empty((s, s), device=dev)))
        # raises if no selector is compiled in for this family (no fallback)
        self.selected = [gemm.select(s, s, s, family=family) for s in SIZES]
        self.configs = gemm.family_configs(family)

    def barrier(self):
        import torch.distributed as dist
        self.torch.cuda.synchronize()
        if self.world > 1:
            dist.barrier(group=self.gloo)

    def sweep(self):
        import torch.distributed as dist
        mine = self.measure.config_shard(len(self.configs), self.rank, self.world)
        cells = {}
        self.barrier()
        t0 = time.perf_counter()
        if not self.args.no_sweep:
            for i, (s, a, b, c) in enumerate(self.probs):
                res = self.gemm.sweep_problem(a, b, [self.configs[j] for j in mine], out=c,
                                              family=self.family, warmup=1,
                                              reps=self.args.sweep_reps, min_sample_ns=20_000.0,
                                              max_cell_ns=5e6)
                cells.update({(i, j): ns for j, ns in zip(mine, res)})
        self.barrier()
        wall = time.perf_counter() - t0
        if self.world > 1:
            walls = [None] * self.world
            dist.all_gather_object(walls, wall, group=self.gloo)
            wall = max(walls)
        self.cells = self.measure.gather_cells(cells, self.world, self.gloo)
        self.sweep_wall = wall

    def timed(self, steps, clocks=None):
        """Per-size kernel ms over `steps` timed steps (L2 flushed before each
        kernel, CUDA events on the launching stream)."""
        import numpy as np
        torch = self.torch
        flush = torch.empty(FLUSH_BYTES // 4, device=self.dev)
        stream = torch.cuda.current_stream()
        n = self.args.warmup + steps
        ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in SIZES] for _ in range(n)]
        launches0 = 0
        if clocks:
            clocks.start()
        for step in range(n):
            if step == self.args.warmup:
                self.barrier()
                if clocks:
                    clocks.mark_begin()
                launches0 = self.gemm.launch_count()
            for i, (s, a, b, c) in enumerate(self.probs):
                flush.zero_()
                ev[step][i][0].record(stream)
                self.gemm.matmul(a, b, None, out=c, family=self.family)
                ev[step][i][1].record(stream)
        self.barrier()
        if clocks:
            clocks.mark_end()
        launches = self.gemm.launch_count() - launches0
        ms = np.array([[ev[st][i][0].elapsed_time(ev[st][i][1]) for i in range(len(SIZES))]
                       for st in range(self.args.warmup, n)])
        return ms, launches

    def report(self, per_size_ms):
        import numpy as np
        mean_ms = per_size_ms.mean(axis=0)
        per_size, ratios = [], []
        for i, s in enumerate(SIZES):
            entry = {"size": s, "config": list(self.selected[i].as_tuple()),
                     "tflops": flops_of(s) / (mean_ms[i] * 1e-3) / 1e12}
            if self.cells:
                row = np.array([self.cells[(i, j)] for j in range(len(self.configs))])
                jbest, jsel = int(row.argmin()), self.configs.index(self.selected[i])
                ratios.append(row[jbest] / row[jsel])
                entry.update(best_config=list(self.configs[jbest].as_tuple()),
                             best_tflops_warm=flops_of(s) / row[jbest] / 1e3,
                             selected_tflops_warm=flops_of(s) / row[jsel] / 1e3)
            per_size.append(entry)
        pct = (100.0 * math.exp(sum(math.log(r) for r in ratios) / len(ratios))
               if ratios else None)
        dom = int(mean_ms.argmax())
        return per_size, pct, dom, mean_ms


def reduce_over_ranks(x, world, group, op="max"):
    """Host-side reduction of a device-timed scalar (gloo group): the max over
    ranks for times, the sum for launch counts."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM, group=group)
    return float(t.item())


def run_gpu(args) -> int:
    import torch
    import torch.distributed as dist

    from paper_2003_06795_b200 import gemm

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # KP_BENCH_SHARE_DEVICE=1 runs every rank on device 0: exercises the
    # multi-rank code path on a one-GPU box
    share = os.environ.get("KP_BENCH_SHARE_DEVICE") == "1"
    dev_index = 0 if share else local
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    gloo = None
    if world > 1:
        # the path has no data-path collective: ranks only exchange host-side
        # timings and sweep cells, over gloo
        dist.init_process_group("gloo")
        gloo = dist.group.WORLD
    step_flops = sum(flops_of(s) for s in SIZES)

    # ---- headline family: FP32 SIMT (the paper's 640-config space) ---------
    f32 = FamilyRun("f32", args, dev, rank, world, gloo)
    f32.sweep()
    clocks = ClockSampler()
    per_size_ms, launches = f32.timed(args.steps, clocks)
    clk = clocks.stop(gpu_index())
    total_ms = reduce_over_ranks(float(per_size_ms.sum()), world, gloo)
    launches = int(reduce_over_ranks(launches, world, gloo, op="sum"))
    value = world * args.steps * step_flops / (total_ms * 1e-3) / 1e12

    # ---- e2e through the host-buffer API --------------------------------
    host = [(a.cpu().pin_memory(), b.cpu().pin_memory(), torch.empty((s, s), pin_memory=True))
            for s, a, b, c in f32.probs]
    pipe = gemm.PinnedPipeline("f32")
    for _ in range(args.warmup):
        pipe.run(host)
    # three windows of `steps` steps each (host jitter: pinned-copy and Python
    # enqueue timing varies between windows); the median window is reported
    e2e_windows = []
    for _ in range(3):
        f32.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            pipe.run(host)
        e2e_windows.append(reduce_over_ranks(time.perf_counter() - t0, world, gloo))
    e2e_s = statistics.median(e2e_windows)
    e2e_value = world * args.steps * step_flops / e2e_s / 1e12

    # ---- tensor-core families (same workload, their own selectors) -------
    families, fam_runs = {}, {}
    fam_steps = max(20, args.steps // 4)
    for fam in ("tf32", "bf16"):
        run = FamilyRun(fam, args, dev, rank, world, gloo)
        run.sweep()
        ms, _ = run.timed(fam_steps)
        tot = reduce_over_ranks(float(ms.sum()), world, gloo)
        fam_runs[fam] = (run.report(ms), tot, len(run.cells),
                         len(run.cells) / run.sweep_wall if run.cells else None)
        del run
    torch.cuda.empty_cache()
    # the peak measurements run seconds of full-power GEMMs (cuBLAS TF32, the
    # FFMA probe): after every timed step, so their power draw cannot lower
    # the clocks of the timed regions
    peaks = family_peaks(dev)
    for fam, ((per, pct, dom, mean), tot, ncells, cps) in fam_runs.items():
        tpk, src = tensor_peak(fam, peaks)
        ach = flops_of(SIZES[dom]) / (mean[dom] * 1e-3) / 1e12
        families[fam] = {
            "value": world * fam_steps * step_flops / (tot * 1e-3) / 1e12, "unit": "TFLOP/s",
            "steps": fam_steps, "pct_oracle_best_in_sample": pct,
            "sweep": {"cells": ncells, "cells_per_s": cps},
            "roofline": {"bound": "tensor", "achieved": ach, "peak": tpk, "unit": "TFLOP/s",
                         "frac": ach / tpk, "peak_source": src,
                         "kernel": f"tc_gemm {per[dom]['config']} @ {SIZES[dom]}^3"},
            "per_size": per, "selector": f"csrc/generated/select_{fam}_nn.h"}

    if rank != 0:
        if world > 1:
            dist.barrier(group=gloo)
            dist.destroy_process_group()
        return 0

    # ---- rank 0: roofline evidence blocks (one GPU's worth) ---------------
    extra = {}
    if not args.no_extra:
        # evidence blocks: a failure is recorded in the line instead of
        # losing the headline measurement
        for name, fn in (("held_out", lambda: held_out_block(dev)),
                         ("large_sizes", lambda: large_sizes_block(dev, peaks)),
                         ("network_roofline", lambda: network_roofline_block(dev, peaks)),
                         ("small_m", lambda: small_m_block(dev, peaks))):
            try:
                extra[name] = fn()
            except Exception as exc:  # noqa: BLE001
                extra[name] = {"error": f"{type(exc).__name__}: {exc}"[:500]}
                torch.cuda.synchronize()
                torch.cuda.empty_cache()

    per_size, pct_best, dom, mean_ms = f32.report(per_size_ms)
    achieved = flops_of(SIZES[dom]) / (mean_ms[dom] * 1e-3) / 1e12
    fp = peaks["_f32"]
    roofline = {"bound": "fp32-ffma", "achieved": achieved, "peak": fp["nominal"],
                "unit": "TFLOP/s", "frac": achieved / fp["nominal"],
                "traffic": traffic_for(f32.selected[dom], SIZES[dom]),
                "kernel": f"simt_gemm {list(f32.selected[dom].as_tuple())} @ {SIZES[dom]}^3",
                "share_of_step": float(mean_ms[dom] / mean_ms.sum()),
                "peak_source": "nominal FP32 SIMT peak, " + fp["nominal_how"] +
                               " (MEASURED_PEAKS.json has no FP32 SIMT figure)",
                "peak_measured": fp["measured"], "frac_of_measured": achieved / fp["measured"],
                "peak_measured_source": fp["measured_how"]}
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": bench_config(world),
        "pct_oracle_best": pct_best,
        "pct_oracle_best_note": "in-sample: squares 64..2048 are in the selector's training "
                                "set; the out-of-sample figures are held_out.*",
        "sweep": {"cells": len(f32.cells), "wall_s": f32.sweep_wall,
                  "cells_per_s": len(f32.cells) / f32.sweep_wall if f32.cells else None,
                  "timing": "warm L2, median of reps, C++ loop (kp_sweep_problem); a "
                            "config > 1 ms and > 8x the size's best so far keeps its first "
                            "timing"},
        "per_size": per_size,
        "roofline": roofline,
        "e2e": {"value": e2e_value, "unit": "TFLOP/s",
                "h2d_bytes_per_step": sum(2 * 4 * s * s for s in SIZES),
                "d2h_bytes_per_step": sum(4 * s * s for s in SIZES),
                "windows_tflops": [world * args.steps * step_flops / w / 1e12 for w in e2e_windows],
                "path": "gemm.PinnedPipeline: pinned H2D (copy stream) + kp_gemm_auto "
                        "(compute stream) + D2H (copy stream), largest problem first, "
                        "2048^3 split into 4 row blocks of A/C so its kernels and D2H run "
                        "under the remaining H2D; synchronised every step; median of three "
                        "windows of `steps` steps"},
        "gpu_launches": launches,
        "clocks": clk,
        "peaks": {"fp32_nominal": fp["nominal"], "fp32_measured": fp["measured"],
                  "tf32_cublas": peaks["tf32"][0], "bf16": peaks["bf16"][0],
                  "hbm_gbs": peaks["_hbm_gbs"], "hbm_source": peaks["_hbm_source"]},
        "families": families,
    }
    line.update(extra)
    if world == 1:
        line["cpu_baseline"] = cpu_baseline(args.cpu_seconds)
        if f32.cells:
            line["host_pipeline"] = host_pipeline(f32.cells, f32.configs)
    print(json.dumps(line))
    if world > 1:
        dist.barrier(group=gloo)
        dist.destroy_process_group()
    return 0


def main(argv=None) -> int:
    args = parse_args(argv)
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
