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
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="bounded CPU-baseline sample length")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    return args


def flops_of(s: int) -> float:
    return 2.0 * s * s * s


# ----------------------------------------------------------- CPU baselines

def cpu_gemm_pass(mats) -> float:
    """One pass of numpy fp32 a@b over the square set; returns seconds."""
    t0 = time.perf_counter()
    for a, b in mats:
        a @ b
    return time.perf_counter() - t0


def cpu_mats(seed=0):
    import numpy as np
    rng = np.random.default_rng(seed)
    return [(rng.uniform(-1, 1, (s, s)).astype(np.float32),
             rng.uniform(-1, 1, (s, s)).astype(np.float32)) for s in SIZES]


def cpu_baseline(seconds: float) -> dict:
    """numpy fp32 GEMM (OpenBLAS, all host threads) on the same square set:
    the CPU restatement of the path (the reference ships no GEMM; its oracle
    restatement is oracle/gemm_ref.c / numpy), timed for a bounded sample."""
    mats = cpu_mats()
    cpu_gemm_pass(mats)  # warm-up
    passes, spent = 0, 0.0
    while spent < seconds or passes < 3:
        spent += cpu_gemm_pass(mats)
        passes += 1
    total = passes * sum(flops_of(s) for s in SIZES)
    return {"value": total / spent / 1e12, "unit": "TFLOP/s", "cores": os.cpu_count(),
            "kind": "port",
            "sample": f"{passes} passes of numpy float32 a@b over squares {list(SIZES)} "
                      f"({spent:.1f} s, OpenBLAS all threads)"}


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
    """--impl reference: the CPU implementation of the path (numpy fp32 GEMM
    over the same workload) on the box's host cores; rank 0 only."""
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    mats = cpu_mats()
    for _ in range(args.warmup):
        cpu_gemm_pass(mats)
    times = [cpu_gemm_pass(mats) for _ in range(args.steps)]
    total = sum(times)
    value = args.steps * sum(flops_of(s) for s in SIZES) / total / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "square GEMM pass 64..2048 (fp32, NN)", "sizes": list(SIZES)},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": os.cpu_count(),
                         "kind": "port",
                         "sample": f"{args.steps} timed passes of numpy float32 a@b "
                                   f"(OpenBLAS, all host threads)"},
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


def tensor_peak(family: str):
    """(peak TFLOP/s, source) for a tcgen05 family: MEASURED_PEAKS.json's bf16
    burst figure (TF32 dense = half of it, NVIDIA's dense ratio), else the
    B200_PROFILING.md fallback."""
    path = ROOT / "MEASURED_PEAKS.json"
    if path.exists():
        bf16 = float(json.loads(path.read_text())["bf16_tflops"])
        src = "MEASURED_PEAKS.json bf16_tflops (burst)"
    else:
        bf16, src = 1590.0, "fallback 1.59 PFLOP/s (B200_PROFILING.md)"
    if family == "tf32":
        return bf16 / 2, src + " / 2 (tf32 dense rate)"
    return bf16, src


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
    import ctypes

    import torch
    import torch.distributed as dist

    from paper_2003_06795_b200 import _native as nat
    from paper_2003_06795_b200 import gemm

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # KP_BENCH_SHARE_DEVICE=1 runs every rank on device 0 with a gloo-only
    # process group: exercises the multi-rank code path on a one-GPU box
    share = os.environ.get("KP_BENCH_SHARE_DEVICE") == "1"
    dev_index = 0 if share else local
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    gloo = None
    if world > 1:
        if share:
            dist.init_process_group("gloo")
            gloo = dist.group.WORLD
        else:
            dist.init_process_group("nccl", device_id=dev)
            gloo = dist.new_group(backend="gloo")
    step_flops = sum(flops_of(s) for s in SIZES)

    # ---- headline family: FP32 SIMT (the paper's 640-config space) ---------
    f32 = FamilyRun("f32", args, dev, rank, world, gloo)
    f32.sweep()
    peak = ctypes.c_double()
    nat.check(nat.lib().kp_fp32_peak(ctypes.byref(peak), None), "kp_fp32_peak")
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
    f32.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        pipe.run(host)
    e2e_s = reduce_over_ranks(time.perf_counter() - t0, world, gloo)
    e2e_value = world * args.steps * step_flops / e2e_s / 1e12

    # ---- tensor-core families (same workload, their own selectors) -------
    families = {}
    fam_steps = max(20, args.steps // 4)
    for fam in ("tf32", "bf16"):
        run = FamilyRun(fam, args, dev, rank, world, gloo)
        run.sweep()
        ms, _ = run.timed(fam_steps)
        tot = reduce_over_ranks(float(ms.sum()), world, gloo)
        per, pct, dom, mean = run.report(ms)
        tpk, src = tensor_peak(fam)
        ach = flops_of(SIZES[dom]) / (mean[dom] * 1e-3) / 1e12
        families[fam] = {
            "value": world * fam_steps * step_flops / (tot * 1e-3) / 1e12, "unit": "TFLOP/s",
            "steps": fam_steps, "pct_oracle_best": pct,
            "sweep": {"cells": len(run.cells), "cells_per_s":
                      len(run.cells) / run.sweep_wall if run.cells else None},
            "roofline": {"bound": "tensor", "achieved": ach, "peak": tpk, "unit": "TFLOP/s",
                         "frac": ach / tpk, "peak_source": src,
                         "kernel": f"tc_gemm {per[dom]['config']} @ {SIZES[dom]}^3"},
            "per_size": per, "selector": f"csrc/generated/select_{fam}_nn.h"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    per_size, pct_best, dom, mean_ms = f32.report(per_size_ms)
    achieved = flops_of(SIZES[dom]) / (mean_ms[dom] * 1e-3) / 1e12
    roofline = {"bound": "fp32-ffma", "achieved": achieved, "peak": peak.value,
                "unit": "TFLOP/s", "frac": achieved / peak.value,
                "traffic": traffic_for(f32.selected[dom], SIZES[dom]),
                "kernel": f"simt_gemm {list(f32.selected[dom].as_tuple())} @ {SIZES[dom]}^3",
                "share_of_step": float(mean_ms[dom] / mean_ms.sum()),
                "peak_source": "measured FFMA microbenchmark (kp_fp32_peak) on this GPU; "
                               "MEASURED_PEAKS.json has no fp32 SIMT figure"}
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": "640-config sweep + runtime-selected FP32 SIMT GEMM pass over "
                               "squares 64..2048 (NN)",
                   "sizes": list(SIZES), "selector": "csrc/generated/select_f32_nn.h",
                   "l2": f"flushed before every timed kernel ({FLUSH_BYTES >> 20} MiB write)",
                   "parallelism": f"replicas x{world}"},
        "pct_oracle_best": pct_best,
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
                "path": "gemm.PinnedPipeline: pinned H2D (copy stream) + kp_gemm_auto "
                        "(compute stream) + D2H (copy stream), largest problem first, "
                        "2048^3 split into 4 row blocks of A/C so its kernels and D2H run "
                        "under the remaining H2D; synchronised every step"},
        "gpu_launches": launches,
        "clocks": clk,
        "families": families,
    }
    if world == 1:
        line["cpu_baseline"] = cpu_baseline(args.cpu_seconds)
        if f32.cells:
            line["host_pipeline"] = host_pipeline(f32.cells, f32.configs)
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def main(argv=None) -> int:
    args = parse_args(argv)
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
