"""The measured sweep: B200 twin of the reference's synthetic.generate.

Reference producer: synthetic.generate(spec) -> list[BenchmarkRecord]
(pkg/src/kernelprune/synthetic.py:92-114): one record per (problem, config),
row-major by problem then canonical config, runtime_ns = 2mnk / gflops.
Here every cell is a real kernel launch timed on the GPU (C++ timing loop,
kp_sweep_problem): operands are allocated once per problem (U[-1,1) fp32,
seeded per problem), every config runs `warmup` untimed launches and `reps`
timed samples of back-to-back launches (each sample >= min_sample_ns), and
the median per-launch time is the cell's runtime. L2 is warm (the same
operands are reused across launches), which the sidecar records.

Multi-GPU: the cell list shards by problem across worker processes, one per
GPU, with no device-to-device traffic (sweep_sharded); records return to the
parent and are merged back into canonical order.
"""

from __future__ import annotations

import json
import os
import time
from dataclasses import dataclass, field

import numpy as np

from .dataset import BenchmarkRecord, KernelConfig, ProblemSize, all_configs


@dataclass
class SweepSpec:
    problems: tuple[ProblemSize, ...]
    family: str = "f32"
    trans_a: bool = False
    trans_b: bool = False
    batch: int = 1
    configs: tuple[KernelConfig, ...] | None = None   # None -> family's full list
    warmup: int = 2
    reps: int = 5
    min_sample_ns: float = 20_000.0
    max_cell_ns: float = 5_000_000.0    # per-cell time budget (kp_gemm_time)
    seed: int = 0


@dataclass
class SweepResult:
    spec: SweepSpec
    configs: tuple[KernelConfig, ...]
    runtime_ns: np.ndarray           # (P, C)
    wall_s: float
    device: dict = field(default_factory=dict)

    @property
    def cells(self) -> int:
        return int(self.runtime_ns.size)

    def gflops(self) -> np.ndarray:
        flops = np.array([2.0 * self.spec.batch * p.m * p.n * p.k for p in self.spec.problems])
        return flops[:, None] / self.runtime_ns

    def records(self) -> list[BenchmarkRecord]:
        """Canonical-order records (problem-major), as synthetic.generate."""
        out = []
        g = self.gflops()
        for i, p in enumerate(self.spec.problems):
            flops = 2 * self.spec.batch * p.m * p.n * p.k
            for j, c in enumerate(self.configs):
                gf = float(g[i, j])
                out.append(BenchmarkRecord(p, c, flops / gf, gf))
        return out


def _operands(problem: ProblemSize, spec: SweepSpec, index: int, device):
    import torch
    gen = torch.Generator(device="cpu").manual_seed(spec.seed * 1_000_003 + index)
    m, k, n, bt = problem.m, problem.k, problem.n, spec.batch
    a_shape = (k, m) if spec.trans_a else (m, k)
    b_shape = (n, k) if spec.trans_b else (k, n)
    if bt > 1:
        a_shape, b_shape = (bt,) + a_shape, (bt,) + b_shape
    dtype = torch.bfloat16 if spec.family == "bf16" else torch.float32
    # tensor-core families load through TMA, which needs 16-byte row pitches:
    # the sweep pads the leading dimension of its own allocations (the
    # logical shape is unchanged; TMA zero-fills past the logical extent)
    align = {"tf32": 4, "bf16": 8}.get(spec.family, 1)

    def alloc(shape):
        inner = -(-shape[-1] // align) * align
        full = (torch.rand(shape[:-1] + (inner,), generator=gen) * 2 - 1)
        return full.to(device=device, dtype=dtype)[..., :shape[-1]]

    a = alloc(a_shape)
    b = alloc(b_shape)
    if spec.trans_a:
        a = a.transpose(-1, -2)
    if spec.trans_b:
        b = b.transpose(-1, -2)
    return a, b


def device_facts(device: int = 0) -> dict:
    import ctypes

    from . import _native as nat
    sm, clk, cc = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    nat.check(nat.lib().kp_device_info(device, ctypes.byref(sm), ctypes.byref(clk),
                                       ctypes.byref(cc)), "kp_device_info")
    import torch
    return {"name": torch.cuda.get_device_name(device), "sm_count": sm.value,
            "sm_clock_max_mhz": clk.value / 1000.0, "cc": cc.value}


def run_sweep(spec: SweepSpec, device: int = 0, progress=None) -> SweepResult:
    """Time every (problem, config) cell of `spec` on one GPU."""
    import torch

    from . import gemm
    torch.cuda.set_device(device)
    configs = tuple(spec.configs) if spec.configs is not None else gemm.family_configs(spec.family)
    rt = np.zeros((len(spec.problems), len(configs)), dtype=np.float64)
    t0 = time.perf_counter()
    for i, p in enumerate(spec.problems):
        a, b = _operands(p, spec, i, torch.device("cuda", device))
        rt[i] = gemm.sweep_problem(a, b, configs, family=spec.family, warmup=spec.warmup,
                                   reps=spec.reps, min_sample_ns=spec.min_sample_ns,
                                   max_cell_ns=spec.max_cell_ns)
        del a, b
        if progress:
            progress(i, p, rt[i])
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    return SweepResult(spec, configs, rt, wall, device_facts(device))


def problem_cost(p: ProblemSize, batch: int = 1) -> float:
    """Relative sweep cost of one problem: its flops over the reference's
    analytic throughput averaged over the config space (synthetic.py:73-89),
    plus a per-config launch floor. Used only to order / balance shards."""
    from .synthetic import analytic_matrix
    mean_gflops = float(analytic_matrix([p], all_configs(), 8192.0).mean())
    return 2.0 * batch * p.m * p.n * p.k / mean_gflops + 640 * 5e3


def plan_shards(problems, n_shards: int, batch: int = 1) -> list[list[int]]:
    """Static longest-processing-time-first partition of problem indices
    (each shard sorted ascending so merged output keeps canonical order)."""
    if n_shards < 1:
        raise ValueError("n_shards must be >= 1")
    order = sorted(range(len(problems)), key=lambda i: (-problem_cost(problems[i], batch), i))
    load = [0.0] * n_shards
    shards: list[list[int]] = [[] for _ in range(n_shards)]
    for i in order:
        s = min(range(n_shards), key=lambda j: (load[j], j))
        shards[s].append(i)
        load[s] += problem_cost(problems[i], batch)
    return [sorted(s) for s in shards]


def plan_tasks(problems, n_devices: int, n_configs: int, batch: int = 1,
               granularity: int = 4) -> list[tuple[int, int, int]]:
    """Sweep tasks (problem, first config, end config), longest first, for a
    dynamic queue over `n_devices` workers. A problem costing more than
    total / (granularity * n_devices) is cut into contiguous config ranges
    (at most 16), so one huge problem (8192^3) cannot hold the last worker
    while the others idle; everything else stays one task per problem
    (operands generated once)."""
    if n_devices < 1:
        raise ValueError("n_devices must be >= 1")
    costs = [problem_cost(p, batch) for p in problems]
    limit = sum(costs) / (granularity * n_devices)
    tasks = []
    for i, c in enumerate(costs):
        k = 1 if n_devices == 1 else min(16, n_configs, max(1, -(-int(c) // max(1, int(limit)))))
        bounds = [round(j * n_configs / k) for j in range(k + 1)]
        tasks += [(i, bounds[j], bounds[j + 1], c * (bounds[j + 1] - bounds[j]) / n_configs)
                  for j in range(k)]
    tasks.sort(key=lambda t: (-t[3], t[0], t[1]))
    return [(i, lo, hi) for i, lo, hi, _ in tasks]


def merge_chunks(n_problems: int, n_configs: int, chunks) -> np.ndarray:
    """Reassemble (problem, lo, hi, runtimes[hi-lo]) chunks into the (P, C)
    grid; every cell must arrive exactly once (complete-grid contract)."""
    grid = np.full((n_problems, n_configs), np.nan)
    count = np.zeros((n_problems, n_configs), dtype=np.int64)
    for i, lo, hi, row in chunks:
        row = np.asarray(row, dtype=float)
        if row.shape != (hi - lo,):
            raise RuntimeError(f"chunk ({i}, {lo}, {hi}) has {row.shape[0]} runtimes")
        grid[i, lo:hi] = row
        count[i, lo:hi] += 1
    if (count > 1).any():
        i, j = np.argwhere(count > 1)[0]
        raise RuntimeError(f"cell ({i}, {j}) measured twice")
    if (count == 0).any():
        missing = sorted({int(i) for i, _ in np.argwhere(count == 0)})
        raise RuntimeError(f"problems never fully measured: {missing}")
    if not np.isfinite(grid).all() or (grid <= 0).any():
        raise RuntimeError("non-positive or non-finite runtime in sweep")
    return grid


def merge_shards(n_problems: int, n_configs: int, parts) -> np.ndarray:
    """Reassemble {problem index: runtimes row} parts into the (P, C) grid;
    every problem must arrive exactly once (complete-grid contract,
    dataset.build_matrix)."""
    grid = np.full((n_problems, n_configs), np.nan)
    seen = np.zeros(n_problems, dtype=bool)
    for part in parts:
        for i, row in part.items():
            if seen[i]:
                raise RuntimeError(f"problem {i} measured twice")
            seen[i] = True
            grid[i] = row
    if not seen.all():
        raise RuntimeError(f"problems never measured: {np.flatnonzero(~seen).tolist()}")
    if not np.isfinite(grid).all() or (grid <= 0).any():
        raise RuntimeError("non-positive or non-finite runtime in sweep")
    return grid


def config_shard(n_configs: int, rank: int, world: int) -> list[int]:
    """Interleaved config shard of one rank (bench.py under torchrun): config
    costs vary smoothly along the canonical order, so striding balances."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return list(range(rank, n_configs, world))


def gather_cells(local: dict, world: int, group=None) -> dict:
    """Merge every rank's {(problem, config): runtime_ns} on all ranks with a
    host-side object all-gather (gloo group); a cell measured twice is an
    error. No device-to-device traffic: the sweep has no data exchange."""
    if world == 1:
        return dict(local)
    import torch.distributed as dist
    parts = [None] * world
    dist.all_gather_object(parts, local, group=group)
    merged: dict = {}
    for part in parts:
        for key, val in part.items():
            if key in merged:
                raise RuntimeError(f"cell {key} measured by two ranks")
            merged[key] = val
    return merged


def _worker(device: int, spec: SweepSpec, task_q, result_q) -> None:
    """One process per GPU: pull problem indices until the queue is empty."""
    os.environ["CUDA_VISIBLE_DEVICES"] = str(device)
    try:
        import torch

        from . import gemm
        torch.cuda.set_device(0)
        configs = (tuple(spec.configs) if spec.configs is not None
                   else gemm.family_configs(spec.family))
        while True:
            task = task_q.get()
            if task is None:
                break
            i, lo, hi = task
            a, b = _operands(spec.problems[i], spec, i, torch.device("cuda", 0))
            row = gemm.sweep_problem(a, b, configs[lo:hi], family=spec.family,
                                     warmup=spec.warmup, reps=spec.reps,
                                     min_sample_ns=spec.min_sample_ns,
                                     max_cell_ns=spec.max_cell_ns)
            del a, b
            result_q.put(("row", device, (i, lo, hi), row))
        result_q.put(("done", device, device_facts(0), None))
    except Exception as exc:  # surfaced by the parent; never silently imputed
        result_q.put(("error", device, repr(exc), None))


def run_sharded(spec: SweepSpec, devices) -> SweepResult:
    """Sweep across several GPUs: a dynamic longest-first work queue of
    (problem, config range) tasks (plan_tasks), one worker process per GPU,
    no device-to-device traffic. A worker error aborts the sweep (a failed
    cell is never imputed)."""
    import multiprocessing as mp
    from . import gemm
    n_cfg = len(spec.configs) if spec.configs is not None else len(gemm.family_configs(spec.family))
    ctx = mp.get_context("spawn")
    task_q, result_q = ctx.Queue(), ctx.Queue()
    for task in plan_tasks(spec.problems, len(devices), n_cfg, spec.batch):
        task_q.put(task)
    for _ in devices:
        task_q.put(None)
    t0 = time.perf_counter()
    procs = [ctx.Process(target=_worker, args=(d, spec, task_q, result_q)) for d in devices]
    for p in procs:
        p.start()
    chunks, done, facts = [], 0, {}
    try:
        while done < len(devices):
            kind, dev, a, b = result_q.get()
            if kind == "row":
                chunks.append((a[0], a[1], a[2], b))
            elif kind == "done":
                done += 1
                facts[dev] = a
            else:
                raise RuntimeError(f"sweep worker on device {dev} failed: {a}")
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.terminate()
    wall = time.perf_counter() - t0
    grid = merge_chunks(len(spec.problems), n_cfg, chunks)
    configs = tuple(spec.configs) if spec.configs is not None else gemm.family_configs(spec.family)
    first = facts[min(facts)] if facts else {}
    return SweepResult(spec, configs, grid, wall, dict(first, devices=len(devices)))


def sidecar(result: SweepResult, extra: dict | None = None) -> dict:
    s = result.spec
    doc = {
        "family": s.family, "trans_a": s.trans_a, "trans_b": s.trans_b, "batch": s.batch,
        "problems": len(s.problems), "configs": len(result.configs), "cells": result.cells,
        "warmup": s.warmup, "reps": s.reps, "min_sample_ns": s.min_sample_ns,
        "max_cell_ns": s.max_cell_ns,
        "statistic": "median of reps samples; each sample = back-to-back launches / count",
        "l2": "warm (operands reused across launches)",
        "timing": "CUDA events on the launching stream (kp_sweep_problem)",
        "wall_s": result.wall_s, "cells_per_s": result.cells / result.wall_s,
        "device": result.device, "host_cores": os.cpu_count(),
    }
    if extra:
        doc.update(extra)
    return doc


def main(argv=None) -> int:
    import argparse
    ap = argparse.ArgumentParser(description="measured config x size sweep (one GPU)")
    ap.add_argument("--sizes", default="64,128,256,512,1024,2048")
    ap.add_argument("--family", default="f32")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--top", type=int, default=5)
    ap.add_argument("--out")
    args = ap.parse_args(argv)
    from .shapes import square_problems
    probs = square_problems(tuple(int(s) for s in args.sizes.split(",")))
    spec = SweepSpec(probs, family=args.family, reps=args.reps, warmup=args.warmup)

    def prog(i, p, row):
        flops = 2.0 * p.m * p.n * p.k
        order = np.argsort(row)
        best = ", ".join(f"{all_configs()[j].as_tuple() if len(row) == 640 else j}:"
                         f"{flops / row[j] / 1e3:.2f}TF" for j in order[:args.top])
        print(f"{p.as_tuple()}: best {best}; worst {flops / row.max() / 1e3:.3f}TF", flush=True)

    res = run_sweep(spec, progress=prog)
    print(json.dumps(sidecar(res)))
    if args.out:
        from .dataset import write_records
        write_records(res.records(), args.out)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
