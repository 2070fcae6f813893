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
    task_log: list = field(default_factory=list)   # per task: device, NVML clocks

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
    log = []
    nvml_index = _visible_index(device)
    t0 = time.perf_counter()
    for i, p in enumerate(spec.problems):
        before = gpu_clocks(nvml_index)
        a, b = _operands(p, spec, i, torch.device("cuda", device))
        rt[i] = gemm.sweep_problem(a, b, configs, family=spec.family, warmup=spec.warmup,
                                   reps=spec.reps, min_sample_ns=spec.min_sample_ns,
                                   max_cell_ns=spec.max_cell_ns)
        del a, b
        log.append({"task": [i, 0, len(configs)], "device": device,
                    "clocks": {"before": before, "after": gpu_clocks(nvml_index)}})
        if progress:
            progress(i, p, rt[i])
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    return SweepResult(spec, configs, rt, wall, device_facts(device), task_log=log)


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


def gpu_clocks(index: int) -> dict | None:
    """SM clock (MHz) and active throttle reasons of one GPU via NVML (None
    when NVML is unavailable). Logged beside every sweep task."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
        mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        mask = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
    except Exception:  # noqa: BLE001 - NVML missing or not permitted
        return None
    names = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
             0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}
    return {"sm_mhz": int(mhz), "reasons": sorted(n for bit, n in names.items() if mask & bit)}


def _visible_index(device: int) -> int:
    """NVML index of logical device `device` under the parent's CUDA_VISIBLE_DEVICES."""
    vis = [v.strip() for v in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if v.strip()]
    if device < len(vis) and vis[device].isdigit():
        return int(vis[device])
    return device


def _worker(device: int, spec: SweepSpec, conn) -> None:
    """One process per GPU: announce readiness, then run the (problem, config
    range) tasks the parent hands over until it sends None. Each result
    carries the NVML clocks sampled before and after the task. `conn` is this
    worker's own duplex pipe (synchronous sends, nothing shared with other
    workers, so a worker killed mid-message cannot wedge the others)."""
    nvml_index = _visible_index(device)
    os.environ["CUDA_VISIBLE_DEVICES"] = str(nvml_index)
    task = None
    try:
        import torch

        from . import gemm
        torch.cuda.set_device(0)
        configs = (tuple(spec.configs) if spec.configs is not None
                   else gemm.family_configs(spec.family))
        conn.send(("ready", device, None, device_facts(0)))
        while True:
            task = conn.recv()
            if task is None:
                break
            i, lo, hi = task
            before = gpu_clocks(nvml_index)
            a, b = _operands(spec.problems[i], spec, i, torch.device("cuda", 0))
            # a config-range task must time exactly like the whole problem
            # would: the early exit for hopeless configs compares against the
            # best median so far, which only a whole-problem task knows
            row = gemm.sweep_problem(a, b, configs[lo:hi], family=spec.family,
                                     warmup=spec.warmup, reps=spec.reps,
                                     min_sample_ns=spec.min_sample_ns,
                                     max_cell_ns=spec.max_cell_ns,
                                     early_exit=(lo, hi) == (0, len(configs)))
            del a, b
            conn.send(("row", device, task, (row, {"before": before,
                                                   "after": gpu_clocks(nvml_index)})))
    except Exception as exc:  # surfaced by the parent; never silently imputed
        conn.send(("error", device, task, repr(exc)))
        raise SystemExit(1)


def _spec_key(spec: SweepSpec, n_cfg: int) -> dict:
    return {"family": spec.family, "trans_a": spec.trans_a, "trans_b": spec.trans_b,
            "batch": spec.batch, "problems": [p.as_tuple() for p in spec.problems],
            "configs": n_cfg, "warmup": spec.warmup, "reps": spec.reps,
            "min_sample_ns": spec.min_sample_ns, "max_cell_ns": spec.max_cell_ns,
            "seed": spec.seed}


class TaskCheckpoint:
    """Per-task result shards of a sharded sweep (resume after a crash): one
    JSON file per finished (problem, config range) task under `directory`,
    plus spec.json naming the sweep they belong to (a mismatch is an error,
    never a silent mix of two sweeps)."""

    def __init__(self, directory, key: dict):
        from pathlib import Path
        self.dir = Path(directory)
        self.dir.mkdir(parents=True, exist_ok=True)
        meta = self.dir / "spec.json"
        key = json.loads(json.dumps(key))  # tuples -> lists, as stored
        if meta.exists():
            if json.loads(meta.read_text()) != key:
                raise RuntimeError(f"{meta} belongs to a different sweep; use a fresh directory")
        else:
            meta.write_text(json.dumps(key))

    def _path(self, task):
        i, lo, hi = task
        return self.dir / f"task_p{i}_c{lo}-{hi}.json"

    def load(self, task):
        path = self._path(task)
        if not path.exists():
            return None
        doc = json.loads(path.read_text())
        return np.asarray(doc["runtime_ns"], dtype=float), doc.get("log", {})

    def save(self, task, row, log):
        path = self._path(task)
        tmp = path.with_suffix(".tmp")
        tmp.write_text(json.dumps({"runtime_ns": [float(x) for x in row], "log": log}))
        os.replace(tmp, path)


def run_sharded(spec: SweepSpec, devices, *, checkpoint_dir=None, max_task_attempts: int = 2,
                max_restarts: int = 2, poll_s: float = 2.0, start_timeout_s: float = 600.0,
                _worker_fn=None) -> SweepResult:
    """Sweep across several GPUs: longest-first (problem, config range) tasks
    (plan_tasks) handed one at a time to one worker process per GPU, no
    device-to-device traffic.

    Robustness (an 8-GPU sweep runs for hours):
      * the parent polls its result queue and checks every worker's liveness,
        so a worker that dies without a message (segfault, OOM kill, driver
        abort) is detected instead of blocking the parent forever;
      * the dead (or failed) worker's in-flight task is re-queued at the front
        and the worker is restarted on its device (up to `max_restarts` per
        device); a task that fails `max_task_attempts` times aborts the sweep
        (a cell is never imputed);
      * with `checkpoint_dir`, every finished task is written as a shard and
        a re-run of the same sweep skips the tasks already on disk.
    Every task's NVML clocks / throttle reasons go into the result's log."""
    import multiprocessing as mp
    from collections import deque
    from multiprocessing import connection as mp_connection

    from . import gemm
    n_cfg = len(spec.configs) if spec.configs is not None else len(gemm.family_configs(spec.family))
    target = _worker_fn or _worker
    ctx = mp.get_context("spawn")
    ckpt = TaskCheckpoint(checkpoint_dir, _spec_key(spec, n_cfg)) if checkpoint_dir else None
    chunks, task_log = [], []
    pending = deque()
    for task in plan_tasks(spec.problems, len(devices), n_cfg, spec.batch):
        got = ckpt.load(task) if ckpt else None
        if got is not None:
            chunks.append((task[0], task[1], task[2], got[0]))
            task_log.append(dict(got[1], task=list(task), resumed=True))
        else:
            pending.append(task)
    slots = {}  # slot -> {"dev", "proc", "conn", "task", "ready", "started", "restarts"}

    def spawn(slot, dev, restarts):
        parent_conn, child_conn = ctx.Pipe(duplex=True)
        proc = ctx.Process(target=target, args=(dev, spec, child_conn), daemon=True)
        proc.start()
        child_conn.close()
        slots[slot] = {"dev": dev, "proc": proc, "conn": parent_conn, "task": None,
                       "ready": False, "started": time.monotonic(), "restarts": restarts}

    attempts: dict = {}
    facts: dict = {}

    def fail_task(slot, why):
        s = slots.pop(slot)
        task = s["task"]
        s["conn"].close()
        s["proc"].join(timeout=30)
        if s["proc"].is_alive():
            s["proc"].terminate()
            s["proc"].join(timeout=10)
        task_log.append({"event": "worker_lost", "device": s["dev"], "task": list(task or ()),
                         "why": why})
        if task is not None:
            attempts[task] = attempts.get(task, 0) + 1
            if attempts[task] >= max_task_attempts:
                raise RuntimeError(f"sweep task {task} failed {attempts[task]} times "
                                   f"(last on device {s['dev']}: {why})")
            pending.appendleft(task)
        if s["restarts"] < max_restarts and pending:
            spawn(slot, s["dev"], s["restarts"] + 1)
        if not slots and pending:
            raise RuntimeError(f"every sweep worker was lost; {len(pending)} tasks left ({why})")

    def hand_out(slot):
        s = slots[slot]
        s["task"] = pending.popleft() if pending else None
        s["conn"].send(s["task"])
        if s["task"] is None:
            s["ready"] = "stopping"

    def busy():
        return pending or any(s["task"] is not None or s["ready"] is False
                              for s in slots.values())

    t0 = time.perf_counter()
    try:
        if pending:
            for slot, dev in enumerate(devices):
                spawn(slot, dev, 0)
        while busy():
            live = {s["conn"]: k for k, s in slots.items() if s["ready"] != "stopping"}
            ready_conns = mp_connection.wait(list(live), timeout=poll_s)
            for conn in ready_conns:
                slot = live[conn]
                if slot not in slots:
                    continue
                try:
                    kind, dev_slot, task, payload = conn.recv()
                except (EOFError, OSError):
                    slots[slot]["proc"].join(timeout=10)  # reap it: exitcode is then set
                    code = slots[slot]["proc"].exitcode
                    fail_task(slot, f"worker exited with code {code} without reporting")
                    continue
                if kind == "ready":
                    slots[slot]["ready"] = True
                    facts.setdefault(dev_slot, payload)
                    hand_out(slot)
                elif kind == "row":
                    row, clocks = payload
                    chunks.append((task[0], task[1], task[2], row))
                    entry = {"task": list(task), "device": dev_slot, "clocks": clocks}
                    task_log.append(entry)
                    if ckpt:
                        ckpt.save(task, row, entry)
                    hand_out(slot)
                else:
                    fail_task(slot, f"worker error: {payload}")
            now = time.monotonic()
            for slot in list(slots):
                s = slots[slot]
                if s["ready"] == "stopping":
                    continue
                code = s["proc"].exitcode
                if code is not None and not s["conn"].poll():
                    fail_task(slot, f"worker exited with code {code} without reporting")
                elif not s["ready"] and now - s["started"] > start_timeout_s:
                    fail_task(slot, "worker never became ready")
    finally:
        for s in slots.values():
            if s["ready"] != "stopping" and s["proc"].is_alive():
                try:
                    s["conn"].send(None)
                except (OSError, ValueError):
                    pass
        for s in slots.values():
            s["proc"].join(timeout=30)
            if s["proc"].is_alive():
                s["proc"].terminate()
    wall = time.perf_counter() - t0
    grid = merge_chunks(len(spec.problems), n_cfg, chunks)
    configs = tuple(spec.configs) if spec.configs is not None else gemm.family_configs(spec.family)
    first = facts[min(facts)] if facts else {}
    return SweepResult(spec, configs, grid, wall, dict(first, devices=len(devices)),
                       task_log=task_log)


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
        "early_exit": "a config > 1 ms and > 8x the best median so far keeps its first timing "
                      "(whole-problem tasks only; config-range tasks time every config fully)",
    }
    if result.task_log:
        # NVML SM clock + throttle reasons before/after every task
        doc["task_clocks"] = result.task_log
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
