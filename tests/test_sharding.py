"""Multi-GPU sweep plumbing on CPU: shard planning, merging, and the
world_size-2 gloo gather used by bench.py (no GPU, no data-path collective)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2003_06795_b200 import measure, shapes
from paper_2003_06795_b200.dataset import ProblemSize


def test_plan_shards_partitions_and_balances():
    probs = shapes.problem_set("networks")
    for n in (1, 2, 4, 8):
        shards = measure.plan_shards(probs, n)
        flat = sorted(i for s in shards for i in s)
        assert flat == list(range(len(probs)))
        loads = [sum(measure.problem_cost(probs[i]) for i in s) for s in shards]
        if n > 1:
            # LPT bound: max load <= mean + largest single task
            assert max(loads) <= sum(loads) / n + max(measure.problem_cost(p) for p in probs)


def test_merge_shards_complete_grid():
    parts = [{0: [1.0, 2.0], 2: [3.0, 4.0]}, {1: [5.0, 6.0]}]
    grid = measure.merge_shards(3, 2, parts)
    assert grid.tolist() == [[1.0, 2.0], [5.0, 6.0], [3.0, 4.0]]
    with pytest.raises(RuntimeError):
        measure.merge_shards(3, 2, [{0: [1.0, 1.0]}])           # missing problems
    with pytest.raises(RuntimeError):
        measure.merge_shards(1, 2, [{0: [1.0, 1.0]}, {0: [1.0, 1.0]}])  # duplicate
    with pytest.raises(RuntimeError):
        measure.merge_shards(1, 2, [{0: [1.0, float("nan")]}])  # never impute


def test_config_shard_covers_space():
    for world in (1, 2, 3, 8):
        got = sorted(j for r in range(world) for j in measure.config_shard(640, r, world))
        assert got == list(range(640))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gather_worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = measure.config_shard(10, rank, world)
    local = {(p, j): float(100 * p + j) for p in range(3) for j in mine}
    merged = measure.gather_cells(local, world)
    out[rank] = sorted(merged.items())
    dist.destroy_process_group()


def test_gloo_world2_gather_cells():
    world = 2
    port = _free_port()
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_gather_worker, args=(world, port, out), nprocs=world, join=True)
    want = sorted(((p, j), float(100 * p + j)) for p in range(3) for j in range(10))
    assert out[0] == want and out[1] == want


def test_sweep_records_canonical_order():
    spec = measure.SweepSpec((ProblemSize(2, 3, 4), ProblemSize(5, 6, 7)))
    from paper_2003_06795_b200.dataset import all_configs
    cfgs = all_configs()[:3]
    rt = np.array([[10.0, 20.0, 40.0], [1.0, 2.0, 4.0]])
    res = measure.SweepResult(spec, cfgs, rt, 1.0)
    recs = res.records()
    assert [r.problem.as_tuple() for r in recs] == [(2, 3, 4)] * 3 + [(5, 6, 7)] * 3
    assert [r.config for r in recs] == list(cfgs) * 2
    assert recs[0].gflops == pytest.approx(2 * 2 * 3 * 4 / 10.0)
    assert recs[0].runtime_ns == pytest.approx(10.0)


def _reduce_worker(rank, world, port, out):
    import sys
    import torch.distributed as dist
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out[rank] = (bench.reduce_over_ranks(1.5 + rank, world, dist.group.WORLD),
                 bench.reduce_over_ranks(10 * (rank + 1), world, dist.group.WORLD, op="sum"))
    dist.destroy_process_group()


def test_bench_reductions_world2():
    """bench.py times every rank on its device and reports the max over ranks
    (launch counts summed); the reduction runs on the host gloo group."""
    port = _free_port()
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_reduce_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0] == out[1] == (2.5, 30.0)


def test_plan_tasks_splits_only_dominant_problems_and_covers_every_cell():
    import numpy as np
    from paper_2003_06795_b200 import measure, shapes
    probs = shapes.problem_set("networks+squares")
    single = measure.plan_tasks(probs, 1, 640)
    # one device: every problem exactly once, whole config range, longest first
    assert sorted(i for i, _, _ in single) == list(range(len(probs)))
    assert all((lo, hi) == (0, 640) for _, lo, hi in single)
    single_costs = [measure.problem_cost(probs[i]) for i, _, _ in single]
    assert single_costs == sorted(single_costs, reverse=True)
    for nd in (2, 4, 8):
        tasks = measure.plan_tasks(probs, nd, 640)
        cover = np.zeros((len(probs), 640), dtype=int)
        for i, lo, hi in tasks:
            assert 0 <= lo < hi <= 640
            cover[i, lo:hi] += 1
        assert (cover == 1).all()
        split = {probs[i].as_tuple() for i, lo, hi in tasks if (lo, hi) != (0, 640)}
        assert (8192, 8192, 8192) in split
        costs = [measure.problem_cost(p) for p in probs]
        # longest first: task costs are non-increasing along the queue
        per_task = [costs[i] * (hi - lo) / 640 for i, lo, hi in tasks]
        assert per_task == sorted(per_task, reverse=True)


def test_merge_chunks_contract():
    import numpy as np
    import pytest
    from paper_2003_06795_b200 import measure
    chunks = [(0, 0, 3, [1.0, 2.0, 3.0]), (1, 0, 2, [4.0, 5.0]), (1, 2, 3, [6.0])]
    grid = measure.merge_chunks(2, 3, chunks)
    assert grid.tolist() == [[1, 2, 3], [4, 5, 6]]
    with pytest.raises(RuntimeError, match="twice"):
        measure.merge_chunks(2, 3, chunks + [(1, 2, 3, [7.0])])
    with pytest.raises(RuntimeError, match="never fully measured"):
        measure.merge_chunks(2, 3, chunks[:2])
    with pytest.raises(RuntimeError, match="non-positive"):
        measure.merge_chunks(1, 1, [(0, 0, 1, [0.0])])
    assert np.isfinite(grid).all()


# ---- run_sharded robustness (fake workers, same protocol, no GPU) ----------

def _fake_spec(n_problems=5, n_configs=7):
    from paper_2003_06795_b200.dataset import KernelConfig
    probs = tuple(ProblemSize(64 * (i + 1), 64, 64) for i in range(n_problems))
    cfgs = tuple(KernelConfig(1, 1, 1, 8, 8) for _ in range(n_configs))
    return measure.SweepSpec(probs, configs=cfgs)


def _expected(spec):
    import _fake_sweep_worker as fw
    return np.array([[fw.cell(i, j) for j in range(len(spec.configs))]
                     for i in range(len(spec.problems))])


@pytest.fixture
def fake_markers(tmp_path, monkeypatch):
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    d = tmp_path / "markers"
    d.mkdir()
    monkeypatch.setenv("KP_FAKE_MARKERS", str(d))
    yield d
    sys.path.remove(os.path.dirname(__file__))


def test_run_sharded_merges_every_task(fake_markers):
    import _fake_sweep_worker as fw
    spec = _fake_spec()
    res = measure.run_sharded(spec, [0, 1], _worker_fn=fw.healthy, poll_s=0.2)
    assert np.array_equal(res.runtime_ns, _expected(spec))
    assert sorted(tuple(e["task"]) for e in res.task_log) == sorted(
        measure.plan_tasks(spec.problems, 2, len(spec.configs)))


def test_run_sharded_requeues_a_dead_workers_task(fake_markers):
    """A worker that dies without a message is detected by the liveness poll,
    its in-flight task re-runs on a restarted worker, and the grid is whole."""
    import _fake_sweep_worker as fw
    spec = _fake_spec()
    res = measure.run_sharded(spec, [0, 1], _worker_fn=fw.crashes_once_on_problem_1,
                              poll_s=0.2)
    assert np.array_equal(res.runtime_ns, _expected(spec))
    lost = [e for e in res.task_log if e.get("event") == "worker_lost"]
    # problem 1 may be cut into config ranges: each range's first attempt dies once
    assert lost and all(e["task"][0] == 1 and "code 9" in e["why"] for e in lost)


def test_run_sharded_aborts_on_a_task_that_keeps_failing(fake_markers):
    import _fake_sweep_worker as fw
    spec = _fake_spec()
    with pytest.raises(RuntimeError, match=r"task \(2, 0, 7\) failed 2 times"):
        measure.run_sharded(spec, [0], _worker_fn=fw.always_fails_on_problem_2, poll_s=0.2)


def test_run_sharded_resumes_from_task_shards(fake_markers, tmp_path):
    import _fake_sweep_worker as fw
    spec = _fake_spec()
    ckpt = tmp_path / "ckpt"
    with pytest.raises(RuntimeError):
        measure.run_sharded(spec, [0], _worker_fn=fw.always_fails_on_problem_2, poll_s=0.2,
                            checkpoint_dir=ckpt)
    done_before = sorted(p.name for p in ckpt.glob("task_*.json"))
    assert done_before and "task_p2_c0-7.json" not in done_before
    res = measure.run_sharded(spec, [0], _worker_fn=fw.healthy, poll_s=0.2,
                              checkpoint_dir=ckpt)
    assert np.array_equal(res.runtime_ns, _expected(spec))
    resumed = {tuple(e["task"]) for e in res.task_log if e.get("resumed")}
    assert len(resumed) == len(done_before)
    other = measure.SweepSpec(spec.problems[:2], configs=spec.configs)
    with pytest.raises(RuntimeError, match="different sweep"):
        measure.run_sharded(other, [0], _worker_fn=fw.healthy, checkpoint_dir=ckpt)
