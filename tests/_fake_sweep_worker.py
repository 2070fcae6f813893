"""Stand-in sweep workers for the CPU tests of measure.run_sharded (same
message protocol as measure._worker, no GPU): runtimes are a pure function of
(problem, config) so merged grids can be checked exactly."""

import os
from pathlib import Path


def cell(i, j):
    return 1000.0 + 10.0 * i + j


def _serve(device, spec, conn, crash_on=None, error_on=None):
    conn.send(("ready", device, None, {"name": "fake", "sm_count": 148}))
    while True:
        task = conn.recv()
        if task is None:
            return
        i, lo, hi = task
        marker = Path(os.environ["KP_FAKE_MARKERS"]) / f"p{i}_{lo}_{hi}"
        first = not marker.exists()
        marker.touch()
        if crash_on is not None and i == crash_on and first:
            os._exit(9)  # dies without a message, like a segfault / OOM kill
        if error_on is not None and i == error_on:
            conn.send(("error", device, task, "RuntimeError('boom')"))
            raise SystemExit(1)
        conn.send(("row", device, task, ([cell(i, j) for j in range(lo, hi)],
                                         {"before": None, "after": None})))


def healthy(device, spec, conn):
    _serve(device, spec, conn)


def crashes_once_on_problem_1(device, spec, conn):
    _serve(device, spec, conn, crash_on=1)


def always_fails_on_problem_2(device, spec, conn):
    _serve(device, spec, conn, error_on=2)
