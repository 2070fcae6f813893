"""K2/K3 parity where the persistent schedules actually persist.

Round-1 tensor-core tests never gave a persistent CTA (wg 16x16, NBUF = 2)
or a CTA pair (row_tile 2, cta_group::2) more than one tile, so the
double-buffered TMEM accumulator (buffer = tile parity, acc_empty phases) and
the TMA ring running across tile boundaries were unchecked. Every case here
gives each persistent CTA / pair >= 3 tiles, in all four layouts and both
families, and the 8192^3 cases cover the configs the large-size table reports.

Checks (float64 oracle, oracle/gemm_oracle.py, on the same rounded inputs):
  * sampled rows -- rows from every 128-row tile, all four TMEM lane
    quarters, the last row -- elementwise within c*K*u*(|A||B|)_ij;
  * column sums 1^T C against (1^T A) B and row sums C 1 against A (B 1),
    within the summed elementwise bound: a wrong element anywhere (a tile
    written from the wrong TMEM buffer, a stale ring stage) shifts a sum.
"""

import numpy as np
import pytest

from oracle.gemm_oracle import gemm_f64

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

U = {"tf32": 2.0 ** -10, "bf16": 2.0 ** -8}
LAYOUTS = [(False, False), (False, True), (True, False), (True, True)]


def _gemm():
    from paper_2003_06795_b200 import gemm
    return gemm


def _tiles_per_worker(cfg, m, n):
    """Tiles each persistent CTA (or CTA pair) runs at one tile per 148 SMs."""
    acc, rt, ct, wr, wc = cfg
    bn = {1: 32, 2: 64, 4: 128, 8: 256}[ct]
    bm = 256 if rt == 2 else 128
    tiles = -(-m // bm) * -(-n // bn)
    workers = 74 if rt == 2 else 148
    return tiles / min(tiles, workers)


def _operands(family, m, k, n, ta, tb, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    dt = torch.bfloat16 if family == "bf16" else torch.float32
    a = (torch.rand((k, m) if ta else (m, k), generator=g, device="cuda") * 2 - 1).to(dt)
    b = (torch.rand((n, k) if tb else (k, n), generator=g, device="cuda") * 2 - 1).to(dt)
    la = a.t() if ta else a
    lb = b.t() if tb else b
    return la, lb


def check_large(family, cfg, m, k, n, ta, tb, seed=0, rows_per_tile=5):
    la, lb = _operands(family, m, k, n, ta, tb, seed)
    got_t = _gemm().matmul(la, lb, cfg, family=family)
    torch.cuda.synchronize()
    assert torch.isfinite(got_t).all()
    got = got_t.double().cpu().numpy()
    an = la.float().cpu().numpy().astype(np.float64)
    bn = lb.float().cpu().numpy().astype(np.float64)
    u = U[family]
    rng = np.random.default_rng(seed)
    rows = set([m - 1])
    for t0 in range(0, m, 128):
        span = min(128, m - t0)
        for q in range(4):  # one row in each TMEM lane quarter
            lo, hi = q * 32, min(span, (q + 1) * 32)
            if lo < hi:
                rows.add(t0 + int(rng.integers(lo, hi)))
        rows.update(t0 + int(r) for r in rng.integers(0, span, rows_per_tile - 4))
    rows = np.array(sorted(rows))
    ref = gemm_f64(an[rows], bn)
    bound = 2.0 * k * u * np.matmul(np.abs(an[rows]), np.abs(bn)) + 1e-30
    err = np.abs(got[rows] - ref)
    worst = float((err / bound).max())
    assert (err <= bound).all(), (family, cfg, (m, k, n, ta, tb), "rows", worst)
    abs_a, abs_b = np.abs(an), np.abs(bn)
    col_ref = an.sum(0) @ bn
    col_bound = 2.0 * k * u * (abs_a.sum(0) @ abs_b) + 1e-9
    assert (np.abs(got.sum(0) - col_ref) <= col_bound).all(), (family, cfg, "column sums")
    row_ref = an @ bn.sum(1)
    row_bound = 2.0 * k * u * (abs_a @ abs_b.sum(1)) + 1e-9
    assert (np.abs(got.sum(1) - row_ref) <= row_bound).all(), (family, cfg, "row sums")


# (config, m, k, n): persistent 1-CTA (NBUF = 2) and CTA pairs, >= 3 tiles each
MULTITILE = [
    ((1, 1, 1, 16, 16), 2048, 512, 2048),   # BN 32: 1024 tiles, ~7 per CTA
    ((4, 1, 2, 16, 16), 2048, 520, 2048),   # BN 64: 512 tiles, ragged K
    ((8, 1, 4, 16, 16), 2176, 256, 4160),   # BN 128: 17 x 33 tiles, M/N tails
    ((8, 1, 8, 16, 16), 4096, 256, 4096),   # BN 256: 512 tiles
    ((2, 2, 4, 16, 16), 4096, 256, 2048),   # pair BN 128: 256 pair tiles
    ((8, 2, 8, 16, 16), 4096, 264, 4352),   # pair BN 256: 272 pair tiles, N tail
]


@pytest.mark.parametrize("family", ["bf16", "tf32"])
@pytest.mark.parametrize("ta,tb", LAYOUTS)
@pytest.mark.parametrize("case", MULTITILE, ids=lambda c: "x".join(map(str, c[0])))
def test_persistent_multitile(family, ta, tb, case):
    cfg, m, k, n = case
    assert _tiles_per_worker(cfg, m, n) >= 3
    check_large(family, cfg, m, k, n, ta, tb, seed=m + n + cfg[0])


@pytest.mark.parametrize("family", ["bf16", "tf32"])
def test_persistent_batched_multitile(family):
    """Batch-major tile order across a persistent CTA's tiles (3-D TMA maps)."""
    gemm = _gemm()
    g = torch.Generator(device="cuda").manual_seed(5)
    dt = torch.bfloat16 if family == "bf16" else torch.float32
    a = (torch.rand((3, 640, 192), generator=g, device="cuda") * 2 - 1).to(dt)
    b = (torch.rand((3, 192, 1536), generator=g, device="cuda") * 2 - 1).to(dt)
    for cfg in [(2, 1, 1, 16, 16), (4, 2, 4, 16, 16)]:
        got = gemm.matmul(a, b, cfg, family=family).double().cpu().numpy()
        an = a.float().cpu().numpy().astype(np.float64)
        bn = b.float().cpu().numpy().astype(np.float64)
        ref = np.matmul(an, bn)
        bound = 2.0 * 192 * U[family] * np.matmul(np.abs(an), np.abs(bn)) + 1e-30
        assert (np.abs(got - ref) <= bound).all(), (family, cfg)


# the configs tools/large_sizes.py reports at 8192^3 (the large-size table)
LARGE_8192 = [(4, 1, 8, 16, 16), (8, 1, 8, 16, 16), (4, 2, 8, 16, 16), (8, 2, 8, 16, 16),
              (4, 1, 8, 8, 8)]


@pytest.mark.parametrize("family", ["bf16", "tf32"])
@pytest.mark.parametrize("cfg", LARGE_8192, ids=lambda c: "x".join(map(str, c)))
def test_8192_cubed_sampled(family, cfg):
    check_large(family, cfg, 8192, 8192, 8192, False, False, seed=81, rows_per_tile=4)


@pytest.mark.parametrize("family", ["bf16", "tf32"])
@pytest.mark.parametrize("ta,tb", [(False, True), (True, False), (True, True)])
def test_8192_cubed_layouts_selected(family, ta, tb):
    cfg = _gemm().select(8192, 8192, 8192, family=family, trans_a=ta, trans_b=tb)
    check_large(family, cfg.as_tuple(), 8192, 8192, 8192, ta, tb, seed=82, rows_per_tile=4)
