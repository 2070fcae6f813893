"""K2/K3 (tcgen05 TF32 / BF16) parity on the B200 through the C-ABI.

Reference: float64 matmul of the same inputs (BF16 inputs are exact in fp64;
TF32 inputs are truncated/rounded by the tensor core, so the bound uses the
TF32 unit roundoff). Tolerance (north_star: "scaled by K"):
    |C - C64| <= c * K * u * (|A| |B|)_ij      c = 2 (bf16, u = 2^-8),
                                               c = 2 (tf32, u = 2^-10, truncation)
plus rel-Frobenius <= 8 * u.
"""

import numpy as np
import pytest

from oracle.gemm_oracle import gemm_f64

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

U = {"tf32": 2.0 ** -10, "bf16": 2.0 ** -8}


def _gemm():
    from paper_2003_06795_b200 import gemm
    return gemm


def _check(family, cfg, m, k, n, ta, tb, batch=1, seed=0):
    rng = np.random.default_rng(seed)
    dt = torch.bfloat16 if family == "bf16" else torch.float32
    a_shape = (k, m) if ta else (m, k)
    b_shape = (n, k) if tb else (k, n)
    if batch > 1:
        a_shape, b_shape = (batch,) + a_shape, (batch,) + b_shape
    a = torch.from_numpy(rng.uniform(-1, 1, a_shape).astype(np.float32)).cuda().to(dt)
    b = torch.from_numpy(rng.uniform(-1, 1, b_shape).astype(np.float32)).cuda().to(dt)
    la = a.transpose(-1, -2) if ta else a
    lb = b.transpose(-1, -2) if tb else b
    got = _gemm().matmul(la, lb, cfg, family=family).cpu().numpy().astype(np.float64)
    an = la.float().cpu().numpy().astype(np.float64)
    bn = lb.float().cpu().numpy().astype(np.float64)
    ref = gemm_f64(an, bn)
    bound = 2.0 * k * U[family] * np.matmul(np.abs(an), np.abs(bn)) + 1e-30
    err = np.abs(got - ref)
    assert (err <= bound).all(), (family, cfg, (m, k, n, ta, tb), float((err / bound).max()))
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert rel <= 8 * U[family], rel


@pytest.mark.parametrize("family", ["bf16", "tf32"])
def test_family_configs_enumerate(family):
    cfgs = _gemm().family_configs(family)
    assert len(cfgs) == 40
    assert list(cfgs) == sorted(cfgs)


@pytest.mark.parametrize("family", ["bf16", "tf32"])
@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False), (True, True)])
def test_all_configs_layouts(family, ta, tb):
    for cfg in _gemm().family_configs(family):
        _check(family, cfg, 200, 136, 264, ta, tb, seed=cfg.acc * 10 + cfg.col_tile)


@pytest.mark.parametrize("family", ["bf16", "tf32"])
@pytest.mark.parametrize("shape", [(1, 8, 8), (128, 64, 256), (257, 520, 136), (1024, 1024, 1024)])
def test_shapes(family, shape):
    for cfg in [(1, 1, 1, 8, 8), (4, 1, 4, 8, 8), (8, 1, 8, 8, 8), (4, 1, 8, 16, 16), (4, 2, 8, 16, 16)]:
        _check(family, cfg, *shape, ta=False, tb=False, seed=7)


@pytest.mark.parametrize("family", ["bf16", "tf32"])
def test_batched(family):
    _check(family, (2, 1, 2, 8, 8), 96, 72, 136, False, False, batch=3, seed=11)
    _check(family, (2, 1, 8, 8, 8), 96, 72, 136, True, True, batch=2, seed=12)


def test_alignment_error():
    from paper_2003_06795_b200 import _native as nat
    a = torch.ones(64, 27, device="cuda")   # row pitch 108 B: not 16-byte aligned
    b = torch.ones(27, 64, device="cuda")
    with pytest.raises(nat.BadProblemShape):
        _gemm().matmul(a, b, (1, 1, 1, 8, 8), family="tf32")


@pytest.mark.parametrize("family", ["bf16", "tf32"])
@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False), (True, True)])
def test_runtime_selection_every_layout(family, ta, tb):
    """kp_gemm_auto has a compiled selector for every tensor-core layout;
    the selected kernel stays within the K-scaled bound."""
    gemm = _gemm()
    for (m, k, n) in [(200, 576, 64), (1000, 128, 264)]:
        cfg = gemm.select(m, k, n, family=family, trans_a=ta, trans_b=tb)
        _check(family, cfg, m, k, n, ta, tb, seed=m + k + n)
