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


def _check_views(family, cfg, la, lb):
    """Run on (possibly unaligned) views and compare with fp64."""
    got = _gemm().matmul(la, lb, cfg, family=family).cpu().numpy().astype(np.float64)
    an = la.float().cpu().numpy().astype(np.float64)
    bn = lb.float().cpu().numpy().astype(np.float64)
    k = an.shape[-1]
    ref = np.matmul(an, bn)
    bound = 2.0 * k * U[family] * np.matmul(np.abs(an), np.abs(bn)) + 1e-30
    assert (np.abs(got - ref) <= bound).all(), (family, cfg, la.shape, lb.shape)


@pytest.mark.parametrize("family", ["bf16", "tf32"])
@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False), (True, True)])
@pytest.mark.parametrize("cfg", [(1, 1, 1, 8, 8), (4, 1, 4, 16, 16), (2, 2, 4, 16, 16)])
def test_unaligned_operands_are_staged(family, ta, tb, cfg):
    """Row pitches that are not 16-byte multiples (K = 27, the VGG conv1_1
    im2col width; odd M / N pitches) and a misaligned base run through the
    stream-ordered padded staging copy instead of failing."""
    g = torch.Generator(device="cuda").manual_seed(3)
    dt = torch.bfloat16 if family == "bf16" else torch.float32
    m, k, n = 300, 27, 77
    a = (torch.rand((k, m) if ta else (m, k), generator=g, device="cuda") * 2 - 1).to(dt)
    b = (torch.rand((n, k) if tb else (k, n), generator=g, device="cuda") * 2 - 1).to(dt)
    _check_views(family, cfg, a.t() if ta else a, b.t() if tb else b)
    # misaligned base: a view starting one element into its storage
    big = (torch.rand(m * k + 1, generator=g, device="cuda") * 2 - 1).to(dt)
    a2 = big[1:].view(m, k)
    _check_views(family, cfg, a2, b.t() if tb else b)


@pytest.mark.parametrize("family", ["bf16", "tf32"])
def test_unaligned_batched_and_broadcast(family):
    g = torch.Generator(device="cuda").manual_seed(4)
    dt = torch.bfloat16 if family == "bf16" else torch.float32
    a = (torch.rand((3, 130, 147), generator=g, device="cuda") * 2 - 1).to(dt)  # ResNet conv1 K
    b = (torch.rand((147, 65), generator=g, device="cuda") * 2 - 1).to(dt)     # broadcast B
    got = _gemm().matmul(a, b, (2, 1, 2, 8, 8), family=family).cpu().double()
    for i in range(3):
        an = a[i].float().cpu().double()
        ref = an @ b.float().cpu().double()
        bound = 2.0 * 147 * U[family] * (an.abs() @ b.float().cpu().double().abs()) + 1e-30
        assert bool(((got[i] - ref).abs() <= bound).all())


@pytest.mark.parametrize("family", ["bf16", "tf32"])
@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False), (True, True)])
def test_runtime_selection_every_layout(family, ta, tb):
    """kp_gemm_auto has a compiled selector for every tensor-core layout;
    the selected kernel stays within the K-scaled bound."""
    gemm = _gemm()
    for (m, k, n) in [(200, 576, 64), (1000, 128, 264)]:
        cfg = gemm.select(m, k, n, family=family, trans_a=ta, trans_b=tb)
        _check(family, cfg, m, k, n, ta, tb, seed=m + k + n)
