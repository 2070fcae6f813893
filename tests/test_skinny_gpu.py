"""Small-M path (kp_gemm_skinny / kp_gemm_auto for m <= 16) on the B200.

The FC-layer GEMMs of the paper's dataset at batch 1-16.
Numerics: fp32 FMA accumulation in a launch-fixed order (warp partials
through shared memory, a warp-shuffle butterfly, split-K partials in split
order), so the check is the float64 oracle within the K-scaled elementwise
bound c*K*u*(|A||B|) with u = 2^-24 (fp32 inputs: F32 and TF32 families) or
the fp32 accumulation bound on exact bf16 products (BF16 family), plus
run-to-run bit-identity (determinism).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

# fp32 accumulation roundoff (the products of bf16 / fp32 inputs are formed
# in fp32 FMA; bf16 x bf16 products are exact in fp32)
U32 = 2.0 ** -24
LAYOUTS = [(False, False), (False, True), (True, False), (True, True)]


def _gemm():
    from paper_2003_06795_b200 import gemm
    return gemm


def _operands(family, m, k, n, ta, tb, seed, batch=1, pad=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    dt = torch.bfloat16 if family == "bf16" else torch.float32
    pre = (batch,) if batch > 1 else ()

    def mk(rows, cols):
        full = torch.rand(pre + (rows, cols + pad), generator=g, device="cuda") * 2 - 1
        return full.to(dt)[..., :cols]
    a = mk(k, m).transpose(-1, -2) if ta else mk(m, k)
    b = mk(n, k).transpose(-1, -2) if tb else mk(k, n)
    return a, b


def _check(got, la, lb, k, c_in=None, alpha=1.0, beta=0.0):
    an = la.float().cpu().numpy().astype(np.float64)
    bn = lb.float().cpu().numpy().astype(np.float64)
    ref = alpha * np.matmul(an, bn)
    bound = 4.0 * k * U32 * abs(alpha) * np.matmul(np.abs(an), np.abs(bn)) + 1e-30
    if c_in is not None:
        ref = ref + beta * c_in
        bound = bound + 2 * U32 * np.abs(beta * c_in)
    g = got.cpu().numpy().astype(np.float64)
    err = np.abs(g - ref)
    assert np.all(err <= bound), f"max err/bound {np.max(err / bound):.3f}"
    rel = np.linalg.norm(g - ref) / max(np.linalg.norm(ref), 1e-30)
    assert rel <= max(1e-5, 8 * np.sqrt(k) * U32), rel


@pytest.mark.parametrize("family", ["f32", "tf32", "bf16"])
@pytest.mark.parametrize("ta,tb", LAYOUTS)
@pytest.mark.parametrize("m", [1, 3, 8, 16])
def test_layouts_rows(family, ta, tb, m):
    gemm = _gemm()
    k, n = 1000, 520
    a, b = _operands(family, m, k, n, ta, tb, seed=m * 10 + 2 * ta + tb)
    c = gemm.matmul(a, b, "skinny", family=family)
    torch.cuda.synchronize()
    _check(c, a, b, k)


@pytest.mark.parametrize("family", ["f32", "bf16"])
@pytest.mark.parametrize("tb", [False, True])
@pytest.mark.parametrize("mkn", [(1, 25088, 4096), (16, 4096, 4096), (4, 4096, 1000),
                                 (2, 2048, 1000), (7, 1280, 1000)])
def test_fc_layers(family, tb, mkn):
    """VGG16 fc6/fc7/fc8, ResNet-50 fc, MobileNetV2 fc shapes (K split
    across many CTAs for fc6)."""
    gemm = _gemm()
    m, k, n = mkn
    a, b = _operands(family, m, k, n, False, tb, seed=k + n + m)
    c = gemm.matmul(a, b, "skinny", family=family)
    torch.cuda.synchronize()
    _check(c, a, b, k)


@pytest.mark.parametrize("family", ["f32", "bf16"])
@pytest.mark.parametrize("ta,tb", LAYOUTS)
def test_ragged_unaligned(family, ta, tb):
    """Odd n / k and row pitches that are not 16-byte multiples: the scalar
    (VEC = 1) kernels."""
    gemm = _gemm()
    m, k, n = 5, 777, 333
    a, b = _operands(family, m, k, n, ta, tb, seed=11, pad=1)
    c = gemm.matmul(a, b, "skinny", family=family)
    torch.cuda.synchronize()
    _check(c, a, b, k)


@pytest.mark.parametrize("family", ["f32", "bf16"])
@pytest.mark.parametrize("tb", [False, True])
def test_alpha_beta_batched(family, tb):
    gemm = _gemm()
    m, k, n, bt = 4, 3000, 384, 3
    a, b = _operands(family, m, k, n, False, tb, seed=5, batch=bt)
    c0 = torch.rand((bt, m, n), device="cuda") * 2 - 1
    c = c0.clone()
    gemm.matmul(a, b, "skinny", family=family, out=c, alpha=0.5, beta=-2.0)
    torch.cuda.synchronize()
    for i in range(bt):
        _check(c[i], a[i], b[i], k, c_in=c0[i].cpu().numpy().astype(np.float64),
               alpha=0.5, beta=-2.0)


@pytest.mark.parametrize("family", ["f32", "bf16"])
@pytest.mark.parametrize("tb", [False, True])
def test_deterministic(family, tb):
    gemm = _gemm()
    m, k, n = 8, 25088, 1024
    a, b = _operands(family, m, k, n, False, tb, seed=3)
    first = gemm.matmul(a, b, "skinny", family=family).clone()
    for _ in range(3):
        again = gemm.matmul(a, b, "skinny", family=family)
        torch.cuda.synchronize()
        assert torch.equal(first, again)


def test_auto_routes_small_m():
    gemm = _gemm()
    assert gemm.auto_config(1, 25088, 4096) == "skinny"
    assert gemm.auto_config(16, 4096, 4096) == "skinny"
    assert gemm.auto_config(4, 4096, 4096, family="bf16") == "skinny"
    assert gemm.auto_config(8, 4096, 4096, family="bf16") != "skinny"
    assert gemm.auto_config(17, 4096, 4096) != "skinny"
    assert gemm.auto_config(4, 32, 4096) != "skinny"  # k < 64: tile path
    prev = gemm.set_skinny(0)
    try:
        assert gemm.auto_config(1, 25088, 4096) != "skinny"
    finally:
        gemm.set_skinny(prev)
    # kp_gemm_auto runs the same path and reports it
    a, b = _operands("f32", 2, 4096, 1000, False, False, seed=9)
    c = gemm.matmul(a, b, None)
    torch.cuda.synchronize()
    _check(c, a, b, 4096)


def test_m_above_16_is_rejected():
    gemm = _gemm()
    from paper_2003_06795_b200._native import UnsupportedVariant
    a, b = _operands("f32", 17, 256, 256, False, False, seed=1)
    with pytest.raises(UnsupportedVariant):
        gemm.matmul(a, b, "skinny")
