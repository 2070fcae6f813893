"""Parity on the BASELINE configs[2] network GEMMs through the runtime selector.

The sweep times every config on these shapes without looking at the output;
here the compiled selectors' picks (kp_gemm_auto, the deployed path) run them
and are checked:
  * FP32 (K1): bit-identical to the sequential-fmaf oracle (oracle/gemm_ref.c)
    on sampled rows -- each C element is one fmaf chain in increasing k, so a
    row subset of A is an exact sub-problem;
  * TF32 / BF16 (K2/K3): float64 oracle on sampled rows within c*K*u*(|A||B|).
Shapes (shapes.py): VGG16 FC6 at batch 1 and 16
(1x25088x4096, 16x25088x4096), VGG conv1_1 at batch 8 (401408x27x64),
ResNet-50 conv1 at batch 4 (50176x147x64), ResNet-50 c5_3x3 at batch 8
(392x4608x512), MobileNetV2 b1_project at batch 2 (25088x32x16).
"""

import numpy as np
import pytest

from oracle.gemm_oracle import gemm_f32_exact, gemm_f64

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

LAYOUTS = [(False, False), (False, True), (True, False), (True, True)]
NET = {
    "fc6_b1": (1, 25088, 4096),
    "fc6_b16": (16, 25088, 4096),
    "conv1_1_b8": (401408, 27, 64),
    "resnet_conv1_b4": (50176, 147, 64),
    "c5_3x3_b8": (392, 4608, 512),
    "mbv2_b1_project_b2": (25088, 32, 16),
}
U = {"tf32": 2.0 ** -10, "bf16": 2.0 ** -8}


def _gemm():
    from paper_2003_06795_b200 import gemm
    return gemm


def _rows(m, seed, count=48):
    rng = np.random.default_rng(seed)
    return np.unique(np.concatenate([[0, m - 1], rng.integers(0, m, min(m, count))]))


def _store(m, k, n, ta, tb, seed, dtype=torch.float32, pad_to=1):
    """Operands in storage orientation; row pitch padded to a multiple of pad_to."""
    g = torch.Generator(device="cuda").manual_seed(seed)

    def mk(rows, cols):
        pitch = -(-cols // pad_to) * pad_to
        t = (torch.rand((rows, pitch), generator=g, device="cuda") * 2 - 1).to(dtype)
        return t[:, :cols]  # slice after the cast: .to() of a padded view would repack it

    a = mk(k, m) if ta else mk(m, k)
    b = mk(n, k) if tb else mk(k, n)
    return a, b


@pytest.mark.parametrize("ta,tb", LAYOUTS)
@pytest.mark.parametrize("name", list(NET))
def test_f32_selected_bit_exact(name, ta, tb):
    m, k, n = NET[name]
    gemm = _gemm()
    a, b = _store(m, k, n, ta, tb, seed=len(name) + 2 * ta + tb)
    la = a.t() if ta else a
    lb = b.t() if tb else b
    cfg = gemm.select(m, k, n, family="f32", trans_a=ta, trans_b=tb)
    got = gemm.matmul(la, lb, cfg).cpu().numpy()  # the tree's tile config
    rows = _rows(m, seed=m + k)
    a_np = a.cpu().numpy()
    b_np = b.cpu().numpy()
    a_sub = a_np[:, rows] if ta else a_np[rows]
    want = gemm_f32_exact(a_sub, b_np, m=len(rows), k=k, n=n, trans_a=ta,
                          trans_b=tb).reshape(len(rows), n)
    np.testing.assert_array_equal(got[rows], want, err_msg=f"{name} {ta}{tb} {cfg.as_tuple()}")
    if gemm.auto_config(m, k, n, family="f32", trans_a=ta, trans_b=tb) == "skinny":
        # kp_gemm_auto runs the small-M path here: fp64 oracle within the bound
        auto = gemm.matmul(la, lb).double().cpu().numpy()
        an = (a_np.T if ta else a_np).astype(np.float64)
        ref = an @ (b_np.T if tb else b_np).astype(np.float64)
        bound = 4.0 * k * 2.0 ** -24 * (np.abs(an) @ np.abs((b_np.T if tb else b_np)
                                                           .astype(np.float64))) + 1e-30
        assert (np.abs(auto - ref) <= bound).all(), name


@pytest.mark.parametrize("family", ["tf32", "bf16"])
@pytest.mark.parametrize("ta,tb", LAYOUTS)
@pytest.mark.parametrize("name", list(NET))
def test_tc_selected_within_bound(family, name, ta, tb):
    m, k, n = NET[name]
    gemm = _gemm()
    dt = torch.bfloat16 if family == "bf16" else torch.float32
    es = 2 if family == "bf16" else 4
    # TMA needs 16-byte row pitches: operands live in padded storage (the
    # logical shape is unchanged; the kernel never reads the pad)
    a, b = _store(m, k, n, ta, tb, seed=len(name) + 2 * ta + tb + 7, dtype=dt, pad_to=16 // es)
    la = a.t() if ta else a
    lb = b.t() if tb else b
    got = gemm.matmul(la, lb, family=family).double().cpu().numpy()
    rows = _rows(m, seed=m + n)
    an = la.float().cpu().numpy().astype(np.float64)
    bn = lb.float().cpu().numpy().astype(np.float64)
    ref = gemm_f64(an[rows], bn)
    bound = 2.0 * k * U[family] * np.matmul(np.abs(an[rows]), np.abs(bn)) + 1e-30
    err = np.abs(got[rows] - ref)
    assert (err <= bound).all(), (family, name, ta, tb, float((err / bound).max()))
