"""Split-K of the tcgen05 1-CTA kernels (kp_set_tc_split) on the B200.

* forced splits (2, 3, 5, 64 -> clamped to the K stages) in all four layouts and
  both families stay within the K-scaled bound of the float64 oracle;
* results are run-to-run bit-identical: the reduce kernel sums every
  element's partials in split order 0..S-1 whatever order the units finish in;
* persistent CTAs (wg 16x16) cycling through several split units, batched
  problems, alpha / beta, and M / N / K tails;
* the auto policy on the under-filled deep-K network GEMM it exists for
  (ResNet-50 c5_3x3 at batch 8, 392 x 4608 x 512).
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


class split_mode:
    def __init__(self, mode):
        self.mode = mode

    def __enter__(self):
        from paper_2003_06795_b200 import _native as nat
        self.prev = nat.lib().kp_set_tc_split(self.mode)
        assert self.prev >= 0

    def __exit__(self, *exc):
        from paper_2003_06795_b200 import _native as nat
        nat.lib().kp_set_tc_split(self.prev)


def _operands(family, m, k, n, ta, tb, seed, batch=1):
    g = torch.Generator(device="cuda").manual_seed(seed)
    dt = torch.bfloat16 if family == "bf16" else torch.float32
    pre = (batch,) if batch > 1 else ()
    a = (torch.rand(pre + ((k, m) if ta else (m, k)), generator=g, device="cuda") * 2 - 1).to(dt)
    b = (torch.rand(pre + ((n, k) if tb else (k, n)), generator=g, device="cuda") * 2 - 1).to(dt)
    return (a.transpose(-1, -2) if ta else a), (b.transpose(-1, -2) if tb else b)


def _check(family, got, la, lb, k, c_in=None, alpha=1.0, beta=0.0):
    an = la.float().cpu().numpy().astype(np.float64)
    bn = lb.float().cpu().numpy().astype(np.float64)
    ref = alpha * np.matmul(an, bn)
    if c_in is not None:
        ref = ref + beta * c_in
    bound = 2.0 * k * U[family] * abs(alpha) * np.matmul(np.abs(an), np.abs(bn)) + 1e-30
    if c_in is not None:
        bound = bound + 2.0 ** -23 * np.abs(beta * c_in) + 1e-6
    err = np.abs(got - ref)
    assert (err <= bound).all(), float((err / bound).max())


@pytest.mark.parametrize("family", ["bf16", "tf32"])
@pytest.mark.parametrize("ta,tb", LAYOUTS)
@pytest.mark.parametrize("splits", [2, 3, 5, 64])
def test_forced_splits_within_bound_and_deterministic(family, ta, tb, splits):
    gemm = _gemm()
    m, k, n = 296, 1000, 200   # 3 x (1..7) tiles, ragged K; 16-byte pitches in every layout
    la, lb = _operands(family, m, k, n, ta, tb, seed=splits * 4 + 2 * ta + tb)
    with split_mode(splits):
        for cfg in [(2, 1, 2, 8, 8), (4, 1, 4, 8, 8), (1, 1, 8, 8, 8)]:
            first = gemm.matmul(la, lb, cfg, family=family)
            again = gemm.matmul(la, lb, cfg, family=family)
            assert torch.equal(first, again), (cfg, "split-K result not deterministic")
            _check(family, first.double().cpu().numpy(), la, lb, k)


@pytest.mark.parametrize("family", ["bf16", "tf32"])
def test_split_persistent_cycles_through_units(family):
    """wg 16x16 configs: a persistent CTA runs several (tile, split) units with
    the double-buffered accumulator; 64 tiles x 3 splits = 192 units > 148."""
    gemm = _gemm()
    la, lb = _operands(family, 1024, 1024, 1024, False, False, seed=3)
    with split_mode(3):
        for cfg in [(4, 1, 4, 16, 16), (2, 1, 1, 16, 16)]:
            got = gemm.matmul(la, lb, cfg, family=family)
            _check(family, got.double().cpu().numpy(), la, lb, 1024)


@pytest.mark.parametrize("family", ["bf16", "tf32"])
def test_split_batched_alpha_beta(family):
    gemm = _gemm()
    la, lb = _operands(family, 136, 520, 72, True, False, seed=9, batch=3)
    c0 = torch.rand((3, 136, 72), device="cuda") * 2 - 1
    c_in = c0.double().cpu().numpy()
    with split_mode(4):
        out = c0.clone()
        gemm.matmul(la, lb, (4, 1, 2, 8, 8), family=family, out=out, alpha=0.5, beta=-2.0)
    _check(family, out.double().cpu().numpy(), la, lb, 520, c_in=c_in, alpha=0.5, beta=-2.0)


@pytest.mark.parametrize("family", ["bf16", "tf32"])
def test_auto_split_on_deep_k_network_gemm(family):
    """c5_3x3 at batch 8: 16 tiles of 128x128 -> auto splits; same bound as
    split-K off, and the split result is deterministic."""
    gemm = _gemm()
    la, lb = _operands(family, 392, 4608, 512, False, True, seed=5)
    cfg = (4, 1, 4, 8, 8)
    with split_mode(1):
        auto1 = gemm.matmul(la, lb, cfg, family=family)
        auto2 = gemm.matmul(la, lb, cfg, family=family)
    with split_mode(0):
        whole = gemm.matmul(la, lb, cfg, family=family)
    assert torch.equal(auto1, auto2)
    _check(family, auto1.double().cpu().numpy(), la, lb, 4608)
    _check(family, whole.double().cpu().numpy(), la, lb, 4608)
    assert not torch.equal(auto1, whole), "auto policy did not split the 16-tile grid"


def test_split_mode_validation():
    from paper_2003_06795_b200 import _native as nat
    lib = nat.lib()
    prev = lib.kp_set_tc_split(1)
    assert lib.kp_set_tc_split(-1) == -1
    assert lib.kp_set_tc_split(65) == -1
    assert lib.kp_set_tc_split(prev) == 1
