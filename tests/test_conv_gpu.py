"""im2col front-end on the B200: conv layers through the runtime-selected NT
GEMM. FP32 is bit-exact against the CPU restatement (numpy im2col + the
sequential-fmaf oracle, accumulation order k = c*kh*kw + r*kw + s); the
tensor-core families within the K-scaled bound of the float64 reference."""

import numpy as np
import pytest

from oracle.gemm_oracle import gemm_f32_exact

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _np_im2col(x, kh, kw, stride, pad):
    b, c, h, w = x.shape
    ho = (h + 2 * pad - kh) // stride + 1
    wo = (w + 2 * pad - kw) // stride + 1
    xp = np.zeros((b, c, h + 2 * pad, w + 2 * pad), dtype=x.dtype)
    xp[:, :, pad:pad + h, pad:pad + w] = x
    cols = np.empty((b, ho, wo, c, kh, kw), dtype=x.dtype)
    for r in range(kh):
        for s in range(kw):
            cols[:, :, :, :, r, s] = xp[:, :, r:r + stride * ho:stride,
                                        s:s + stride * wo:stride].transpose(0, 2, 3, 1)
    return cols.reshape(b * ho * wo, c * kh * kw), ho, wo


@pytest.mark.parametrize("case", [
    dict(b=2, c=3, h=17, w=15, co=8, k=3, s=1, p=1),     # VGG conv1-like, K = 27
    dict(b=1, c=16, h=14, w=14, co=32, k=1, s=1, p=0),   # pointwise
    dict(b=2, c=4, h=23, w=19, co=12, k=7, s=2, p=3),    # ResNet stem-like
])
def test_conv2d_f32_bit_exact(case):
    from paper_2003_06795_b200 import conv
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, (case["b"], case["c"], case["h"], case["w"])).astype(np.float32)
    wt = rng.uniform(-1, 1, (case["co"], case["c"], case["k"], case["k"])).astype(np.float32)
    got = conv.conv2d(torch.from_numpy(x).cuda(), torch.from_numpy(wt).cuda(), case["s"],
                      case["p"], nhwc=True).cpu().numpy()
    cols, ho, wo = _np_im2col(x, case["k"], case["k"], case["s"], case["p"])
    m, k = cols.shape
    want = gemm_f32_exact(cols, wt.reshape(case["co"], k), m=m, k=k, n=case["co"],
                          trans_b=True).reshape(case["b"], ho, wo, case["co"])
    np.testing.assert_array_equal(got, want)
    ref = torch.nn.functional.conv2d(torch.from_numpy(x).double(), torch.from_numpy(wt).double(),
                                     stride=case["s"], padding=case["p"]).numpy()
    np.testing.assert_allclose(got.transpose(0, 3, 1, 2), ref, rtol=1e-4, atol=1e-5)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("shape", [
    (2, 5, 9, 11, 3, 2, 2, 1),      # K = 30: scalar gather
    (2, 8, 33, 31, 3, 3, 1, 1),     # K = 72: 16-byte vector stores (both dtypes)
    (3, 4, 64, 64, 1, 1, 1, 0),     # K = 4: f32 vectors, bf16 scalar
    (1, 3, 50, 50, 7, 7, 2, 3),     # stem-like, K = 147
])
def test_im2col_matches_numpy(shape, dtype):
    from paper_2003_06795_b200 import conv
    b, c, h, w, kh, kw, st, pad = shape
    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, (b, c, h, w)).astype(np.float32)
    xt = torch.from_numpy(x).cuda()
    if dtype == "bf16":
        xt = xt.to(torch.bfloat16)
        x = xt.float().cpu().numpy()
    got = conv.im2col(xt, kh, kw, stride=st, padding=pad,
                      family=dtype).float().cpu().numpy()
    xp = np.zeros((b, c, h + 2 * pad, w + 2 * pad), dtype=np.float32)
    xp[:, :, pad:pad + h, pad:pad + w] = x
    ho, wo = (h + 2 * pad - kh) // st + 1, (w + 2 * pad - kw) // st + 1
    want = np.empty((b, ho, wo, c, kh, kw), dtype=np.float32)
    for r in range(kh):
        for s in range(kw):
            want[..., r, s] = xp[:, :, r:r + st * ho:st, s:s + st * wo:st].transpose(0, 2, 3, 1)
    np.testing.assert_array_equal(got, want.reshape(b * ho * wo, c * kh * kw))


@pytest.mark.parametrize("family", ["tf32", "bf16"])
def test_conv2d_tensor_core(family):
    from paper_2003_06795_b200 import conv
    rng = np.random.default_rng(2)
    dt = torch.bfloat16 if family == "bf16" else torch.float32
    x = torch.from_numpy(rng.uniform(-1, 1, (2, 16, 12, 12)).astype(np.float32)).cuda().to(dt)
    wt = torch.from_numpy(rng.uniform(-1, 1, (64, 16, 3, 3)).astype(np.float32)).cuda().to(dt)
    got = conv.conv2d(x, wt, 1, 1, family=family).double().cpu()
    ref = torch.nn.functional.conv2d(x.double().cpu(), wt.double().cpu(), stride=1, padding=1)
    u = 2.0 ** -10 if family == "tf32" else 2.0 ** -8
    bound = 2.0 * 144 * u * torch.nn.functional.conv2d(x.double().cpu().abs(),
                                                       wt.double().cpu().abs(), padding=1)
    assert bool(((got - ref).abs() <= bound + 1e-30).all())


@pytest.mark.parametrize("family", ["tf32", "bf16"])
@pytest.mark.parametrize("layer", [(2, 3, 32, 32, 64, 3, 3, 1, 1),     # VGG conv1_1: K = 27
                                   (2, 3, 64, 64, 64, 7, 7, 2, 3)])    # ResNet conv1: K = 147
def test_conv2d_tensor_core_unaligned_k(family, layer):
    """First layers whose K = Cin*kh*kw is not a 16-byte multiple: the im2col
    rows get a padded pitch (zero columns) and the weights are staged."""
    from paper_2003_06795_b200 import _native as nat, conv
    import ctypes
    b, c, h, w, co, kh, kw, st, pad = layer
    rng = np.random.default_rng(5)
    dt = torch.bfloat16 if family == "bf16" else torch.float32
    x = torch.from_numpy(rng.uniform(-1, 1, (b, c, h, w)).astype(np.float32)).cuda().to(dt)
    wt = torch.from_numpy(rng.uniform(-1, 1, (co, c, kh, kw)).astype(np.float32)).cuda().to(dt)
    got = conv.conv2d(x, wt, st, pad, family=family).double().cpu()
    ref = torch.nn.functional.conv2d(x.double().cpu(), wt.double().cpu(), stride=st, padding=pad)
    u = 2.0 ** -10 if family == "tf32" else 2.0 ** -8
    k = c * kh * kw
    bound = 2.0 * k * u * torch.nn.functional.conv2d(x.double().cpu().abs(),
                                                     wt.double().cpu().abs(), stride=st,
                                                     padding=pad)
    assert bool(((got - ref).abs() <= bound + 1e-30).all())
    # the workspace query reports the padded pitch
    d = conv._desc(x, wt, st, pad)
    need = ctypes.c_int64()
    nat.check(nat.lib().kp_conv_workspace_elems(nat.family_id(family), ctypes.byref(d),
                                                ctypes.byref(need)))
    al = 4 if family == "tf32" else 8
    ho, wo = conv.output_shape(x.shape, wt.shape, st, pad)
    assert need.value == b * ho * wo * (-(-k // al) * al)
