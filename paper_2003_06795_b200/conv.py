"""Convolution layers through the runtime-selected GEMM library (im2col).

SURVEY §8(f) item 2: the reference scopes GEMM-size extraction out
(SPEC.md:13); here the network-derived shapes of `shapes.py` are produced by
real convolution layers and executed end to end: an im2col gather kernel
(kp_im2col) followed by the NT GEMM chosen by the compiled decision tree
(kp_gemm_auto), i.e. exactly the (m, k, n) = (B*Ho*Wo, Cin*kh*kw, Cout)
problems the selectors were trained on.
"""

from __future__ import annotations

import ctypes

from . import _native as nat
from .gemm import _family_dtype, _stream_handle, _torch, check_device


def _desc(x, w, stride, padding) -> nat.KpConvDesc:
    b, c_in, h, wd = x.shape
    c_out, c_in2, kh, kw = w.shape
    if c_in != c_in2:
        raise nat.BadProblemShape(f"input has {c_in} channels, weights expect {c_in2}")
    sh, sw = (stride, stride) if isinstance(stride, int) else stride
    ph, pw = (padding, padding) if isinstance(padding, int) else padding
    return nat.KpConvDesc(b, c_in, h, wd, c_out, kh, kw, sh, sw, ph, pw)


def output_shape(x_shape, w_shape, stride=1, padding=0) -> tuple[int, int]:
    lib = nat.lib()
    d = nat.KpConvDesc(x_shape[0], x_shape[1], x_shape[2], x_shape[3], w_shape[0], w_shape[2],
                       w_shape[3], *((stride, stride) if isinstance(stride, int) else stride),
                       *((padding, padding) if isinstance(padding, int) else padding))
    ho, wo = ctypes.c_int64(), ctypes.c_int64()
    nat.check(lib.kp_conv_output_shape(ctypes.byref(d), ctypes.byref(ho), ctypes.byref(wo)),
              "kp_conv_output_shape")
    return ho.value, wo.value


def im2col(x, kh: int, kw: int, stride=1, padding=0, family="f32"):
    """cols [B*Ho*Wo, Cin*kh*kw] of an NCHW CUDA tensor (zero padding)."""
    torch = _torch()
    fam = nat.family_id(family)
    if x.dtype != _family_dtype(fam):
        raise nat.BadProblemShape(f"family {family!r} expects {_family_dtype(fam)} input")
    check_device(x)
    w_shape = (1, x.shape[1], kh, kw)
    ho, wo = output_shape(x.shape, w_shape, stride, padding)
    x = x.contiguous()
    cols = torch.empty((x.shape[0] * ho * wo, x.shape[1] * kh * kw), dtype=x.dtype,
                       device=x.device)
    d = nat.KpConvDesc(x.shape[0], x.shape[1], x.shape[2], x.shape[3], 1, kh, kw,
                       *((stride, stride) if isinstance(stride, int) else stride),
                       *((padding, padding) if isinstance(padding, int) else padding))
    with torch.cuda.device(x.device):
        nat.check(nat.lib().kp_im2col(fam, ctypes.byref(d), x.data_ptr(), cols.data_ptr(),
                                      _stream_handle(x.device)), "kp_im2col")
    return cols


def conv2d(x, w, stride=1, padding=0, *, family="f32", nhwc: bool = False, workspace=None):
    """y = conv2d(x, w) with x NCHW, w [Cout, Cin, kh, kw]; returns NCHW (or
    the GEMM's native NHWC view when nhwc=True). Runs kp_conv2d_auto: the
    im2col gather, then the selector-chosen NT GEMM kernel."""
    torch = _torch()
    fam = nat.family_id(family)
    want = _family_dtype(fam)
    if x.dtype != want or w.dtype != want:
        raise nat.BadProblemShape(f"family {family!r} expects {want} tensors")
    check_device(x, w, workspace)
    d = _desc(x, w, stride, padding)
    ho, wo = output_shape(x.shape, w.shape, stride, padding)
    k = d.c_in * d.kh * d.kw
    x = x.contiguous()
    wmat = w.reshape(d.c_out, k).contiguous()
    need = ctypes.c_int64()
    nat.check(nat.lib().kp_conv_workspace_elems(fam, ctypes.byref(d), ctypes.byref(need)),
              "kp_conv_workspace_elems")
    if workspace is None or workspace.numel() < need.value or workspace.dtype != want:
        workspace = torch.empty(need.value, dtype=want, device=x.device)
    y = torch.empty((d.batch, ho, wo, d.c_out), dtype=torch.float32, device=x.device)
    chosen = nat.KpConfig()
    with torch.cuda.device(x.device):
        nat.check(nat.lib().kp_conv2d_auto(fam, ctypes.byref(d), x.data_ptr(), wmat.data_ptr(),
                                           y.data_ptr(), workspace.data_ptr(),
                                           _stream_handle(x.device), ctypes.byref(chosen)),
                  "kp_conv2d_auto")
    return y if nhwc else y.permute(0, 3, 1, 2)
