"""ctypes binding of libkp.so (the C-ABI declared in include/kp_abi.h).

The library is built in-tree by ``paper_2003_06795_b200.build``; there is no
fallback: if it is missing or fails to load, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

from .errors import DataError

import os

LIB_PATH = Path(os.environ.get("KP_LIB_PATH") or Path(__file__).resolve().parent / "libkp.so")

F32_SIMT, TF32_TC, BF16_TC = 0, 1, 2
FAMILIES = {"f32": F32_SIMT, "tf32": TF32_TC, "bf16": BF16_TC}

KP_OK = 0
KP_ERR_INVALID_CONFIG = 1
KP_ERR_BAD_SHAPE = 2
KP_ERR_ALIGNMENT = 3
KP_ERR_UNSUPPORTED = 4
KP_ERR_CUDA = 5
KP_ERR_INVALID_ARG = 6

# every symbol include/kp_abi.h declares (checked by tests/test_abi.py)
EXPORTS = ("kp_abi_version", "kp_num_configs", "kp_config_at", "kp_config_valid",
           "kp_gemm", "kp_gemm_time", "kp_sweep_problem", "kp_select", "kp_gemm_auto",
           "kp_status_string", "kp_last_error", "kp_launch_count", "kp_device_info",
           "kp_fp32_peak", "kp_conv_output_shape", "kp_im2col", "kp_conv2d_auto",
           "kp_set_schedule", "kp_sweep_problem_ex", "kp_set_tc_split",
           "kp_gemm_skinny", "kp_set_skinny", "kp_auto_config", "kp_im2col_pitched",
           "kp_conv_workspace_elems", "kp_select_ex")


class KpConfig(ctypes.Structure):
    _fields_ = [("acc", ctypes.c_uint32), ("row_tile", ctypes.c_uint32),
                ("col_tile", ctypes.c_uint32), ("wg_rows", ctypes.c_uint32),
                ("wg_cols", ctypes.c_uint32)]

    def as_tuple(self):
        return (self.acc, self.row_tile, self.col_tile, self.wg_rows, self.wg_cols)


class KpGemmDesc(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int64), ("m", ctypes.c_int64), ("k", ctypes.c_int64),
                ("n", ctypes.c_int64), ("trans_a", ctypes.c_int32), ("trans_b", ctypes.c_int32),
                ("lda", ctypes.c_int64), ("ldb", ctypes.c_int64), ("ldc", ctypes.c_int64),
                ("stride_a", ctypes.c_int64), ("stride_b", ctypes.c_int64),
                ("stride_c", ctypes.c_int64), ("alpha", ctypes.c_float), ("beta", ctypes.c_float)]


class KpConvDesc(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int64) for f in ("batch", "c_in", "h", "w", "c_out", "kh", "kw",
                                              "stride_h", "stride_w", "pad_h", "pad_w")]


class KernelLibraryError(RuntimeError):
    """The native library is missing, failed to load, or a CUDA call failed."""


class InvalidKernelConfig(DataError):
    pass


class BadProblemShape(DataError):
    pass


class UnsupportedVariant(KernelLibraryError):
    pass


_lock = threading.Lock()
_lib = None


def _declare(lib):
    P = ctypes.POINTER
    c = ctypes
    sig = {
        "kp_abi_version": (c.c_int32, []),
        "kp_num_configs": (c.c_int32, [c.c_int]),
        "kp_config_at": (c.c_int, [c.c_int, c.c_int32, P(KpConfig)]),
        "kp_config_valid": (c.c_int, [c.c_int, KpConfig]),
        "kp_gemm": (c.c_int, [c.c_int, KpConfig, P(KpGemmDesc), c.c_void_p, c.c_void_p,
                              c.c_void_p, c.c_void_p]),
        "kp_gemm_time": (c.c_int, [c.c_int, KpConfig, P(KpGemmDesc), c.c_void_p, c.c_void_p,
                                   c.c_void_p, c.c_int32, c.c_int32, c.c_double,
                                   c.c_double, P(c.c_double), c.c_void_p]),
        "kp_sweep_problem": (c.c_int, [c.c_int, P(KpConfig), c.c_int32, P(KpGemmDesc),
                                       c.c_void_p, c.c_void_p, c.c_void_p, c.c_int32,
                                       c.c_int32, c.c_double, c.c_double, P(c.c_double),
                                       c.c_void_p]),
        "kp_sweep_problem_ex": (c.c_int, [c.c_int, P(KpConfig), c.c_int32, P(KpGemmDesc),
                                          c.c_void_p, c.c_void_p, c.c_void_p, c.c_int32,
                                          c.c_int32, c.c_double, c.c_double, c.c_int32,
                                          P(c.c_double), c.c_void_p]),
        "kp_select": (c.c_int, [c.c_int, c.c_int32, c.c_int32, c.c_int64, c.c_int64,
                                c.c_int64, P(KpConfig)]),
        "kp_gemm_auto": (c.c_int, [c.c_int, P(KpGemmDesc), c.c_void_p, c.c_void_p,
                                   c.c_void_p, c.c_void_p, P(KpConfig)]),
        "kp_status_string": (c.c_char_p, [c.c_int]),
        "kp_last_error": (c.c_char_p, []),
        "kp_launch_count": (c.c_int64, []),
        "kp_device_info": (c.c_int, [c.c_int32, P(c.c_int32), P(c.c_int32), P(c.c_int32)]),
        "kp_fp32_peak": (c.c_int, [P(c.c_double), c.c_void_p]),
        "kp_set_schedule": (c.c_int32, [c.c_int32]),
        "kp_set_tc_split": (c.c_int32, [c.c_int32]),
        "kp_set_skinny": (c.c_int32, [c.c_int32]),
        "kp_auto_config": (c.c_int, [c.c_int, c.c_int32, c.c_int32, c.c_int64, c.c_int64,
                                     c.c_int64, c.c_int64, P(KpConfig)]),
        "kp_select_ex": (c.c_int, [c.c_int, c.c_int32, c.c_int32, c.c_int64, c.c_int64,
                                   c.c_int64, c.c_int64, P(KpConfig)]),
        "kp_gemm_skinny": (c.c_int, [c.c_int, P(KpGemmDesc), c.c_void_p, c.c_void_p,
                                     c.c_void_p, c.c_void_p]),
        "kp_conv_output_shape": (c.c_int, [P(KpConvDesc), P(c.c_int64), P(c.c_int64)]),
        "kp_im2col": (c.c_int, [c.c_int, P(KpConvDesc), c.c_void_p, c.c_void_p, c.c_void_p]),
        "kp_im2col_pitched": (c.c_int, [c.c_int, P(KpConvDesc), c.c_void_p, c.c_void_p,
                                        c.c_int64, c.c_void_p]),
        "kp_conv_workspace_elems": (c.c_int, [c.c_int, P(KpConvDesc), P(c.c_int64)]),
        "kp_conv2d_auto": (c.c_int, [c.c_int, P(KpConvDesc), c.c_void_p, c.c_void_p, c.c_void_p,
                                     c.c_void_p, c.c_void_p, P(KpConfig)]),
    }
    partial = os.environ.get("KP_ABI_PARTIAL") == "1"  # A/B tooling against older builds
    for name, (res, args) in sig.items():
        if partial and not hasattr(lib, name):
            continue
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def lib():
    """The loaded library; raises KernelLibraryError (never falls back)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise KernelLibraryError(
                    f"{LIB_PATH} is missing: run `python -m paper_2003_06795_b200.build`")
            try:
                handle = ctypes.CDLL(str(LIB_PATH))
            except OSError as exc:
                raise KernelLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
            _declare(handle)
            _lib = handle
    return _lib


def check(status: int, what: str = "kp call") -> None:
    """Raise the Python exception matching a kp_status."""
    if status == KP_OK:
        return
    msg = lib().kp_last_error().decode(errors="replace")
    text = f"{what}: {lib().kp_status_string(status).decode()}: {msg}"
    if status == KP_ERR_INVALID_CONFIG:
        raise InvalidKernelConfig(text)
    if status in (KP_ERR_BAD_SHAPE, KP_ERR_ALIGNMENT, KP_ERR_INVALID_ARG):
        raise BadProblemShape(text)
    if status == KP_ERR_UNSUPPORTED:
        raise UnsupportedVariant(text)
    raise KernelLibraryError(text)


def family_id(family) -> int:
    if isinstance(family, int):
        return family
    try:
        return FAMILIES[family]
    except KeyError:
        raise ValueError(f"unknown kernel family {family!r}, expected one of {tuple(FAMILIES)}")


SKINNY = "skinny"  # the small-M path's config name (all-zero kp_config)


def to_kp_config(cfg) -> KpConfig:
    if isinstance(cfg, str):
        if cfg != SKINNY:
            raise ValueError(f"unknown config name {cfg!r}")
        return KpConfig(0, 0, 0, 0, 0)
    t = cfg.as_tuple() if hasattr(cfg, "as_tuple") else tuple(cfg)
    return KpConfig(*[int(v) for v in t])
