"""TEST INFRASTRUCTURE ONLY -- CPU oracles for the GEMM kernel families.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this module; the product path never does.

* ``gemm_f32_exact``: ctypes binding of oracle/gemm_ref.c, the
  sequential-k fmaf restatement that K1 (FP32 SIMT) must match bit for bit.
* ``gemm_f64``: numpy float64 matmul of the same (pre-rounded) inputs, the
  reference value for the tcgen05 TF32/BF16 families, with
  ``tolerance_bound`` giving the elementwise error bound c*K*u*(|A||B|)_ij.

Provenance: the reference ships no GEMM (the kernels live in the
un-vendored SYCL-DNN, no pinned version), so GEMM parity is
"unpinned" at the reference boundary and anchored on these restatements of
C = alpha*op(A)@op(B) + beta*C with the reference's row-major m x k / k x n
shapes (dataset.py:89-100) and 2mnk FLOP convention (synthetic.py:110-113).
"""

from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle_gemm.so"
_lib = None

# unit roundoff per input format
UNIT_ROUNDOFF = {"f32": 2.0 ** -24, "tf32": 2.0 ** -11, "bf16": 2.0 ** -8}


def _load():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            import sys
            sys.path.insert(0, str(HERE.parent))
            from paper_2003_06795_b200.build import build_oracle
            build_oracle()
        lib = ctypes.CDLL(str(LIB_PATH))
        i64, i32, f32 = ctypes.c_int64, ctypes.c_int32, ctypes.c_float
        vp = ctypes.c_void_p
        lib.kp_oracle_gemm_f32.restype = ctypes.c_int
        lib.kp_oracle_gemm_f32.argtypes = [i64, i64, i64, i64, i32, i32, i64, i64, i64,
                                           i64, i64, i64, f32, f32, vp, vp, vp]
        lib.kp_oracle_set_threads.restype = ctypes.c_int
        lib.kp_oracle_set_threads.argtypes = [ctypes.c_int]
        _lib = lib
    return _lib


def gemm_f32_exact(a_store: np.ndarray, b_store: np.ndarray, *, m: int, k: int, n: int,
                   trans_a: bool = False, trans_b: bool = False, batch: int = 1,
                   lda: int | None = None, ldb: int | None = None, ldc: int | None = None,
                   stride_a: int = 0, stride_b: int = 0, stride_c: int | None = None,
                   alpha: float = 1.0, beta: float = 0.0, c_init: np.ndarray | None = None):
    """Sequential-fmaf GEMM over raw float32 storage (same args as kp_gemm)."""
    lda = lda if lda is not None else (m if trans_a else k)
    ldb = ldb if ldb is not None else (k if trans_b else n)
    ldc = ldc if ldc is not None else n
    stride_c = stride_c if stride_c is not None else m * ldc
    a = np.ascontiguousarray(a_store, dtype=np.float32)
    b = np.ascontiguousarray(b_store, dtype=np.float32)
    size_c = (batch - 1) * stride_c + (m - 1) * ldc + n
    c = (np.zeros(size_c, dtype=np.float32) if c_init is None
         else np.ascontiguousarray(c_init, dtype=np.float32).reshape(-1).copy())
    rc = _load().kp_oracle_gemm_f32(batch, m, k, n, int(trans_a), int(trans_b), lda, ldb, ldc,
                                    stride_a, stride_b, stride_c, alpha, beta,
                                    a.ctypes.data, b.ctypes.data, c.ctypes.data)
    if rc != 0:
        raise ValueError(f"oracle rejected the problem (rc={rc})")
    return c


def set_threads(n: int) -> int:
    """Host threads (OpenMP) the fmaf oracle uses; returns the previous count."""
    return int(_load().kp_oracle_set_threads(int(n)))


def gemm_f64(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """float64 reference of logical op(A) @ op(B) (inputs already rounded)."""
    return np.matmul(np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64))


def tolerance_bound(a: np.ndarray, b: np.ndarray, fmt: str, c: float = 2.0) -> np.ndarray:
    """Elementwise bound c*K*u*(|A||B|)_ij, u the input format's roundoff."""
    k = a.shape[-1]
    return c * k * UNIT_ROUNDOFF[fmt] * np.matmul(np.abs(a).astype(np.float64),
                                                  np.abs(b).astype(np.float64))


def round_tf32(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> tf32 (10 explicit mantissa bits)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> 13) & 1
    u = (u + 0xFFF + lsb) & 0xFFFFE000
    return u.astype(np.uint32).view(np.float32)


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bfloat16 value (kept as float32)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = (u + 0x7FFF + lsb) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)
