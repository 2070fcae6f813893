"""Pin the GEMM oracles themselves (test infrastructure): the sequential-fmaf
C restatement against an exact pure-Python evaluation on small cases and
against float64 numpy within the fp32 bound; the tf32/bf16 rounding helpers
against known bit patterns."""

import math

import numpy as np
import pytest

from oracle.gemm_oracle import (gemm_f32_exact, gemm_f64, round_bf16, round_tf32,
                                tolerance_bound)


def _fmaf(a, b, c):
    """Correctly rounded fp32 fma via exact float64 product (|a*b| < 2^53 ulps)."""
    return np.float32(math.fsum([float(a) * float(b), float(c)]))


def _python_gemm(a, b):
    m, k = a.shape
    n = b.shape[1]
    out = np.zeros((m, n), dtype=np.float32)
    for i in range(m):
        for j in range(n):
            acc = np.float32(0.0)
            for p in range(k):
                acc = _fmaf(a[i, p], b[p, j], acc)
            out[i, j] = acc
    return out


@pytest.mark.parametrize("shape", [(1, 1, 1), (3, 5, 2), (7, 9, 4)])
def test_fmaf_oracle_matches_python_loop(shape):
    m, k, n = shape
    rng = np.random.default_rng(m * 100 + k)
    a = rng.uniform(-1, 1, (m, k)).astype(np.float32)
    b = rng.uniform(-1, 1, (k, n)).astype(np.float32)
    got = gemm_f32_exact(a, b, m=m, k=k, n=n).reshape(m, n)
    np.testing.assert_array_equal(got, _python_gemm(a, b))


def test_fmaf_oracle_layouts_and_epilogue():
    rng = np.random.default_rng(3)
    m, k, n = 6, 5, 7
    a = rng.uniform(-1, 1, (m, k)).astype(np.float32)
    b = rng.uniform(-1, 1, (k, n)).astype(np.float32)
    base = gemm_f32_exact(a, b, m=m, k=k, n=n)
    for ta in (False, True):
        for tb in (False, True):
            sa = a.T.copy() if ta else a
            sb = b.T.copy() if tb else b
            got = gemm_f32_exact(sa, sb, m=m, k=k, n=n, trans_a=ta, trans_b=tb)
            np.testing.assert_array_equal(got, base)
    c0 = rng.uniform(-1, 1, (m, n)).astype(np.float32)
    got = gemm_f32_exact(a, b, m=m, k=k, n=n, alpha=2.0, beta=0.5, c_init=c0).reshape(m, n)
    want = np.array([[np.float32(math.fsum([0.5 * float(c0[i, j]),
                                            float(np.float32(2.0 * base.reshape(m, n)[i, j]))]))
                      for j in range(n)] for i in range(m)], dtype=np.float32)
    np.testing.assert_array_equal(got, want)


def test_fmaf_oracle_within_fp32_bound_of_f64():
    rng = np.random.default_rng(4)
    a = rng.uniform(-1, 1, (64, 300)).astype(np.float32)
    b = rng.uniform(-1, 1, (300, 48)).astype(np.float32)
    got = gemm_f32_exact(a, b, m=64, k=300, n=48).reshape(64, 48)
    ref = gemm_f64(a, b)
    assert (np.abs(got - ref) <= tolerance_bound(a, b, "f32")).all()
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-6


def test_rounding_helpers():
    x = np.array([1.0, 1.0 + 2 ** -11, 1.0 + 2 ** -10 + 2 ** -11, 3.14159265], dtype=np.float32)
    t = round_tf32(x)
    assert t[0] == 1.0
    assert t[1] == 1.0                      # tie -> even
    assert t[2] == np.float32(1.0 + 2 ** -9)  # tie -> even (up)
    assert (t.view(np.uint32) & 0x1FFF == 0).all()
    bf = round_bf16(x)
    assert (bf.view(np.uint32) & 0xFFFF == 0).all()
    assert abs(float(bf[3]) - 3.14159265) < 2 ** -7 * 4
