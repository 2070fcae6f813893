"""ctypes binding of libkp_host.so (include/kp_host.h): host-only native
helpers, usable without a GPU. Built in-tree on first use (g++, seconds)."""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

LIB_PATH = Path(os.environ.get("KP_HOST_LIB_PATH")
                or Path(__file__).resolve().parent / "libkp_host.so")

KP_CSV_OK, KP_CSV_DEFER, KP_CSV_IO = 0, 1, 2

# every symbol include/kp_host.h declares (checked by tests/test_host_csv.py)
EXPORTS = ("kp_csv_load_matrix", "kp_csv_free")


class KpCsvMatrix(ctypes.Structure):
    _fields_ = [("n_problems", ctypes.c_int64), ("n_configs", ctypes.c_int64),
                ("problems", ctypes.POINTER(ctypes.c_int64)),
                ("configs", ctypes.POINTER(ctypes.c_uint32)),
                ("gflops", ctypes.POINTER(ctypes.c_double))]


_lock = threading.Lock()
_lib = None


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if "KP_HOST_LIB_PATH" not in os.environ:
                from .build import build_host_library
                build_host_library()
            h = ctypes.CDLL(str(LIB_PATH))
            h.kp_csv_load_matrix.restype = ctypes.c_int32
            h.kp_csv_load_matrix.argtypes = [ctypes.c_char_p, ctypes.POINTER(KpCsvMatrix),
                                             ctypes.POINTER(ctypes.c_int64)]
            h.kp_csv_free.restype = None
            h.kp_csv_free.argtypes = [ctypes.POINTER(KpCsvMatrix)]
            _lib = h
        return _lib


def load_matrix(path):
    """(problems [P,3] int64, configs [C,5] int64, gflops [P,C] float64) or
    (None, bad_line) when the input leaves the fast grammar."""
    import numpy as np
    h = lib()
    m = KpCsvMatrix()
    bad = ctypes.c_int64(0)
    rc = h.kp_csv_load_matrix(os.fsencode(str(path)), ctypes.byref(m), ctypes.byref(bad))
    if rc != KP_CSV_OK:
        return None, (rc, bad.value)
    try:
        p, c = m.n_problems, m.n_configs
        probs = np.ctypeslib.as_array(m.problems, shape=(p, 3)).copy()
        cfgs = np.ctypeslib.as_array(m.configs, shape=(c, 5)).astype(np.int64)
        vals = np.ctypeslib.as_array(m.gflops, shape=(p, c)).copy()
    finally:
        h.kp_csv_free(ctypes.byref(m))
    return (probs, cfgs, vals), None
