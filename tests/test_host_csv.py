"""Native CSV ingestion (libkp_host.so, include/kp_host.h).

dataset.load_matrix must equal build_matrix(load_records(path)) -- the
reference's composition (dataset.py:188-270) -- on every valid input, and
raise exactly the reference's DataError (type and line-numbered message) on
every invalid one. CPU only."""

import ctypes
import re
import shutil
from pathlib import Path

import numpy as np
import pytest

from paper_2003_06795_b200 import _host, dataset, pipeline, synthetic

ROOT = Path(__file__).resolve().parents[1]
HEADER = ",".join(dataset.CSV_COLUMNS)


def _python_path(path):
    return dataset.build_matrix(dataset.load_records(path))


def _same(a, b):
    assert a.problems == b.problems
    assert a.configs == b.configs
    assert a.values.dtype == b.values.dtype
    np.testing.assert_array_equal(a.values, b.values)


def test_header_declares_what_binding_expects():
    text = (ROOT / "include" / "kp_host.h").read_text()
    assert sorted(set(re.findall(r"\b(kp_[a-z0-9_]+)\s*\(", text))) == sorted(_host.EXPORTS)
    lib = _host.lib()
    for name in _host.EXPORTS:
        assert hasattr(lib, name)


@pytest.mark.parametrize("name", ["f32_nn", "f32_nt", "tf32_nn", "bf16_nt"])
def test_measured_sweeps_match_python_loader(name):
    path = pipeline.materialize(ROOT / "data" / f"b200_{name}_train.csv.gz")
    got, why = _host.load_matrix(path)
    assert got is not None, why          # the sweep files are inside the fast grammar
    _same(dataset.load_matrix(path), _python_path(path))


def test_reference_synthetic_dataset(tmp_path):
    """The reference's canonical generator output (write_records' repr reals)."""
    spec = synthetic.SyntheticSpec(synthetic.canonical_problems(40, 7), 7)
    path = tmp_path / "bench.csv"
    dataset.write_records(synthetic.generate(spec), path)
    assert _host.load_matrix(path)[0] is not None
    _same(dataset.load_matrix(path), _python_path(path))


ROWS = ["64,64,64,4,4,4,8,8,1000.0,524.288",
        "64,64,64,4,4,4,16,16,2000.0,262.144",
        "32,64,16,4,4,4,8,8,250.5,262.1",
        "32,64,16,4,4,4,16,16,125.25,524.2"]


def _write(tmp_path, text, name="t.csv"):
    p = tmp_path / name
    p.write_bytes(text.encode("utf-8") if isinstance(text, str) else text)
    return p


@pytest.mark.parametrize("text,fast", [
    (HEADER + "\n" + "\n".join(ROWS) + "\n", True),
    (HEADER + "\n" + "\n".join(ROWS), True),                              # no final newline
    (HEADER + "\r\n" + "\r\n".join(ROWS) + "\r\n", True),                 # CRLF
    (HEADER + "\n" + "\n".join(r.replace("1000.0", "1e3") for r in ROWS) + "\n", True),
    (HEADER + "\n" + "\n".join(r.replace("524.288", "+.524288E3") for r in ROWS) + "\n", True),
    (HEADER + "\n" + "\n".join(r.replace("64,64,64,", "0064,64,64,") for r in ROWS) + "\n", True),
    # valid for Python's int()/float()/csv but outside the fast grammar -> deferred
    (HEADER + "\n" + "\n".join(r.replace("1000.0", " 1000.0") for r in ROWS) + "\n", False),
    (HEADER + "\n" + "\n".join(r.replace("1000.0", "1_000.0") for r in ROWS) + "\n", False),
    (HEADER + "\n" + "\n".join(r.replace("1000.0", '"1000.0"') for r in ROWS) + "\n", False),
])
def test_valid_inputs_match(tmp_path, text, fast):
    p = _write(tmp_path, text)
    assert (_host.load_matrix(p)[0] is not None) == fast
    _same(dataset.load_matrix(p), _python_path(p))


@pytest.mark.parametrize("text", [
    "",                                                                   # empty file
    HEADER + "\n",                                                        # no rows
    "m,k,n,acc,row_tile,col_tile,wg_rows,wg_cols,runtime_ns\n" + ROWS[0] + "\n",
    "k,m,n,acc,row_tile,col_tile,wg_rows,wg_cols,runtime_ns,gflops\n" + ROWS[0] + "\n",
    "﻿" + HEADER + "\n" + ROWS[0] + "\n",                            # BOM
    HEADER + "\n" + ROWS[0] + ",\n",                                      # 11 fields
    HEADER + "\n" + ROWS[0] + "\n\n" + ROWS[1] + "\n",                    # blank line
    HEADER + "\n" + ROWS[0] + "\n\n",                                     # trailing blank line
    HEADER + "\n" + ROWS[0].replace("64,64,64", "64,6.4,64") + "\n",      # non-integer
    HEADER + "\n" + ROWS[0].replace("64,64,64", "64,0,64") + "\n",        # non-positive
    HEADER + "\n" + ROWS[0].replace("1000.0", "nan") + "\n",
    HEADER + "\n" + ROWS[0].replace("1000.0", "inf") + "\n",
    HEADER + "\n" + ROWS[0].replace("1000.0", "-1000.0") + "\n",
    HEADER + "\n" + ROWS[0].replace("524.288", "0") + "\n",
    HEADER + "\n" + ROWS[0].replace("524.288", "1e999") + "\n",           # overflows: inf
    HEADER + "\n" + ROWS[0].replace("4,4,4,8,8", "3,4,4,8,8") + "\n",     # bad tile
    HEADER + "\n" + ROWS[0].replace("4,4,4,8,8", "4,4,4,8,9") + "\n",     # bad work-group
    HEADER + "\n" + ROWS[0] + "\n" + ROWS[0] + "\n",                      # duplicate cell
    HEADER + "\n" + "\n".join(ROWS[:3]) + "\n",                           # hole
    HEADER + "\n" + ROWS[0] + "\n" + ROWS[1] + "\n" + ROWS[0] + "\n" + ROWS[2] + "\n",
])
def test_invalid_inputs_raise_the_reference_error(tmp_path, text):
    p = _write(tmp_path, text)
    got, why = _host.load_matrix(p)
    assert got is None and why[0] == _host.KP_CSV_DEFER
    with pytest.raises(dataset.DataError) as want:
        _python_path(p)
    with pytest.raises(type(want.value)) as have:
        dataset.load_matrix(p)
    assert str(have.value) == str(want.value)


def test_defer_reports_the_line(tmp_path):
    rows = list(ROWS)
    rows[2] = rows[2].replace("250.5", "x")
    p = _write(tmp_path, HEADER + "\n" + "\n".join(rows) + "\n")
    assert _host.load_matrix(p)[1] == (_host.KP_CSV_DEFER, 4)
    with pytest.raises(dataset.MalformedNumber, match="line 4"):
        dataset.load_matrix(p)


def test_missing_file_is_an_io_status(tmp_path):
    got, why = _host.load_matrix(tmp_path / "nope.csv")
    assert got is None and why[0] == _host.KP_CSV_IO
    with pytest.raises(FileNotFoundError):
        dataset.load_matrix(tmp_path / "nope.csv")


def test_free_is_idempotent():
    m = _host.KpCsvMatrix()
    _host.lib().kp_csv_free(ctypes.byref(m))
    _host.lib().kp_csv_free(ctypes.byref(m))
    _host.lib().kp_csv_free(None)


def test_pipeline_uses_native_loader(tmp_path):
    src = pipeline.materialize(ROOT / "data" / "b200_bf16_nn_train.csv.gz")
    dst = tmp_path / "x.csv"
    shutil.copy(src, dst)
    a = pipeline.load_matrix(dst)
    b = dataset.normalize(_python_path(dst))
    np.testing.assert_array_equal(a.values, b.values)
    assert a.problems == b.problems and a.configs == b.configs
