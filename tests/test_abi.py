"""The C-ABI library (libkp.so) loads without a GPU and exports every symbol
include/kp_abi.h declares; config enumeration and argument validation work
host-side (no compute call is made here)."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_2003_06795_b200 import _native as nat
from paper_2003_06795_b200 import dataset

HEADER = Path(__file__).resolve().parents[1] / "include" / "kp_abi.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(kp_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_what_binding_expects():
    assert sorted(nat.EXPORTS) == declared_symbols()


def test_library_exports_every_declared_symbol():
    lib = nat.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.kp_abi_version() == 1


def test_config_space_matches_reference_order():
    lib = nat.lib()
    assert lib.kp_num_configs(nat.F32_SIMT) == 640
    cfg = nat.KpConfig()
    for i, want in enumerate(dataset.all_configs()):
        assert lib.kp_config_at(nat.F32_SIMT, i, ctypes.byref(cfg)) == nat.KP_OK
        assert cfg.as_tuple() == want.as_tuple()
    assert lib.kp_config_at(nat.F32_SIMT, 640, ctypes.byref(cfg)) == nat.KP_ERR_INVALID_ARG


@pytest.mark.parametrize("bad", [(3, 4, 4, 8, 8), (4, 16, 4, 8, 8), (4, 4, 4, 4, 4),
                                 (0, 1, 1, 1, 64)])
def test_invalid_config_status(bad):
    lib = nat.lib()
    assert lib.kp_config_valid(nat.F32_SIMT, nat.KpConfig(*bad)) == nat.KP_ERR_INVALID_CONFIG
    assert b"domain" in lib.kp_last_error()


def _desc(**kw):
    d = dict(batch=1, m=4, k=4, n=4, trans_a=0, trans_b=0, lda=4, ldb=4, ldc=4, stride_a=0,
             stride_b=0, stride_c=16, alpha=1.0, beta=0.0)
    d.update(kw)
    return nat.KpGemmDesc(**d)


@pytest.mark.parametrize("kw,status", [
    (dict(m=0), nat.KP_ERR_BAD_SHAPE), (dict(k=-1), nat.KP_ERR_BAD_SHAPE),
    (dict(lda=3), nat.KP_ERR_BAD_SHAPE), (dict(ldb=2), nat.KP_ERR_BAD_SHAPE),
    (dict(ldc=1), nat.KP_ERR_BAD_SHAPE), (dict(batch=2, stride_c=3), nat.KP_ERR_BAD_SHAPE),
])
def test_shape_validation_before_any_launch(kw, status):
    lib = nat.lib()
    d = _desc(**kw)
    buf = ctypes.c_void_p(16)  # never dereferenced: validation fails first
    rc = lib.kp_gemm(nat.F32_SIMT, nat.KpConfig(4, 4, 4, 8, 8), ctypes.byref(d), buf, buf, buf, None)
    assert rc == status
    with pytest.raises(dataset.DataError):
        nat.check(rc, "kp_gemm")


def test_null_pointers_rejected():
    lib = nat.lib()
    d = _desc()
    assert lib.kp_gemm(nat.F32_SIMT, nat.KpConfig(4, 4, 4, 8, 8), ctypes.byref(d), None, None,
                       None, None) == nat.KP_ERR_INVALID_ARG


def test_selector_table_consistent():
    """kp_select answers from the compiled generated headers, or reports
    UNSUPPORTED for variants without one; answers are valid configs."""
    from paper_2003_06795_b200 import libgen
    lib = nat.lib()
    installed = set(libgen.installed())
    cfg = nat.KpConfig()
    for fam, fid in nat.FAMILIES.items():
        for trans in libgen.TRANS:
            rc = lib.kp_select(fid, int(trans[0] == "t"), int(trans[1] == "t"), 256, 256, 256,
                               ctypes.byref(cfg))
            if (fam, trans) in installed:
                assert rc == nat.KP_OK
                assert lib.kp_config_valid(fid, cfg) == nat.KP_OK
            else:
                assert rc == nat.KP_ERR_UNSUPPORTED


def test_status_strings():
    lib = nat.lib()
    for st in range(7):
        assert lib.kp_status_string(st)


LEAN = Path(__file__).resolve().parents[1] / "paper_2003_06795_b200" / "libkp_lean.so"


@pytest.mark.skipif(not LEAN.exists(), reason="lean library not built (build --lean)")
def test_lean_library_only_has_selected_kernels():
    """The paper's deployment build: only selector-reachable FP32 kernels are
    compiled; any other config is rejected before a launch."""
    import json
    lib = ctypes.CDLL(str(LEAN))
    nat._declare(lib)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    sel = json.loads((Path(__file__).resolve().parents[1] / "selectors" / "f32_nn" /
                      "selection.json").read_text())
    chosen = {(c["acc"], c["row_tile"], c["col_tile"]) for c in sel["configs"]}
    missing = next(c for c in dataset.all_configs() if c.as_tuple()[:3] not in chosen)
    d = _desc(m=8, k=8, n=8, lda=8, ldb=8, ldc=8, stride_c=64)
    buf = ctypes.c_void_p(16)
    rc = lib.kp_gemm(nat.F32_SIMT, nat.KpConfig(*missing.as_tuple()), ctypes.byref(d), buf, buf,
                     buf, None)
    assert rc == nat.KP_ERR_UNSUPPORTED
    assert b"lean" in lib.kp_last_error()
    assert LEAN.stat().st_size < nat.LIB_PATH.stat().st_size


def test_batched_selector_dispatch():
    """kp_select_ex: batch 1 answers from the plain tree; batch > 1 from the
    strided-batched tree of the same (family, layout) when one is compiled in
    (selector variant <layout>_b<N>), else from the plain tree."""
    from paper_2003_06795_b200 import codegen, libgen, selector_models
    root = Path(__file__).resolve().parents[1]
    lib = nat.lib()
    cfg = nat.KpConfig()
    batched = {(f, t[:2]): libgen.variant_batch(t) for f, t in libgen.installed() if "_b" in t}
    for fam, fid in nat.FAMILIES.items():
        plain = codegen.export_tree(selector_models.load_model(
            root / "selectors" / f"{fam}_nn" / "model.json"))
        for (m, k, n) in [(784, 576, 64), (3136, 1152, 128), (49, 4608, 512)]:
            assert lib.kp_select_ex(fid, 0, 0, 1, m, k, n, ctypes.byref(cfg)) == nat.KP_OK
            assert cfg.as_tuple() == codegen.traverse_document(plain, m, k, n).as_tuple()
            assert lib.kp_select_ex(fid, 0, 0, 8, m, k, n, ctypes.byref(cfg)) == nat.KP_OK
            if (fam, "nn") in batched:
                bt = codegen.export_tree(selector_models.load_model(
                    root / "selectors" / f"{fam}_nn_b{batched[(fam, 'nn')]}" / "model.json"))
                assert cfg.as_tuple() == codegen.traverse_document(bt, m, k, n).as_tuple()
            else:
                assert cfg.as_tuple() == codegen.traverse_document(plain, m, k, n).as_tuple()
    assert lib.kp_select_ex(0, 0, 0, 0, 8, 8, 8, ctypes.byref(cfg)) == nat.KP_ERR_BAD_SHAPE


def test_selector_variant_names_and_table():
    """Variant keys: layout, optionally _b<batch> (one selector per (family,
    trans, batch)); the generated table lists each with its batch."""
    from paper_2003_06795_b200 import libgen
    from paper_2003_06795_b200.errors import DataError
    assert libgen.variant_batch("nn") == 1
    assert libgen.variant_batch("tt") == 1
    assert libgen.variant_batch("nn_b8") == 8
    for bad in ("xx", "nn_b", "nn_8", "nnb8"):
        with pytest.raises(DataError):
            libgen.variant_batch(bad)
    table = (libgen.GEN_DIR / "selectors.h").read_text()
    for fam, trans in libgen.installed():
        sym = libgen.symbol_for(fam, trans)
        ta = "true" if trans[0] == "t" else "false"
        tb = "true" if trans[1] == "t" else "false"
        row = (f"{{{libgen.FAMILY_IDS[fam]}, {ta}, {tb}, {libgen.variant_batch(trans)}, "
               f"kp_wrap_{sym}, \"{sym}.h\"}},")
        assert row in table, row


def test_skinny_config_is_not_a_kernel_config():
    """The all-zero config names the small-M path in kp_gemm / kp_gemm_time /
    sweeps, but kp_config_valid (the reference's KernelConfig validation)
    still rejects it."""
    lib = nat.lib()
    zero = nat.to_kp_config(nat.SKINNY)
    assert zero.as_tuple() == (0, 0, 0, 0, 0)
    for fam in (nat.F32_SIMT, nat.TF32_TC, nat.BF16_TC):
        assert lib.kp_config_valid(fam, zero) == nat.KP_ERR_INVALID_CONFIG
    with pytest.raises(ValueError):
        nat.to_kp_config("fast")
