"""CPU-side checks of the C ABI boundary: the library builds, loads and exports every
function include/vfmm.h declares; host-only entry points behave (no GPU needed)."""
import ctypes
import os
import re

import pytest

import paper_1110_2921_b200 as vf


def _declared():
    src = open(vf.HEADER_PATH).read()
    return sorted(set(re.findall(r"\b(vfmm_[a-z_]+)\s*\(", src)))


def test_header_declares_the_documented_entry_points():
    names = _declared()
    for f in vf.EXPORTS:
        assert f in names


def test_library_exports_every_declared_symbol():
    L = vf.load_library()
    for name in _declared():
        assert hasattr(L, name), name


def test_host_only_functions():
    L = vf.load_library()
    assert L.vfmm_abi_version() == 2
    assert ctypes.sizeof(vf.c_stats) == 10 * 8 + 4 * 8 + 2 * 4 + 2 * 8 + 2 * 8
    p = vf.c_params()
    L.vfmm_params_default(ctypes.byref(p))
    assert p.p == 10 and p.image_levels == 3 and p.depth == 0
    assert abs(p.box_len - 6.2831855) < 1e-6 and abs(p.box_lo + 3.1415927) < 1e-6
    assert L.vfmm_strerror(-2).decode().startswith("VFMM_EDOMAIN")
    assert L.vfmm_strerror(0).decode() == "VFMM_OK"


def test_create_rejects_bad_params_without_touching_the_gpu():
    L = vf.load_library()
    ctx = ctypes.c_void_p()
    for bad in (dict(p=0), dict(p=17), dict(sigma=0.0), dict(sigma=float("nan")),
                dict(depth=11), dict(depth=-2), dict(image_levels=7), dict(scheme=2), dict(mode=9),
                dict(mode=5), dict(mode=-1),
                dict(box_len=-1.0)):
        prm = vf.Params(**bad).to_c()
        assert L.vfmm_create(ctypes.byref(ctx), ctypes.byref(prm), 0) == vf.VFMM_EINVAL
        assert not ctx.value


def test_tree_entry_rejects_a_null_context_without_touching_the_gpu():
    """vfmm_evaluate_tree (NEXT-4) validates its arguments before any CUDA call."""
    L = vf.load_library()
    L.vfmm_evaluate_tree.argtypes = [ctypes.c_void_p, ctypes.c_int64] + [ctypes.c_void_p] * 4 + [
        ctypes.c_float, ctypes.c_int32, ctypes.c_void_p]
    L.vfmm_evaluate_tree.restype = ctypes.c_int
    buf = (ctypes.c_float * 6)()
    a = ctypes.cast(buf, ctypes.c_void_p)
    assert L.vfmm_evaluate_tree(None, 1, a, a, a, a, 0.5, 64, None) == vf.VFMM_EINVAL
    assert vf.MODE_HYBRID == 4


def test_no_oracle_in_product_path():
    """The product package must not import or link the oracle."""
    pkg = os.path.dirname(vf.__file__)
    for root, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cpp", ".h")):
                txt = open(os.path.join(root, fn)).read()
                assert "import oracle" not in txt and "liboracle" not in txt, fn
                assert "from oracle" not in txt, fn


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: without libvfmm.so the binding raises instead of computing."""
    import importlib

    mod = importlib.reload(vf)
    try:
        mod._LIB = None
        with pytest.raises(OSError):
            mod.load_library(str(tmp_path / "missing.so"))
    finally:
        importlib.reload(vf)


def test_partition_helper_without_gpu():
    lo, hi = vf.partition(6, 8, 7)
    assert hi == 1 << 18 and lo == 7 * (1 << 15)
