"""The C-ABI boundary on CPU: the library loads, exports every symbol include/pflu.h declares, and
validates arguments (LAPACK-style negative codes) before touching the device."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "pflu.h")).read()
    return sorted(set(re.findall(r"\b(pflu_[a-z_0-9]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    from paper_1804_07017_b200 import _lib

    L = _lib.load()
    syms = _header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), f"{s} declared in pflu.h but not exported"
    assert sorted(_lib.EXPORTS) == syms


def test_header_is_plain_c():
    txt = open(os.path.join(ROOT, "include", "pflu.h")).read()
    assert 'extern "C"' in txt and "torch" not in txt.lower().replace("no torch types", "")
    for s in _header_symbols():
        assert s in txt


def test_built_for_sm100a():
    out = os.popen(f"cuobjdump --list-elf {ROOT}/paper_1804_07017_b200/libpflu.so 2>&1").read()
    assert "sm_100a" in out


def test_argument_validation_codes_without_gpu():
    from paper_1804_07017_b200 import _lib

    L = _lib.load()
    a = np.zeros((4, 8))
    piv = np.zeros(8, dtype=np.int64)
    info = ctypes.c_int64(0)
    # m < n -> -3 (n invalid), lda < n -> -4, b < 1 -> -5, lookahead 2 -> -6, null ipiv -> -7
    assert L.pflu_getrf(a.ctypes.data, 4, 8, 8, 2, 1, piv.ctypes.data, ctypes.byref(info), None) == -3
    b = np.zeros((8, 8))
    assert L.pflu_getrf(b.ctypes.data, 8, 8, 4, 2, 1, piv.ctypes.data, ctypes.byref(info), None) == -4
    assert L.pflu_getrf(b.ctypes.data, 8, 8, 8, 0, 1, piv.ctypes.data, ctypes.byref(info), None) == -5
    assert L.pflu_getrf(b.ctypes.data, 8, 8, 8, 2, 2, piv.ctypes.data, ctypes.byref(info), None) == -6
    assert L.pflu_getrf(b.ctypes.data, 8, 8, 8, 2, 1, None, ctypes.byref(info), None) == -7
    assert L.pflu_getrf(None, 8, 8, 8, 2, 1, piv.ctypes.data, ctypes.byref(info), None) == -1
    assert L.pflu_gemm_update(None, 1, None, 1, None, 1, 1, 1, 1, 0, None) == -1
    assert L.pflu_laswp(b.ctypes.data, 8, 5, 3, piv.ctypes.data, 0, 1, None) == -4
    tau = np.zeros(8)
    assert L.pflu_geqrf(a.ctypes.data, 4, 8, 8, 2, 1, tau.ctypes.data) == -3
    assert L.pflu_geqrf(b.ctypes.data, 8, 8, 4, 2, 1, tau.ctypes.data) == -4
    assert L.pflu_geqrf(b.ctypes.data, 8, 8, 8, 0, 1, tau.ctypes.data) == -5
    assert L.pflu_geqrf(b.ctypes.data, 8, 8, 8, 2, 2, tau.ctypes.data) == -6
    assert L.pflu_geqrf(b.ctypes.data, 8, 8, 8, 2, 1, None) == -7
    assert L.pflu_geqrf_device(None, 8, 8, 8, 2, 1, None, None, None, 0, None) == -1


def test_no_device_fails_loudly():
    """Without a B200 the product path raises -- there is no CPU fallback."""
    import torch
    from paper_1804_07017_b200 import lu_factor

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(RuntimeError):
        lu_factor(np.eye(8), b=4)
    from paper_1804_07017_b200 import Kind, Matrix, CacheConfig, dmf_la, qr_factor

    with pytest.raises(RuntimeError):
        qr_factor(np.eye(8), b=4)
    with pytest.raises(RuntimeError):
        dmf_la(Matrix.zeros(8, 8), CacheConfig(b=4), None, Kind.QR)


def test_mg_bookkeeping_matches_dist():
    """pflu_mg_local_cols (the C++ multi-GPU driver's block-cyclic layout) == dist.local_cols (the
    torch.distributed driver's), and the multi-GPU entry point validates its arguments on CPU."""
    from paper_1804_07017_b200 import _lib, dist

    L = _lib.load()
    for n, b, P in [(1, 1, 1), (97, 16, 3), (2048, 128, 8), (32768, 256, 8), (65536, 512, 4), (48, 16, 4)]:
        cols = [L.pflu_mg_local_cols(n, b, P, r) for r in range(P)]
        assert cols == [dist.local_cols(n, b, P, r) for r in range(P)]
        assert sum(cols) == n
    assert L.pflu_mg_local_cols(10, 2, 2, 2) == -1
    a = np.zeros((8, 8))
    piv = np.zeros(8, dtype=np.int64)
    info = ctypes.c_int64(0)
    opt = _lib.options()
    assert L.pflu_getrf_mg(None, 8, 8, 2, 1, 2, piv.ctypes.data, ctypes.byref(info), ctypes.byref(opt), None, 0, None) == -1
    assert L.pflu_getrf_mg(a.ctypes.data, 8, 4, 2, 1, 2, piv.ctypes.data, ctypes.byref(info), ctypes.byref(opt), None, 0, None) == -3
    assert L.pflu_getrf_mg(a.ctypes.data, 8, 8, 2, 2, 2, piv.ctypes.data, ctypes.byref(info), ctypes.byref(opt), None, 0, None) == -5
    assert L.pflu_getrf_mg(a.ctypes.data, 8, 8, 2, 1, 0, piv.ctypes.data, ctypes.byref(info), ctypes.byref(opt), None, 0, None) == -6
    assert L.pflu_init(0, None) == -1
