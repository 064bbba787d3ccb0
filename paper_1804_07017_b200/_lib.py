"""ctypes binding of libpflu.so (C ABI in include/pflu.h).

The CUDA library is the ONLY compute path: if it is missing or no B200 is visible, calls
fail loudly (RuntimeError) -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PFLU_LIB_PATH") or os.path.join(_HERE, "libpflu.so")

PFLU_OK = 0
PFLU_ERR_CUDA = 1
PFLU_ERR_NOMEM = 2
PFLU_ERR_UNSUPPORTED = 3

TRACE_LABELS = {0: "PF", 1: "TU", 2: "TU_L", 3: "TU_R", 4: "GEMM", 5: "BCAST"}

#: every symbol include/pflu.h declares (checked by tests/test_boundary.py)
EXPORTS = (
    "pflu_version", "pflu_launch_count", "pflu_set_trace_mask", "pflu_last_error", "pflu_default_options", "pflu_device_count",
    "pflu_getrf", "pflu_getrf_device", "pflu_panel", "pflu_laswp", "pflu_swap_trsm",
    "pflu_trsm", "pflu_gemm_update", "pflu_info_reset", "pflu_info_read", "pflu_pivot_plan",
    "pflu_swap_trsm_plan", "pflu_copy2d", "pflu_release_workspace", "pflu_diag_inv", "pflu_swap_trsm_inv",
    "pflu_geqrf", "pflu_geqrf_device", "pflu_qr_panel", "pflu_larft", "pflu_apply_block_reflector",
    "pflu_init", "pflu_finalize", "pflu_mg_size", "pflu_mg_uses_nccl", "pflu_mg_local_cols", "pflu_getrf_mg",
)


class Options(ctypes.Structure):
    _fields_ = [("exact", ctypes.c_int), ("panel_ctas", ctypes.c_int),
                ("leaf_width", ctypes.c_int), ("panel_kernel", ctypes.c_int), ("malleable", ctypes.c_int),
                ("reserved", ctypes.c_int * 3)]


class TraceEvent(ctypes.Structure):
    _fields_ = [("label", ctypes.c_int32), ("k", ctypes.c_int32),
                ("start_ms", ctypes.c_float), ("end_ms", ctypes.c_float), ("flop", ctypes.c_double)]


_lib = None
_lock = threading.Lock()

_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
_pi64 = ctypes.POINTER(ctypes.c_int64)


def load():
    """Load libpflu.so (raises RuntimeError if it has not been built)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"libpflu.so not found at {LIB_PATH}: build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        L.pflu_version.restype = ctypes.c_int
        L.pflu_version.argtypes = []
        L.pflu_launch_count.restype = ctypes.c_longlong
        L.pflu_launch_count.argtypes = []
        L.pflu_set_trace_mask.restype = ctypes.c_uint
        L.pflu_set_trace_mask.argtypes = [ctypes.c_uint]
        L.pflu_last_error.restype = ctypes.c_char_p
        L.pflu_last_error.argtypes = []
        L.pflu_default_options.restype = None
        L.pflu_default_options.argtypes = [ctypes.POINTER(Options)]
        L.pflu_device_count.restype = ctypes.c_int
        L.pflu_device_count.argtypes = []
        L.pflu_getrf.restype = ctypes.c_int
        L.pflu_getrf.argtypes = [_vp, _i64, _i64, _i64, _i64, ctypes.c_int, _vp, _pi64, ctypes.POINTER(Options)]
        L.pflu_getrf_device.restype = ctypes.c_int
        L.pflu_getrf_device.argtypes = [_vp, _i64, _i64, _i64, _i64, ctypes.c_int, _vp, _pi64, _vp,
                                        ctypes.POINTER(Options), ctypes.POINTER(TraceEvent), ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_int)]
        L.pflu_panel.restype = ctypes.c_int
        L.pflu_panel.argtypes = [_vp, _i64, _i64, _i64, _i64, _i64, _vp, _pi64, _vp, ctypes.POINTER(Options)]
        L.pflu_laswp.restype = ctypes.c_int
        L.pflu_laswp.argtypes = [_vp, _i64, _i64, _i64, _vp, _i64, _i64, _vp]
        L.pflu_swap_trsm.restype = ctypes.c_int
        L.pflu_swap_trsm.argtypes = [_vp, _i64, _i64, _i64, _i64, _vp, _i64, _i64, _vp]
        L.pflu_trsm.restype = ctypes.c_int
        L.pflu_trsm.argtypes = [_vp, _i64, _i64, _vp, _i64, _i64, _vp]
        L.pflu_gemm_update.restype = ctypes.c_int
        L.pflu_gemm_update.argtypes = [_vp, _i64, _vp, _i64, _vp, _i64, _i64, _i64, _i64, ctypes.c_int, _vp]
        L.pflu_info_reset.restype = ctypes.c_int
        L.pflu_info_reset.argtypes = [_vp]
        L.pflu_info_read.restype = ctypes.c_int
        L.pflu_info_read.argtypes = [_pi64, _vp]
        L.pflu_pivot_plan.restype = ctypes.c_int
        L.pflu_pivot_plan.argtypes = [_vp, _i64, _i64, _vp, _vp]
        L.pflu_copy2d.restype = ctypes.c_int
        L.pflu_copy2d.argtypes = [_vp, _i64, _vp, _i64, _i64, _i64, _vp]
        L.pflu_release_workspace.restype = ctypes.c_int
        L.pflu_release_workspace.argtypes = []
        L.pflu_swap_trsm_plan.restype = ctypes.c_int
        L.pflu_swap_trsm_plan.argtypes = [_vp, _i64, _i64, _i64, _vp, _i64, _i64, _vp, _i64, _vp]
        L.pflu_diag_inv.restype = ctypes.c_int
        L.pflu_diag_inv.argtypes = [_vp, _i64, _i64, _vp, _vp]
        L.pflu_swap_trsm_inv.restype = ctypes.c_int
        L.pflu_swap_trsm_inv.argtypes = [_vp, _i64, _i64, _i64, _vp, _i64, _i64, _vp, _i64, _vp, _vp]
        _pd = ctypes.c_void_p
        L.pflu_geqrf.restype = ctypes.c_int
        L.pflu_geqrf.argtypes = [_vp, _i64, _i64, _i64, _i64, ctypes.c_int, _pd]
        L.pflu_geqrf_device.restype = ctypes.c_int
        L.pflu_geqrf_device.argtypes = [_vp, _i64, _i64, _i64, _i64, ctypes.c_int, _pd, _vp,
                                        ctypes.POINTER(TraceEvent), ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        L.pflu_qr_panel.restype = ctypes.c_int
        L.pflu_qr_panel.argtypes = [_vp, _i64, _i64, _i64, _i64, _i64, _pd, _vp]
        L.pflu_larft.restype = ctypes.c_int
        L.pflu_larft.argtypes = [_vp, _i64, _i64, _i64, _pd, _pd, _i64, _vp]
        L.pflu_apply_block_reflector.restype = ctypes.c_int
        L.pflu_apply_block_reflector.argtypes = [_vp, _i64, _i64, _i64, _pd, _vp, _i64, _i64, _vp]
        L.pflu_init.restype = ctypes.c_int
        L.pflu_init.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        L.pflu_finalize.restype = ctypes.c_int
        L.pflu_finalize.argtypes = []
        L.pflu_mg_size.restype = ctypes.c_int
        L.pflu_mg_size.argtypes = []
        L.pflu_mg_uses_nccl.restype = ctypes.c_int
        L.pflu_mg_uses_nccl.argtypes = []
        L.pflu_mg_local_cols.restype = ctypes.c_int64
        L.pflu_mg_local_cols.argtypes = [_i64, _i64, ctypes.c_int, ctypes.c_int]
        L.pflu_getrf_mg.restype = ctypes.c_int
        L.pflu_getrf_mg.argtypes = [_vp, _i64, _i64, _i64, ctypes.c_int, ctypes.c_int, _vp, _pi64,
                                    ctypes.POINTER(Options), ctypes.POINTER(TraceEvent), ctypes.c_int,
                                    ctypes.POINTER(ctypes.c_int)]
        _lib = L
        return L


def check(rc: int, what: str) -> None:
    """Map a C-ABI return code to the reference's exception types (ValueError for invalid
    arguments, factor.py:293-297 / kernels.py:282-291; RuntimeError for device failures)."""
    if rc == PFLU_OK:
        return
    if rc < 0:
        raise ValueError(f"{what}: invalid argument #{-rc}")
    msg = load().pflu_last_error().decode(errors="replace")
    raise RuntimeError(f"{what} failed (code {rc}): {msg}")


PANEL_AUTO, PANEL_GRID, PANEL_CLUSTER, PANEL_RECURSIVE, PANEL_MCLUSTER = 0, 1, 2, 3, 4


#: pflu_options.malleable: dynamic tile scheduling (default), SM-partitioned LA, LA_MB (join grid)
SCHED_DYNAMIC, SCHED_LA, SCHED_LA_MB = 0, 1, 2


def options(exact: bool = False, panel_ctas: int = 0, leaf_width: int = 0, panel_kernel: int = PANEL_AUTO,
            malleable: int = SCHED_DYNAMIC) -> Options:
    o = Options()
    load().pflu_default_options(ctypes.byref(o))
    o.exact = 1 if exact else 0
    o.panel_ctas = int(panel_ctas)
    o.leaf_width = int(leaf_width)
    o.panel_kernel = int(panel_kernel)
    o.malleable = int(malleable)
    return o
