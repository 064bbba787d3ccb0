"""paper_1804_07017_b200: B200-native blocked LU with partial pivoting and static look-ahead.

A from-scratch sm_100a implementation of the hot path of the reference package `panelforge`
(arXiv 1804.07017): the Kind.LU factorization behind dmf_la (look-ahead depth 1) and dmf_mtb
(depth 0), and the Kind.QR (Householder) factorization of the same drivers.  Compute runs only in libpflu.so (C ABI: include/pflu.h); see DESIGN.md.
"""
from .api import (CacheConfig, Kind, LuOutput, Matrix, Strategy, TraceEvent, dmf_la, dmf_mtb, flops,
                  getrf_device, getrf_host, lu_factor, QrOutput, geqrf_device, geqrf_host, qr_factor,
                  init_gpus, finalize_gpus, getrf_mg)
from . import _lib

__version__ = "0.1.0"

__all__ = [
    "CacheConfig", "Kind", "LuOutput", "Matrix", "Strategy", "TraceEvent", "dmf_la", "dmf_mtb", "flops",
    "getrf_device", "getrf_host", "lu_factor", "QrOutput", "geqrf_device", "geqrf_host", "qr_factor",
    "init_gpus", "finalize_gpus", "getrf_mg", "__version__",
]
