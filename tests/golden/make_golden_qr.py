"""Golden vectors for the QR path (Kind.QR), made by running the
UNMODIFIED reference (`panelforge`) in this container -- test infrastructure, run by hand here,
never on the GPU box.  Imports the reference from a scratch COPY (default /tmp/refpkg/src; make it
with `cp -r /root/reference/pkg /tmp/refpkg`).

Output (committed): qr_cases.npz -- for every case `<tag>_a` (input, row-major), `<tag>_f` (the
reference's factors: R on/above the diagonal, reflectors below, row-major), `<tag>_tau`, `<tag>_b`.
Cases `unb_*` are reference qr_unb panels (bitwise pins of the panel kernel); `mtb_*` / `la_*` are
dmf_mtb / dmf_la with kind=Kind.QR.

Usage: REF_PKG_SRC=/tmp/refpkg/src python tests/golden/make_golden_qr.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.environ.get("REF_PKG_SRC", "/tmp/refpkg/src"))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import panelforge as pf  # noqa: E402  (the reference)
from panelforge import CacheConfig, Kind, Matrix, Pool  # noqa: E402


def main() -> None:
    out = {}
    rng = np.random.default_rng
    unb = {
        "unb_n20x5": rng(9).standard_normal((20, 5)),
        "unb_zero3x2": np.array([[0.0, 1.0], [0.0, 2.0], [0.0, 3.0]]),
        "unb_triu6": np.triu(rng(4).random((6, 6))) + np.eye(6),
        "unb_u100x32": rng(21).uniform(-1.0, 1.0, (100, 32)),
    }
    for tag, a in unb.items():
        m = Matrix.from_array(a.copy())
        tau = pf.qr_unb(m.view())
        out[f"{tag}_a"] = a
        out[f"{tag}_f"] = np.ascontiguousarray(m.array)
        out[f"{tag}_tau"] = np.asarray(tau)
        out[f"{tag}_b"] = np.array(a.shape[1])
    zc = rng(13).uniform(-1.0, 1.0, (48, 48))
    zc[:, 5] = 0.0
    full = {
        "mtb_u64b16": (rng(11).uniform(-1.0, 1.0, (64, 64)), 16, "mtb"),
        "la_u64b16": (rng(11).uniform(-1.0, 1.0, (64, 64)), 16, "la"),
        "mtb_tall80x48b16": (rng(12).standard_normal((80, 48)), 16, "mtb"),
        "mtb_zerocol48b8": (zc, 8, "mtb"),
        "la_u256b32": (rng(14).uniform(-1.0, 1.0, (256, 256)), 32, "la"),
        "la_rag300x200b64": (rng(15).standard_normal((300, 200)), 64, "la"),
    }
    with Pool(4) as pool:
        for tag, (a, b, strat) in full.items():
            m = Matrix.from_array(a.copy())
            cfg = CacheConfig(b=b)
            res = pf.dmf_la(m, cfg, pool, Kind.QR) if strat == "la" else pf.dmf_mtb(m, cfg, pool, Kind.QR)
            out[f"{tag}_a"] = a
            out[f"{tag}_f"] = np.ascontiguousarray(res.matrix.array)
            out[f"{tag}_tau"] = np.asarray(res.tau)
            out[f"{tag}_b"] = np.array(b)
            f_, o_ = pf.qr_residual(a, res)
            print(tag, a.shape, b, strat, "factor", f_.value, "ortho", o_.value)
    np.savez_compressed(os.path.join(HERE, "qr_cases.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
