"""Generate golden vectors for the LU hot path by running the UNMODIFIED reference
(`panelforge`, arXiv 1804.07017 package) in this container.

This script is test infrastructure: it is run by hand, here, never on the GPU box.
It imports the reference from a scratch COPY (default /tmp/refpkg/src; make it with
`cp -r /root/reference/pkg /tmp/refpkg`) so numba's cache never writes into the
read-only reference tree.

Outputs (committed):
  small_cases.npz   -- tiny LU / laswp / trsm / gemm cases with the reference's outputs
  configs.json      -- BASELINE configs C1..C3: sha256 of the reference factors (row-major
                       float64 bytes), sha256 of the first 256 rows, info, timings
  configs_pivots.npz -- full 0-based pivot vectors for those configs (int32)

Usage: REF_PKG_SRC=/tmp/refpkg/src python tests/golden/make_golden.py [small|c1|c2|c2s|c3|c4 ...]
(GOLDEN_OUT=dir writes configs.json / configs_pivots.npz there instead; c4 takes ~50 min on 8 cores.)
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.environ.get("REF_PKG_SRC", "/tmp/refpkg/src"))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import panelforge as pf  # noqa: E402  (the reference)
from panelforge import CacheConfig, Kind, Matrix, Pool  # noqa: E402

PREFIX_ROWS = 256


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def config_matrix(name: str) -> tuple[np.ndarray, int]:
    """Seeded BASELINE inputs, SURVEY.md §8(d) (row-major float64)."""
    if name == "c1":
        return np.random.default_rng(0).uniform(-1.0, 1.0, size=(2048, 2048)), 128
    if name in ("c2", "c2s"):
        a = np.random.default_rng(1).uniform(-1.0, 1.0, size=(8192, 8192))
        if name == "c2s":
            a[np.diag_indices(8192)] += 8192.0
        return a, 256
    if name == "c3":
        return np.random.default_rng(2).standard_normal((16384, 16384)), 256
    if name == "c4":
        return np.random.default_rng(3).uniform(-1.0, 1.0, size=(32768, 32768)), 256
    raise KeyError(name)


def run_ref_lu(a: np.ndarray, b: int, pool, depth: int = 1):
    m = Matrix.from_array(a)
    cfg = CacheConfig(b=b)
    t0 = time.perf_counter()
    if depth == 1:
        out = pf.dmf_la(m, cfg, pool, Kind.LU)
    else:
        out = pf.dmf_mtb(m, cfg, pool, Kind.LU)
    dt = time.perf_counter() - t0
    return np.ascontiguousarray(out.matrix.array), np.asarray(out.pivots) - 1, int(out.info), dt


def gen_small(pool):
    cases = {}

    def add(tag, a, b, depth=0):
        a = np.ascontiguousarray(a, dtype=np.float64)
        f, piv, info, _ = run_ref_lu(a.copy(), b, pool, depth)
        cases[f"{tag}__a"] = a
        cases[f"{tag}__f"] = f
        cases[f"{tag}__piv"] = piv.astype(np.int64)
        cases[f"{tag}__meta"] = np.array([b, info, depth], dtype=np.int64)

    # reference known-answer shapes (test_factor.py:24-79, 266-420)
    add("swap2", [[0.0, 1.0], [1.0, 0.0]], 16)
    add("diag4", np.diag([5.0, 4.0, 3.0, 2.0]), 16)
    add("zero3", [[1.0, 0.0, 2.0], [2.0, 0.0, 1.0], [4.0, 0.0, 3.0]], 16)
    b = 16
    for n in (b, 2 * b, 5 * b, 5 * b + 17):
        add(f"grid{n}", np.random.default_rng(1000 + n).random((n, n)), b, depth=1)
    add("u300", np.random.default_rng(5).uniform(-1, 1, (300, 300)), 16, depth=1)
    add("n200", np.random.default_rng(19).random((200, 200)), 16)
    add("tall57x32", np.random.default_rng(18).random((3 * b + 9, 2 * b)), b)
    sing = np.random.default_rng(21).random((48, 48))
    sing[:, 5] = 0.0
    add("sing48", sing, b)
    add("la6b", np.random.default_rng(15).random((96, 96)), b, depth=1)
    add("la4b7", np.random.default_rng(16).random((71, 71)), b, depth=1)
    add("n257b64", np.random.default_rng(7).standard_normal((257, 257)), 64, depth=1)
    # ties: integer-valued columns with equal magnitudes -> smallest row wins
    tie = np.array([[1.0, 2.0, 3.0, 1.0], [-3.0, 1.0, 0.5, 2.0],
                    [3.0, -2.0, 1.0, 0.0], [-3.0, 4.0, 2.0, 1.0]])
    add("tie4", tie, 2)

    # level-2/3 kernel known answers (test_kernels.py:241-396)
    rng = np.random.default_rng(31)
    x = rng.random((40, 24))
    piv = np.array([3, 3, 40, 5, 17, 6, 40], dtype=np.int64)          # 1-based, row_offset 0
    lm = Matrix.from_array(x.copy())
    pf.laswp(lm.view(), piv)
    cases["laswp__a"], cases["laswp__piv1"], cases["laswp__out"] = x, piv, np.ascontiguousarray(lm.array)
    l11 = rng.standard_normal((24, 24))
    xs = rng.standard_normal((24, 37))
    tm = Matrix.from_array(xs.copy())
    pf.trsm_llnu(Matrix.from_array(l11).view(), tm.view())
    cases["trsm__l"], cases["trsm__x"], cases["trsm__out"] = l11, xs, np.ascontiguousarray(tm.array)
    c0 = rng.standard_normal((45, 38))
    a0 = rng.standard_normal((45, 19))
    b0 = rng.standard_normal((19, 38))
    cm = Matrix.from_array(c0.copy())
    neg = Matrix.from_array(np.negative(b0))
    pf.gemm(cm.view(), Matrix.from_array(a0).view(), neg.view(), cfg=CacheConfig(b=16, nc=256, kc=8, mc=24, mr=8, nr=6))
    cases["gemm__c"], cases["gemm__a"], cases["gemm__b"], cases["gemm__out"] = c0, a0, b0, np.ascontiguousarray(cm.array)
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **cases)
    print("small cases:", len([k for k in cases if k.endswith("__a")]))


OUT = os.environ.get("GOLDEN_OUT", HERE)


def gen_config(name, pool):
    a, b = config_matrix(name)
    n = int(a.shape[0])
    f, piv, info, dt = run_ref_lu(a, b, pool, depth=1)
    del a
    path = os.path.join(OUT, "configs.json")
    meta = json.load(open(path)) if os.path.exists(path) else {}
    meta[name] = {
        "n": n, "b": b, "depth": 1, "info": info,
        "sha256_factors": sha(f), f"sha256_rows_0_{PREFIX_ROWS}": sha(f[:PREFIX_ROWS]),
        "ref_seconds": round(dt, 2), "ref_threads": pool.t,
        "first_pivots": [int(p) for p in piv[:8]],
        "max_abs_L": float(np.max(np.abs(np.tril(f, -1)))),
    }
    json.dump(meta, open(path, "w"), indent=1, sort_keys=True)
    pz = os.path.join(OUT, "configs_pivots.npz")
    d = dict(np.load(pz)) if os.path.exists(pz) else {}
    d[name] = piv.astype(np.int32)
    np.savez_compressed(pz, **d)
    print(name, meta[name])


if __name__ == "__main__":
    what = sys.argv[1:] or ["small", "c1"]
    with Pool(int(os.environ.get("PANELFORGE_THREADS", os.cpu_count() or 1))) as pool:
        for w in what:
            if w == "small":
                gen_small(pool)
            else:
                gen_config(w, pool)
