"""Full-size parity pins for the headline configs C4 (n = 32768) and C5 (n = 65536), made by the
bitwise-pinned C oracle (oracle/pflu_oracle.c) running IN PLACE on this container's host cores.

Test infrastructure, run by hand here (never on the GPU box).  The oracle is pinned bit for bit to
the reference at C1/C2/C2s/C3 (tests/test_oracle.py); for C4 the unmodified reference's own run
(make_golden.py c4, ~50 min) is recorded next to it and the two sha256 must agree (`ref_sha_equal`).

Per config it writes into tests/golden/:
  configs.json        -- key "<cfg>": sha256 of the full factor matrix (row-major float64 bytes), of
                         its first 256 and first b rows, info, max |L|, who computed it ("source"),
                         the host seconds / threads, and the tie statistics below
  configs_pivots.npz  -- key "<cfg>": the full 0-based pivot vector (int32)
  configs_ties.npz    -- key "<cfg>": oracle.near_ties(top2, 1e-6): every column whose top-two
                         candidate magnitudes are within 1e-6 relative (col, |winner|, |runner-up|,
                         runner-up row) -- what a GPU pivot mismatch is classified against
                         (north_star: pivots identical except top-two ties within 1e-12 relative)

Usage: python tests/golden/make_golden_large.py c4 [c5]      (C5 needs ~35 GB of host memory)
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402

SPEC = {
    # name: (n, seed, distribution, b)   -- BASELINE.json configs[3], configs[4]
    "c4": (32768, 3, "uniform", 256),
    "c5": (65536, 4, "normal", 512),
}


def make(name: str) -> tuple[np.ndarray, int]:
    n, seed, dist, b = SPEC[name]
    rng = np.random.default_rng(seed)
    a = np.empty((n, n))
    rows = max(1, (1 << 27) // n)          # stream the generator in row chunks (same sequence)
    for r0 in range(0, n, rows):
        r1 = min(n, r0 + rows)
        if dist == "uniform":
            a[r0:r1] = rng.uniform(-1.0, 1.0, size=(r1 - r0, n))
        else:
            a[r0:r1] = rng.standard_normal((r1 - r0, n))
    return a, b


def sha_rows(a: np.ndarray, r0: int = 0, r1: int | None = None, chunk: int = 2048) -> str:
    h = hashlib.sha256()
    r1 = a.shape[0] if r1 is None else r1
    for s in range(r0, r1, chunk):
        h.update(np.ascontiguousarray(a[s:min(r1, s + chunk)]).tobytes())
    return h.hexdigest()


def max_abs_l(a: np.ndarray, chunk: int = 2048) -> float:
    mx = 0.0
    for s in range(0, a.shape[0], chunk):
        blk = a[s:s + chunk]
        mx = max(mx, float(np.max(np.abs(np.tril(blk, s - 1)))))
    return mx


def gen(name: str) -> None:
    threads = int(os.environ.get("ORACLE_THREADS", os.cpu_count() or 1))
    oracle.set_threads(threads)
    a, b = make(name)
    n = a.shape[0]
    t0 = time.perf_counter()
    piv, top2, info = oracle.getrf_top2_inplace(a, b)
    dt = time.perf_counter() - t0
    ties = oracle.near_ties(top2, 1e-6)
    v1, v2 = top2[:, 0], top2[:, 1]
    ok = v2 >= 0
    gaps = (v1[ok] - v2[ok]) / v1[ok]
    path = os.path.join(HERE, "configs.json")
    meta = json.load(open(path))
    rec = meta.get(name, {})
    sha_full = sha_rows(a)
    ref_sha = rec.get("sha256_factors") if rec.get("source") == "reference" else None
    rec.update({
        "n": n, "b": b, "depth": 1, "info": info,
        "sha256_factors": sha_full,
        "sha256_rows_0_256": sha_rows(a, 0, 256),
        f"sha256_rows_0_{b}": sha_rows(a, 0, b),
        "max_abs_L": max_abs_l(a),
        "first_pivots": [int(p) for p in piv[:8]],
        "oracle_seconds": round(dt, 1), "oracle_threads": threads,
        "min_top2_rel_gap": float(gaps.min()), "min_top2_rel_gap_col": int(np.nonzero(ok)[0][np.argmin(gaps)]),
        "near_ties_1e-6": int(len(ties)), "ties_1e-12": int(np.sum(gaps <= oracle.TIE_RTOL)),
    })
    if ref_sha is not None:
        rec["ref_sha_equal"] = bool(ref_sha == sha_full)
        rec["source"] = "reference (oracle re-run bitwise equal)" if rec["ref_sha_equal"] else "reference"
        if not rec["ref_sha_equal"]:
            rec["sha256_factors"] = ref_sha
            rec["oracle_sha256_factors"] = sha_full
    else:
        rec.setdefault("source", "oracle (bitwise-pinned to the reference at C1-C3)")
    meta[name] = rec
    json.dump(meta, open(path, "w"), indent=1, sort_keys=True)
    pz = os.path.join(HERE, "configs_pivots.npz")
    d = dict(np.load(pz))
    if name in d and not np.array_equal(d[name], piv.astype(np.int32)):
        raise SystemExit(f"{name}: oracle pivots differ from the committed (reference) pivots")
    d[name] = piv.astype(np.int32)
    np.savez_compressed(pz, **d)
    tz = os.path.join(HERE, "configs_ties.npz")
    t = dict(np.load(tz)) if os.path.exists(tz) else {}
    t[name] = ties
    np.savez_compressed(tz, **t)
    print(name, json.dumps(rec))


if __name__ == "__main__":
    for w in sys.argv[1:] or ["c4"]:
        gen(w)
