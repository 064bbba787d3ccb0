"""Panel kernel timing sweep: median of repeated launches per (m, CTAs, leaf width).

    python tools/panel_sweep.py [lib.so] --m 32768,8192 --ctas 0,16,32 --leaf 0,8,16,32 --w 256
"""
import argparse
import ctypes
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_1804_07017_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("lib", nargs="?", default=None)
ap.add_argument("--m", default="32768,16384,8192,2048")
ap.add_argument("--w", type=int, default=256)
ap.add_argument("--ctas", default="0")
ap.add_argument("--leaf", default="0")
ap.add_argument("--reps", type=int, default=9)
ap.add_argument("--kernel", default="0", help="panel_kernel values: 0 auto, 1 grid, 2 cluster, 3 recursive")
ap.add_argument("--tag", default="")
args = ap.parse_args()
if args.lib:
    _lib.LIB_PATH = args.lib
L = _lib.load()
dev = torch.device("cuda:0")
st = torch.cuda.current_stream().cuda_stream
w = args.w
for m in [int(x) for x in args.m.split(",")]:
    x0 = torch.rand(m, w, dtype=torch.float64, device=dev) * 2 - 1
    x = x0.clone()
    piv = torch.zeros(w, dtype=torch.int64, device=dev)
    for ctas in [int(x) for x in args.ctas.split(",")]:
        for leaf, kern in [(int(x), int(y)) for x in args.leaf.split(",") for y in args.kernel.split(",")]:
            opt = _lib.options(exact=False, panel_ctas=ctas, leaf_width=leaf, panel_kernel=kern)
            times = []
            ok = True
            for r in range(args.reps + 2):
                x.copy_(x0)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                rc = L.pflu_panel(x.data_ptr(), w, m, 0, 0, w, piv.data_ptr(), None, st, ctypes.byref(opt))
                e1.record()
                if rc != 0:
                    ok = False
                    break
                torch.cuda.synchronize()
                if r >= 2:
                    times.append(e0.elapsed_time(e1))
            if not ok:
                print(f"{args.tag} m={m} ctas={ctas} leaf={leaf} kernel={kern}: unsupported")
                continue
            print(f"{args.tag} m={m} w={w} ctas={ctas} leaf={leaf} kernel={kern}: median {statistics.median(times):.3f} ms "
                  f"min {min(times):.3f} max {max(times):.3f}")
