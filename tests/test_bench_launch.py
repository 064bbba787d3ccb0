"""bench.py's multi-GPU launcher (CPU): `python bench.py --gpus N` outside torchrun re-launches itself
with N ranks and rank 0 reports n_gpus = N (VERDICT r1 "next" 2).  The self-test mode joins a gloo
group instead of touching GPUs, so the spawning logic is exercised here without CUDA."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("n", [2, 3])
def test_bench_spawns_n_ranks(n):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--selftest-launch"],
                         capture_output=True, text=True, env=env, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout          # exactly one JSON line, from rank 0
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == n and rec["ranks_seen"] == n and rec["argv_gpus"] == n


def test_bench_refuses_missing_gpus():
    """Without enough visible GPUs the launcher fails loudly instead of measuring fewer ranks."""
    import torch

    if torch.cuda.device_count() >= 64:
        pytest.skip("box has >= 64 GPUs")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "64"],
                         capture_output=True, text=True, env=env, timeout=300, cwd=ROOT)
    assert out.returncode != 0
    assert "64" in out.stderr and not any(ln.startswith("{") for ln in out.stdout.splitlines())
