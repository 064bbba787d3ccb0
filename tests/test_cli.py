"""The reference-compatible bench CLI (paper_1804_07017_b200.cli), CPU parts."""
import hashlib
import io

import numpy as np
import pytest

from paper_1804_07017_b200 import cli

# sha256 of panelforge.bench.make_instance(seed, "lu", n).array (row-major bytes), computed with the
# reference itself when this test was written
REF_INSTANCE_SHA = {
    (0, 64): "074c14c1263aaf3b7daef2d870f5c82e6ae518fa4a4b88b4d127879f471642a4",
    (0, 300): "bb896681aafd3d3423e1ffec87f1205439757c89fc39cd6399a558430664232b",
    (7, 129): "fa32eec2bd10bbc28da6afe52e79d0e613a1ae2f682a68bf5c7e03dff36c901d",
}


@pytest.mark.parametrize("seed,n", sorted(REF_INSTANCE_SHA))
def test_instances_match_reference(seed, n):
    a = cli.make_instance(seed, "lu", n)
    assert hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest() == REF_INSTANCE_SHA[(seed, n)]


def test_csv_round_trip():
    recs = [cli.BenchRecord("LU", "LA", 2048, 128, 1, 0.0123, 465.5, 0.0571),
            cli.BenchRecord("LU", "MTB", 4096, 256, 1, 0.1, 916.3, None)]
    buf = io.StringIO()
    cli.emit_csv(recs, buf)
    text = buf.getvalue()
    assert text.splitlines()[0] == "kind,strategy,n,b,threads,seconds,gflops,residual"
    assert cli.parse_csv(text) == recs
    with pytest.raises(ValueError):
        cli.parse_csv("bad header\n")


def test_parser_and_scope():
    args = cli.build_parser().parse_args(["--strategy", "la", "--n-min", "512", "--n-max", "1024", "--check"])
    assert args.strategy == "la" and args.check and args.n_step == 256
    with pytest.raises(SystemExit):
        cli.build_parser().parse_args(["--strategy", "rtm"])
    with pytest.raises(ValueError):
        cli.run_sweep("gemm", ["la"], [64], 16, 1, 0, False)
