"""The N > 1 bench path end to end on one GPU:
two ranks launched by torch.distributed.run with the gloo backend (NCCL refuses two
ranks on one GPU; the data path has no collective, so the ranks never wait on each
other's kernels).  Exercises everything bench.py does at N > 1: per-rank input
generation for its shard, per-rank oracle parity, the max-over-ranks timing, the e2e
leg, the all-gather of sampled G/S shards with the bitwise check against a
recomputation, and one JSON line printed by rank 0 only."""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("config,scaling,extra", [(2, "weak", []), (6, "strong", ["--no-e2e"])])
def test_two_ranks_gloo_bench(config, scaling, extra):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dist-backend", "gloo", "--config", str(config),
           "--scaling", scaling, "--steps", "3", "--warmup", "3", "--e2e-steps", "1", *extra]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1                       # rank 0 alone prints
    line = lines[0]
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["scaling"] == scaling
    assert line["parity"]["pass"] and line["parity"]["worst_all_ranks"] <= line["parity"]["tolerance"]
    v = line["multi_gpu_validation"]
    assert v["pass"] and v["backend"] == "gloo" and v["chars_checked"] > 0 and v["chunks"] >= 2
    ranks = {e["rank"] for t in v["types"].values() for e in t}
    assert ranks == {0, 1}
    if scaling == "weak":                        # rank 1 owns global characters [n, 2n)
        first = [e["first_char"] for t in v["types"].values() for e in t if e["rank"] == 1]
        assert min(first) >= 100_000
        assert line["e2e"]["value"] > 0 and line["e2e"]["matches_device_path"]
