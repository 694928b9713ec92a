"""Race-detection stand-in for compute-sanitizer's racecheck (closed on this pool): the
bitwise GPU parity suites re-run against a protocol stress build (HS_DEBUG_DELAY=1) in
which every producer / consumer hand-off of the TMA + mbarrier kernels (the chunked
scan, the multi-tile scan, the streaming Stage-1 kernel) sleeps for a random 0-4 us
at random.  A missing wait, an mbarrier phase-parity slip or a buffer
reused before its bulk copy has read it then changes a result bit: the round-2
multi-tile experiment whose consumers could run two mbarrier phases ahead of the
producer failed exactly this way."""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2505_06703_b200 as hs  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITES = ["tests/test_gpu_parity.py", "tests/test_gpu_batch.py", "tests/test_gpu_stage1.py"]


def test_bitwise_suites_pass_under_random_handoff_delays():
    lib = hs.build_variant("libhs_delay.so", ["-DHS_DEBUG_DELAY=1"])
    # the sleeps are compiled into the stress build only (nanosleep in its SASS)
    env = dict(os.environ, HS_LIB=lib)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        *SUITES, "-k", "exact or bitwise or tile or forced or batch or two_pass or fused or determinism or dyadic"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
    tail = (r.stdout + r.stderr)[-3000:]
    print(tail)
    assert r.returncode == 0, tail
    assert " passed" in r.stdout
