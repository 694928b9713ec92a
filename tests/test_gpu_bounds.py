"""Memory-safety stand-in for compute-sanitizer (closed on this pool): the GPU parity
suites re-run against a debug build (HS_DEBUG_BOUNDS=1) in which every shared-memory
slot index, TMA byte count, inverse-bind row and LBS palette index of the chunked
kernel is checked against its buffer and a violation traps."""
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
SUITES = ["tests/test_gpu_fuzz.py", "tests/test_gpu_batch.py", "tests/test_gpu_lbs.py",
          "tests/test_gpu_stage1.py", "tests/test_gpu_parity.py"]


def test_parity_suites_pass_under_the_bounds_checked_build():
    lib = hs.build_variant("libhs_bounds.so", ["-DHS_DEBUG_BOUNDS=1"])
    # the checks are compiled into the debug build and only there
    assert b"hs bounds violated" in open(lib, "rb").read()
    assert b"hs bounds violated" not in open(hs.LIB_PATH, "rb").read()
    env = dict(os.environ, HS_LIB=lib)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        *SUITES, "-k", "not c_client and not capture"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    tail = (r.stdout + r.stderr)[-3000:]
    print(tail)
    assert "hs bounds violated" not in r.stdout + r.stderr
    assert r.returncode == 0, tail
