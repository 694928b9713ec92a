"""The oracle and the product share no code (tier rule ③): neither imports, includes or
links the other; only the seeded generators (hsgen/, no method arithmetic) serve both.
Static checks on the sources (CPU)."""
from __future__ import annotations

import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _files(d, exts):
    for dp, _, fs in os.walk(os.path.join(ROOT, d)):
        for f in fs:
            if f.endswith(exts):
                yield os.path.join(dp, f)


def test_product_never_touches_the_oracle():
    for f in _files("paper_2505_06703_b200", (".py", ".cpp", ".cu", ".cuh", ".hpp", ".h")):
        src = open(f).read()
        assert not re.search(r"^\s*(import|from)\s+oracle\b", src, re.M), f
        assert "liboracle" not in src and "oracle/" not in src, f
        assert "orc_" not in src, f


def test_oracle_never_touches_the_product():
    for f in _files("oracle", (".py", ".c", ".h")):
        src = open(f).read()
        assert not re.search(r"^\s*(import|from)\s+paper_2505_06703_b200\b", src, re.M), f
        assert "libhs" not in src and "csrc" not in src and "hs.h" not in src, f
        assert not re.search(r"\bhs_[a-z]+\(", src), f


def test_generators_hold_no_method_arithmetic():
    # hsgen produces inputs only: no compose / scan / skinning entry points
    for f in _files("hsgen", (".py", ".c", ".cu")):
        src = open(f).read()
        for word in ("compose", "orc_scan", "hs_scan", "skin_vertices", "animate"):
            assert word not in src, (f, word)
