"""The ctypes mirrors in the Python binding match include/hs.h's structs and enums
byte for byte (compiled here with gcc against the header; no GPU)."""
from __future__ import annotations

import ctypes
import os
import subprocess
import tempfile

import pytest

import paper_2505_06703_b200 as hs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROBE = r"""
#include <stddef.h>
#include <stdio.h>
#include "hs.h"
int main(void) {
    printf("hs_create_opts %zu\n", sizeof(hs_create_opts));
    printf("hs_scan_opts %zu\n", sizeof(hs_scan_opts));
    printf("hs_batch_item %zu %zu %zu\n", sizeof(hs_batch_item), offsetof(hs_batch_item, n_chars),
           offsetof(hs_batch_item, skin_out));
    printf("hs_animate_opts %zu %zu\n", sizeof(hs_animate_opts), offsetof(hs_animate_opts, workspace_bytes));
    printf("hs_skin_opts %zu %zu\n", sizeof(hs_skin_opts), offsetof(hs_skin_opts, workspace_bytes));
    printf("hs_layer %zu\n", sizeof(hs_layer));
    printf("HS_MAX_BATCH %d\n", HS_MAX_BATCH);
    printf("HS_ALGO_BLOCKED %d\n", (int)HS_ALGO_BLOCKED);
    printf("HS_ERR_UNSUPPORTED %d\n", (int)HS_ERR_UNSUPPORTED);
    return 0;
}
"""


@pytest.fixture(scope="module")
def c_layout():
    with tempfile.TemporaryDirectory() as d:
        src, exe = os.path.join(d, "probe.c"), os.path.join(d, "probe")
        open(src, "w").write(PROBE)
        subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), src, "-o", exe], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    return {ln.split()[0]: [int(x) for x in ln.split()[1:]] for ln in out.splitlines()}


def test_struct_sizes_and_offsets(c_layout):
    assert c_layout["hs_create_opts"] == [ctypes.sizeof(hs._CreateOpts)]
    assert c_layout["hs_scan_opts"] == [ctypes.sizeof(hs._ScanOpts)]
    assert c_layout["hs_batch_item"] == [ctypes.sizeof(hs._BatchItem), hs._BatchItem.n_chars.offset,
                                         hs._BatchItem.skin_out.offset]
    assert c_layout["hs_animate_opts"] == [ctypes.sizeof(hs._AnimateOpts), hs._AnimateOpts.workspace_bytes.offset]
    assert c_layout["hs_skin_opts"] == [ctypes.sizeof(hs._SkinOpts), hs._SkinOpts.workspace_bytes.offset]
    assert c_layout["hs_layer"] == [hs.LAYER_DTYPE.itemsize]


def test_enums_and_limits(c_layout):
    assert c_layout["HS_MAX_BATCH"] == [hs.MAX_BATCH]
    assert c_layout["HS_ALGO_BLOCKED"] == [hs.ALGO["blocked"]]
    assert c_layout["HS_ERR_UNSUPPORTED"] == [hs.HS_ERR_UNSUPPORTED]


def test_c_client_builds_against_the_header():
    """include/hs.h is plain C11 (no C++ in the ABI): the example client compiles with
    -Wall -Wextra -Werror and links against libhs.so (running it needs a GPU:
    tests/test_gpu_parity.py::test_c_client_runs)."""
    import __graft_entry__ as ge
    hs.build()
    out = ge.build_examples()
    assert os.path.exists(out) and os.access(out, os.X_OK)
