#!/usr/bin/env python
"""HBM speed of light for the hot path's traffic mix (tools/sol_stream.cu): read 48 B,
write 2 x 48 B per joint with no arithmetic, at the C5 tree1024 launch's size
(333,333 characters x 1024 joints: 16.4 GB in, 32.8 GB out), by TMA bulk streaming (the
chunked kernel's producer alone) and by SIMT float4 loads / stores; plus the plain 1:1
copy for comparison with MEASURED_PEAKS.json.  Median of 10 CUDA-event-timed launches
after 3 warm-ups; GB/s = bytes read + written / time.

    python tools/sol_stream.py [--out profiles/r02_sol_stream.json]"""
import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "build", "libsol.so")


def build():
    src = os.path.join(ROOT, "tools", "sol_stream.cu")
    if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(src):
        os.makedirs(os.path.dirname(SO), exist_ok=True)
        subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler",
                        "-fPIC", src, "-o", SO], check=True)
    L = ctypes.CDLL(SO)
    vp, i32 = ctypes.c_void_p, ctypes.c_int
    L.sol_tma_launch.argtypes = [vp, vp, vp, ctypes.c_int64, i32, i32, i32, vp]
    L.sol_simt_launch.argtypes = [vp, vp, vp, ctypes.c_int64, i32, i32, vp]
    L.sol_tma_launch.restype = L.sol_simt_launch.restype = i32
    return L


def timed(fn):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts), min(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    L = build()
    joints = 333_333 * 1024
    nbytes = joints * 48
    tile = 48 * 1024                    # the chunked kernel's tree1024 tile: 1024 joints x 48 B
    n_tiles = nbytes // tile
    x = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda").uniform_()
    o0, o1 = torch.empty_like(x), torch.empty_like(x)
    st = torch.cuda.current_stream().cuda_stream
    rows = []

    def rec(name, n_out, ms):
        b = nbytes * (1 + n_out)
        rows.append({"kernel": name, "writes_per_read": n_out, "ms_median": ms[0], "ms_min": ms[1],
                     "gbs_median": b / ms[0] / 1e6, "gbs_best": b / ms[1] / 1e6})
        print(rows[-1], flush=True)

    for n_out in (2, 1):
        for stages in (3, 4):
            rec(f"sol_tma stages={stages}", n_out,
                timed(lambda: L.sol_tma_launch(x.data_ptr(), o0.data_ptr(), o1.data_ptr(), n_tiles, tile, stages,
                                               n_out, st)))
        for bps in (2, 4):
            rec(f"sol_simt blocks/SM={bps}", n_out,
                timed(lambda: L.sol_simt_launch(x.data_ptr(), o0.data_ptr(), o1.data_ptr(), nbytes // 16, bps,
                                                n_out, st)))
    rec("torch copy_", 1, timed(lambda: o0.copy_(x)))
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    res = {"bytes_in": nbytes, "tile_bytes": tile, "measured_peaks_hbm_gbs": peaks.get("hbm_gbs"),
           "device": torch.cuda.get_device_name(), "rows": rows}
    if args.out:
        json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    sys.exit(main())
