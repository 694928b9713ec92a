#!/usr/bin/env python
"""Tuning aid: chunked-kernel time vs tile size (hs_create_opts.tile_joints) on the C5
skeletons at bench size and on the Fig. 7 300-joint tree (CUDA-event median of 7)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hsgen  # noqa: E402
import paper_2505_06703_b200 as hs  # noqa: E402


def timed(fn):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return round(statistics.median(ts), 4)


cases = [(name, hsgen.skeleton(name), n, seed, type_) for name, n, seed, type_, _ in hsgen.CONFIGS[5]]
cases.append(("fig7-300-d60", hsgen.random_tree(60, 300, 60), 10_000, 1, 0))
for name, par, n, seed, type_ in cases:
    J = len(par)
    x = torch.empty((n, J, 3, 4), device="cuda")
    hsgen.lib_cuda().hsg_cuda_local_poses(seed, type_, J, 0, n, x.data_ptr(), torch.cuda.current_stream().cuda_stream)
    g, s = torch.empty_like(x), torch.empty_like(x)
    res = {}
    for tj in (256, 512, 1024, 2048):
        try:
            sk = hs.Skeleton(par, hsgen.inv_bind(2, J), tile_joints=tj)
        except Exception as e:  # noqa: BLE001
            res[tj] = str(e)[:30]
            continue
        res[f"{tj} (C={sk.query('tile_chars')})"] = timed(lambda: sk.scan_into(x, g, s))
    print(name, res, flush=True)
    del x, g, s
    torch.cuda.empty_cache()
