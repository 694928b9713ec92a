#!/usr/bin/env python
"""Tuning aid: per-call time of hs_animate on the C5 skeletons at bench size, fused and
two-pass placements and workspace sizes (median of 10 after 3 warm-ups, CUDA events)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import hsgen  # noqa: E402
import paper_2505_06703_b200 as hs  # noqa: E402

n = 333_333
res = {}
for name in ["hum64", "chain256", "tree1024"]:
    par = hsgen.skeleton(name)
    J = len(par)
    sk = hs.Skeleton(par, hsgen.inv_bind(2, J))
    cs = hs.ClipSet(sk, hsgen.clips(100, J, 8, 31), 30.0, 1)
    lay = hsgen.layers(5, n, 2, 8, 1.5)
    layers = torch.from_numpy(lay.view(np.int32).reshape(n, 2, 4)).cuda()
    g = torch.empty((n, J, 3, 4), device="cuda")
    s = torch.empty_like(g)
    for mode, ws in (("fused", 0), ("two_pass", 0), ("two_pass_256M", 256 << 20), ("two_pass_48M", 48 << 20)):
        m = mode[:8]
        for _ in range(3):
            hs.animate(sk, cs, layers, g, s, mode=m, workspace_bytes=ws)
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            hs.animate(sk, cs, layers, g, s, mode=m, workspace_bytes=ws)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[f"{name} {mode}"] = round(statistics.median(ts), 3)
print(os.environ.get("HS_LIB", "default"), res, flush=True)
for mode in ("fused", "two_pass", "two_pass_256M", "two_pass_48M"):
    print(mode, "total", round(sum(v for k, v in res.items() if k.endswith(mode)), 3), flush=True)
