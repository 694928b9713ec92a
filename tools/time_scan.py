#!/usr/bin/env python
"""Tuning aid: per-launch time of hs_scan on the C5 skeletons at bench size, and of one
hs_scan_batch over all three (median of 10 launches after 3 warm-ups, CUDA events)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hsgen  # noqa: E402
import paper_2505_06703_b200 as hs  # noqa: E402


def timed(fn, n=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return round(statistics.median(ts), 3)


items, res = [], {}
for name, n, seed, type_, ib_seed in hsgen.CONFIGS[5]:
    par = hsgen.skeleton(name)
    J = len(par)
    sk = hs.Skeleton(par, hsgen.inv_bind(ib_seed, J))
    x = torch.empty((n, J, 3, 4), device="cuda")
    assert hsgen.lib_cuda().hsg_cuda_local_poses(seed, type_, J, 0, n, x.data_ptr(),
                                                 torch.cuda.current_stream().cuda_stream) == 0
    g, s = torch.empty_like(x), torch.empty_like(x)
    items.append((sk, x, g, s))
    res[name] = timed(lambda: sk.scan_into(x, g, s))
res["sum"] = round(sum(res.values()), 3)
res["batch"] = timed(lambda: hs.scan_batch(items))
print(os.environ.get("HS_LIB", "default"), res, flush=True)
# the multi-segment kernel on one skeleton: each crowd as two halves
two = {}
for sk, x, g, s in items:
    h = x.shape[0] // 2
    halves = [(sk, x[:h], g[:h], s[:h]), (sk, x[h:], g[h:], s[h:])]
    two[sk.n_joints] = timed(lambda: hs.scan_batch(halves))
print("as 2 segments", two, "hum64+chain256 batch", timed(lambda: hs.scan_batch(items[:2])), flush=True)
