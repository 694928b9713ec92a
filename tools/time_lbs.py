#!/usr/bin/env python
"""Tuning aid: hs_scan_skin per C5 skeleton at bench size with a 1000-vertex mesh, both
placements (CUDA-event median of 5)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hsgen  # noqa: E402
import paper_2505_06703_b200 as hs  # noqa: E402

res = {}
for name, n, seed, type_, ib_seed in hsgen.CONFIGS[5]:
    par = hsgen.skeleton(name)
    J = len(par)
    sk = hs.Skeleton(par, hsgen.inv_bind(ib_seed, J))
    mesh = hs.Mesh(sk, *hsgen.mesh(200 + type_, par, 1000, type_=type_))
    x = torch.empty((n, J, 3, 4), device="cuda")
    hsgen.lib_cuda().hsg_cuda_local_poses(seed, type_, J, 0, n, x.data_ptr(),
                                          torch.cuda.current_stream().cuda_stream)
    g, s = torch.empty_like(x), torch.empty_like(x)
    v = torch.empty((n, 1000, 3), device="cuda")
    for mode in ("fused", "two_pass"):
        for _ in range(2):
            hs.scan_skin(sk, mesh, x, g, s, v, mode=mode)
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            hs.scan_skin(sk, mesh, x, g, s, v, mode=mode)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[f"{name} {mode}"] = round(statistics.median(ts), 3)
    del x, g, s, v
    torch.cuda.empty_cache()
print(res)
for mode in ("fused", "two_pass"):
    print(mode, "total", round(sum(v for k, v in res.items() if k.endswith(mode)), 3))
