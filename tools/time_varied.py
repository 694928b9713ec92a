#!/usr/bin/env python
"""Per-character topology (hs_scan_varied) vs the planned scan of one shared skeleton,
at C2 / C3 / C4 sizes (each varied character gets its own SPEC random tree of the same
size and depth).  CUDA-event median of 10; algorithmic HBM bytes 48 + 4 (+48 per-
character IB) in, 96 out per joint."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import hsgen  # noqa: E402
import paper_2505_06703_b200 as hs  # noqa: E402


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
    return statistics.median(ts)


rows = []
for name, n in (("hum64", 100_000), ("chain256", 50_000), ("tree1024", 20_000)):
    par = hsgen.skeleton(name)
    J = len(par)
    # per-character skeletons: the template's own depth, random shapes (labels shuffled)
    lev = np.zeros(J, int)
    for i in range(J):
        lev[i] = 1 if par[i] < 0 else lev[par[i]] + 1
    depth = int(lev.max())
    rng = np.random.default_rng(1)
    pars = np.stack([hsgen.relabel(hsgen.random_tree(int(rng.integers(1 << 30)), J, depth),
                                   rng.permutation(J).astype(np.int32))[0] for _ in range(256)])
    p = torch.from_numpy(pars[np.arange(n) % 256]).cuda()
    x = torch.empty((n, J, 3, 4), device="cuda")
    hsgen.lib_cuda().hsg_cuda_local_poses(7, 0, J, 0, n, x.data_ptr(), torch.cuda.current_stream().cuda_stream)
    ib = torch.empty_like(x)
    hsgen.lib_cuda().hsg_cuda_local_poses(8, 0, J, 0, n, ib.data_ptr(), torch.cuda.current_stream().cuda_stream)
    g, s = torch.empty_like(x), torch.empty_like(x)
    sk = hs.Skeleton(par, hsgen.inv_bind(2, J))
    t_fixed = timed(lambda: sk.scan_into(x, g, s))
    t_var = timed(lambda: hs.scan_varied(p, x, ib, g, s))
    joints = n * J
    rows.append(dict(skeleton=name, chars=n, depth=depth, fixed_ms=t_fixed, varied_ms=t_var,
                     varied_gjoints_s=joints / t_var / 1e6, varied_hbm_gbs=joints * 196 / t_var / 1e6))
    print(rows[-1], flush=True)
