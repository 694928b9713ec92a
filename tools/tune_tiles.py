#!/usr/bin/env python
"""Tuning aid: HS_ALGO_TILES on C6 (2,000 x tree16384) across tile sizes / stage counts;
median of 7 launches after 2 warm-ups (CUDA events), GB/s at 144 B/joint.  --dfs: the
same trees with depth-first labels (few cross-tile parents)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hsgen  # noqa: E402
import paper_2505_06703_b200 as hs  # noqa: E402

(name, n, seed, type_, ib_seed), = hsgen.CONFIGS[6]
par = hsgen.skeleton(name)
DFS = "--dfs" in sys.argv   # the same trees labelled in depth-first order (heavy child first)
if DFS:
    par = hsgen.dfs_labels(par)
J = len(par)
x = torch.empty((n, J, 3, 4), device="cuda")
assert hsgen.lib_cuda().hsg_cuda_local_poses(seed, type_, J, 0, n, x.data_ptr(),
                                             torch.cuda.current_stream().cuda_stream) == 0
g, s = torch.empty_like(x), torch.empty_like(x)
ref = None
QUICK = "--quick" in sys.argv   # the library defaults only
for kw in [{}] if QUICK else ([{}, {"tile_joints": 1024, "chunk": 5}, {"tile_joints": 1024, "chunk": 5, "stages": 2},
            {"tile_joints": 768, "chunk": 3}, {"tile_joints": 1024, "chunk": 7}] if DFS else
           [{}, {"tile_joints": 672, "sbufs": 1}, {"tile_joints": 672, "stages": 2},
            {"tile_joints": 672, "stages": 2, "sbufs": 1}, {"tile_joints": 640, "sbufs": 1},
            {"tile_joints": 608}]):
    kw = dict(kw)
    ctas = kw.pop("ctas", 0)
    try:
        sk = hs.Skeleton(par, hsgen.inv_bind(ib_seed, J), force_split=True, **kw)
    except hs.HSError as e:
        print(kw, "create failed", e)
        continue
    for _ in range(2):
        sk.scan_into(x, g, s, algo="tiles", tile_ctas=ctas)
    ts = []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sk.scan_into(x, g, s, algo="tiles", tile_ctas=ctas)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    print(kw, "ctas/SM", ctas or 1, "K", sk.query("seq_chunk"), "sbufs", sk.query("seq_sbufs"), "F", sk.query("seq_tile_joints"), "KT", sk.query("seq_tiles"), "smem", sk.query("seq_smem_bytes"),
          f"{ms:.4f} ms {144 * n * J / ms / 1e6:.0f} GB/s", flush=True)
    sk.close()
