#!/usr/bin/env python
"""Multi-CTA skeletons: time of HS_ALGO_TILES (multi-tile kernel) and
HS_ALGO_SPLIT (three-kernel path) on tree16384 (16,384 joints, L = 1024) across crowd
sizes; median of 7 launches after 2 warm-ups (CUDA events), GB/s at 144 B/joint.
Prints one JSON line."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hsgen  # noqa: E402
import paper_2505_06703_b200 as hs  # noqa: E402


def timed(fn, n=7):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


name = sys.argv[1] if len(sys.argv) > 1 else "tree16384"
par = hsgen.skeleton(name) if not name.startswith("chain") else hsgen.chain(int(name[5:]))
J = len(par)
sk = hs.Skeleton(par, hsgen.inv_bind(6, J))
out = {"skeleton": name, "J": J, "tiles": sk.query("seq_tiles"), "F": sk.query("seq_tile_joints"),
       "exports": sk.query("seq_exports"), "smem": sk.query("seq_smem_bytes"), "runs": {}}
for n in (37, 148, 296, 592, 2000):
    x = torch.empty((n, J, 3, 4), device="cuda")
    assert hsgen.lib_cuda().hsg_cuda_local_poses(6, 0, J, 0, n, x.data_ptr(),
                                                 torch.cuda.current_stream().cuda_stream) == 0
    g, s = torch.empty_like(x), torch.empty_like(x)
    row = {}
    for algo in ("tiles", "split"):
        ms = timed(lambda: sk.scan_into(x, g, s, algo=algo))
        row[algo] = {"ms": round(ms, 4), "gbs": round(144 * n * J / ms / 1e6, 1)}
    out["runs"][n] = row
    print(n, row, flush=True)
    del x, g, s
    torch.cuda.empty_cache()
print(json.dumps(out))
