#!/usr/bin/env python
"""Per-phase cycle split of the multi-tile kernel (consumer thread 0, clock64) on C6
(2,000 x tree16384): builds the HS_PROF_HOOKS=1 variant and prints hs prof lines.
Options: --dfs (depth-first labels), create options as key=value (tile_joints=672)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["HS_DEBUG_PROF"] = "1"
import torch  # noqa: E402

import hsgen  # noqa: E402
import paper_2505_06703_b200 as hs  # noqa: E402

hs.use_library(hs.build_variant("libhs_prof.so", ["-DHS_PROF_HOOKS=1"]))
(name, n, seed, type_, ib_seed), = hsgen.CONFIGS[6]
par = hsgen.skeleton(name)
if "--dfs" in sys.argv:   # the same trees with depth-first labels
    par = hsgen.dfs_labels(par)
kw = {k: int(v) for k, v in (x.split("=") for x in sys.argv[1:] if "=" in x)}   # e.g. tile_joints=672
J = len(par)
sk = hs.Skeleton(par, hsgen.inv_bind(ib_seed, J), **kw)
x = torch.empty((n, J, 3, 4), device="cuda")
assert hsgen.lib_cuda().hsg_cuda_local_poses(seed, type_, J, 0, n, x.data_ptr(),
                                             torch.cuda.current_stream().cuda_stream) == 0
g, s = torch.empty_like(x), torch.empty_like(x)
for _ in range(3):
    sk.scan_into(x, g, s, algo="tiles")
torch.cuda.synchronize()
print("F", sk.query("seq_tile_joints"), "tiles", sk.query("seq_tiles"))
