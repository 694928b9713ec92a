#!/usr/bin/env python
"""ncu target: three HS_ALGO_TILES launches on C6 (2,000 x tree16384, L = 1024; --dfs:
C7, the same trees in depth-first labels);
capture the third with  ncu -k regex:seq_kernel -s 2 -c 1 ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hsgen  # noqa: E402
import paper_2505_06703_b200 as hs  # noqa: E402

(name, n, seed, type_, ib_seed), = hsgen.CONFIGS[7 if "--dfs" in sys.argv else 6]   # --dfs: C7
par = hsgen.skeleton(name)
J = len(par)
sk = hs.Skeleton(par, hsgen.inv_bind(ib_seed, J))
x = torch.empty((n, J, 3, 4), device="cuda")
assert hsgen.lib_cuda().hsg_cuda_local_poses(seed, type_, J, 0, n, x.data_ptr(),
                                             torch.cuda.current_stream().cuda_stream) == 0
g, s = torch.empty_like(x), torch.empty_like(x)
for _ in range(3):
    sk.scan_into(x, g, s, algo="tiles")
torch.cuda.synchronize()
print("ok", sk.query("seq_tiles"), sk.query("seq_tile_joints"), sk.query("seq_exports"))
