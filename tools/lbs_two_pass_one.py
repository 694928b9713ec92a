#!/usr/bin/env python
"""Profiling target: hs_scan_skin two-pass on hum64 (100k characters, 1000-vertex mesh):
the joint-sorted lbs_kernel, small enough for ncu --set full."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hsgen  # noqa: E402
import paper_2505_06703_b200 as hs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
par = hsgen.skeleton("hum64")
sk = hs.Skeleton(par, hsgen.inv_bind(2, 64))
mesh = hs.Mesh(sk, *hsgen.mesh(200, par, 1000))
x = torch.from_numpy(hsgen.local_poses(5, 64, n)).cuda()
g, s = torch.empty_like(x), torch.empty_like(x)
v = torch.empty((n, 1000, 3), device="cuda")
for _ in range(4):
    hs.scan_skin(sk, mesh, x, g, s, v, mode="two_pass")
torch.cuda.synchronize()
print("ok", n)
