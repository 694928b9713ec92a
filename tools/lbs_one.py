#!/usr/bin/env python
"""Profiling target: a few hs_scan_skin launches (tree1024 by default, 20k characters,
1000-vertex mesh) — small enough to run under ncu --set full."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hsgen  # noqa: E402
import paper_2505_06703_b200 as hs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "tree1024"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20_000
par = hsgen.skeleton(name)
J = len(par)
sk = hs.Skeleton(par, hsgen.inv_bind(4, J))
mesh = hs.Mesh(sk, *hsgen.mesh(202, par, 1000, type_=2))
x = torch.from_numpy(hsgen.local_poses(5, J, n, type_=2)).cuda()
g, s = torch.empty_like(x), torch.empty_like(x)
v = torch.empty((n, 1000, 3), device="cuda")
mode = os.environ.get("HS_SKIN_MODE", "auto")
for _ in range(4):
    hs.scan_skin(sk, mesh, x, g, s, v, mode=mode)
torch.cuda.synchronize()
print("ok", name, n)
