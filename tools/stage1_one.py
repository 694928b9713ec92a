#!/usr/bin/env python
"""Profiling target: a few hs_animate launches on one skeleton (default tree1024, 50k
characters, 2 layers) — small enough to run under ncu --set full.  HS_ANIMATE_MODE =
fused (default) | two_pass."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import hsgen  # noqa: E402
import paper_2505_06703_b200 as hs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "tree1024"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 50_000
par = hsgen.skeleton(name)
J = len(par)
sk = hs.Skeleton(par, hsgen.inv_bind(4, J))
cs = hs.ClipSet(sk, hsgen.clips(102, J, 8, 31, type_=2), 30.0, 1)
lay = hsgen.layers(5, n, 2, 8, 1.5, type_=2)
layers = torch.from_numpy(lay.view(np.int32).reshape(n, 2, 4)).cuda()
g = torch.empty((n, J, 3, 4), device="cuda")
s = torch.empty_like(g)
mode = os.environ.get("HS_ANIMATE_MODE", "fused")
for _ in range(4):
    hs.animate(sk, cs, layers, g, s, mode=mode)
torch.cuda.synchronize()
print("ok", name, n)
