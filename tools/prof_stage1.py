#!/usr/bin/env python
"""Debug aid: per-phase cycle split (HS_DEBUG_PROF) of the chunked kernel with and
without the fused Stage 1, on each C5 skeleton at bench size."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import hsgen  # noqa: E402
import paper_2505_06703_b200 as hs  # noqa: E402

# the phase-profile hooks are compiled out of the product build (they cost ~3 %)
hs.use_library(hs.build_variant("libhs_prof.so", ["-DHS_PROF_HOOKS=1"]))

n = int(sys.argv[1]) if len(sys.argv) > 1 else 333_333
for name in sys.argv[2:] or ["hum64", "chain256", "tree1024"]:
    par = hsgen.skeleton(name)
    J = len(par)
    ib = hsgen.inv_bind(2, J)
    sk = hs.Skeleton(par, ib)
    keys = hsgen.clips(100, J, 8, 31)
    cs = hs.ClipSet(sk, keys, 30.0, 1)
    lay = hsgen.layers(5, n, 2, 8, 1.5)
    layers = torch.from_numpy(lay.view(np.int32).reshape(n, 2, 4)).cuda()
    g = torch.empty((n, J, 3, 4), device="cuda")
    s = torch.empty_like(g)
    x = torch.from_numpy(hsgen.local_poses(5, J, n)).cuda()
    for _ in range(2):
        hs.animate(sk, cs, layers, g, s)
        sk.scan_into(x, g, s)
    torch.cuda.synchronize()
    os.environ["HS_DEBUG_PROF"] = "1"
    print(name, "stage1:", flush=True)
    hs.animate(sk, cs, layers, g, s)
    torch.cuda.synchronize()
    print(name, "scan only:", flush=True)
    sk.scan_into(x, g, s)
    torch.cuda.synchronize()
    del os.environ["HS_DEBUG_PROF"]
