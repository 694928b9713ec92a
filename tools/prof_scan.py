#!/usr/bin/env python
"""Debug aid: per-phase cycle split (HS_DEBUG_PROF) of the chunked scan kernel on the
C5 skeletons at bench size."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hsgen  # noqa: E402
import paper_2505_06703_b200 as hs  # noqa: E402

# the phase-profile hooks are compiled out of the product build (they cost ~3 %)
hs.use_library(hs.build_variant("libhs_prof.so", ["-DHS_PROF_HOOKS=1"]))

for name, n, seed, type_, ib_seed in hsgen.CONFIGS[5]:
    par = hsgen.skeleton(name)
    J = len(par)
    sk = hs.Skeleton(par, hsgen.inv_bind(ib_seed, J))
    x = torch.empty((n, J, 3, 4), device="cuda")
    hsgen.lib_cuda().hsg_cuda_local_poses(seed, type_, J, 0, n, x.data_ptr(),
                                          torch.cuda.current_stream().cuda_stream)
    g, s = torch.empty_like(x), torch.empty_like(x)
    for _ in range(3):
        sk.scan_into(x, g, s)
    torch.cuda.synchronize()
    os.environ["HS_DEBUG_PROF"] = "1"
    sk.scan_into(x, g, s)
    torch.cuda.synchronize()
    del os.environ["HS_DEBUG_PROF"]
