#!/usr/bin/env python
"""ncu target: hs_scan_varied on 20,000 per-character 1024-joint random trees (depth 300,
shuffled labels) — the C4-sized NEXT-3 case of tools/time_varied.py; three launches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import hsgen  # noqa: E402
import paper_2505_06703_b200 as hs  # noqa: E402

J, n, depth = 1024, 20_000, 300
rng = np.random.default_rng(1)
pars = np.stack([hsgen.relabel(hsgen.random_tree(int(rng.integers(1 << 30)), J, depth),
                               rng.permutation(J).astype(np.int32))[0] for _ in range(64)])
p = torch.from_numpy(pars[np.arange(n) % 64]).cuda()
x = torch.empty((n, J, 3, 4), device="cuda")
hsgen.lib_cuda().hsg_cuda_local_poses(7, 0, J, 0, n, x.data_ptr(), torch.cuda.current_stream().cuda_stream)
ib = torch.empty_like(x)
hsgen.lib_cuda().hsg_cuda_local_poses(8, 0, J, 0, n, ib.data_ptr(), torch.cuda.current_stream().cuda_stream)
g, s = torch.empty_like(x), torch.empty_like(x)
for _ in range(3):
    hs.scan_varied(p, x, ib, g, s)
torch.cuda.synchronize()
print("ok")
