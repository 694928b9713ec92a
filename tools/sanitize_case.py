"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck / synccheck):
every chunked variant, the split path and the comparison kernels on a few characters."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import hsgen
import oracle
import paper_2505_06703_b200 as hs

cases = [("hum64", {}, "auto"), ("chain256", {}, "auto"), ("tree1024", {}, "auto"),
         ("tree1024", {"chunking": 2}, "auto"), ("hum32", {"pbuf": 1}, "auto"),
         ("tree1024", {"force_split": True}, "auto"), ("hum64", {}, "doubling"),
         ("hum64", {}, "gateau"), ("hum64", {}, "leaf")]
for name, create, algo in cases:
    par = hsgen.skeleton(name)
    J = len(par)
    n = 5
    local = hsgen.exact_poses(3, J, n)
    ib = hsgen.exact_inv_bind(3, J)
    sk = hs.Skeleton(par, ib, **create)
    g, s = sk.scan(torch.from_numpy(local).cuda(), algo=algo)
    torch.cuda.synchronize()
    G, S = oracle.scan(par, local, ib)
    ok = np.array_equal(g.cpu().numpy(), G) and np.array_equal(s.cpu().numpy(), S)
    print(name, create, algo, "ok" if ok else "MISMATCH")
    assert ok
    sk.close()
print("all sanitizer cases passed")
