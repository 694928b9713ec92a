"""Debug aid: create each config's skeleton with both chunked kernels and run a tiny scan."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np, hsgen, paper_2505_06703_b200 as hs
for name in ["hum32", "hum64", "chain256", "tree1024"]:
    for kern in (1, 2):
        par = hsgen.skeleton(name)
        try:
            sk = hs.Skeleton(par, kernel=kern)
            print(name, kern, {q: sk.query(q) for q in ["threads", "smem_bytes", "stages", "sbufs", "pbufs",
                                                       "tile_chars", "anchors", "ib_placement"]})
            x = torch.zeros((50, len(par), 3, 4), device="cuda")
            x[..., 0, 0] = 1; x[..., 1, 1] = 1; x[..., 2, 2] = 1
            g, s = sk.scan(x); torch.cuda.synchronize(); print("  ok", bool((g == x).all()))
        except Exception as e:
            print("  ERR", e)
