import os, sys, statistics
sys.path.insert(0, os.getcwd())
import numpy as np, torch, hsgen
import paper_2505_06703_b200 as hs
n = 333_333
for name in ["hum64", "chain256", "tree1024"]:
    par = hsgen.skeleton(name); J = len(par)
    lay = hsgen.layers(5, n, 2, 8, 1.5)
    layers = torch.from_numpy(lay.view(np.int32).reshape(n, 2, 4)).cuda()
    g = torch.empty((n, J, 3, 4), device="cuda"); s = torch.empty_like(g)
    res = {}
    for K in (3, 5, 7):
        try:
            sk = hs.Skeleton(par, hsgen.inv_bind(2, J), chunk=K)
        except Exception as e:
            res[K] = str(e)[:40]; continue
        cs = hs.ClipSet(sk, hsgen.clips(100, J, 8, 31), 30.0, 1)
        for mode in ("fused", "two_pass"):
            if mode == "fused" and sk.query("path") != 1:
                res[f"K{K} fused"] = "multi-CTA"; continue
            for _ in range(2): hs.animate(sk, cs, layers, g, s, mode=mode)
            ts = []
            for _ in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); hs.animate(sk, cs, layers, g, s, mode=mode); b.record(); torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            res[f"K{K} {mode}"] = round(statistics.median(ts), 3)
    print(name, res, flush=True)
