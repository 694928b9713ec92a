#!/usr/bin/env python
"""Tuning aid: is a character's result independent of the tile size (characters per
CTA tile)?  Bitwise comparison of hs_scan across tile_joints, per C5 skeleton."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch, numpy as np, hsgen
import paper_2505_06703_b200 as hs
for name in ("hum32", "hum64", "chain256", "tree1024"):
    par = hsgen.skeleton(name); J = len(par)
    x = torch.from_numpy(hsgen.local_poses(3, J, 300)).cuda()
    ref = None; out = {}
    for tj in (0, 64, 128, 256, 512, 2048):
        sk = hs.Skeleton(par, hsgen.inv_bind(3, J), tile_joints=tj)
        g, s = sk.scan(x)
        torch.cuda.synchronize()
        if ref is None: ref = (g, s)
        out[f"{tj}(C={sk.query('tile_chars')},ch={sk.query('chunking')})"] = bool(torch.equal(g, ref[0]) and torch.equal(s, ref[1]))
    print(name, out, flush=True)
