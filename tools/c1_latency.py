#!/usr/bin/env python
"""Tuning aid: C1 (1,000 x hum32, launch-latency config) GPU time per launch from a
CUDA graph, vs the tile size (characters per CTA tile)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hsgen  # noqa: E402
import paper_2505_06703_b200 as hs  # noqa: E402

par = hsgen.skeleton("hum32")
J = len(par)
for n in (1000, 100, 10000):
    x = torch.from_numpy(hsgen.local_poses(1, J, n)).cuda()
    g, s = torch.empty_like(x), torch.empty_like(x)
    res = {}
    for tj in (0, 64, 128, 256, 512, 1024):   # 0 = the default (small-crowd program per call)
        sk = hs.Skeleton(par, hsgen.inv_bind(1, J), tile_joints=tj)
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            sk.scan_into(x, g, s, stream=st)
            st.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=st):
                for _ in range(20):
                    sk.scan_into(x, g, s, stream=st)
        for _ in range(3):
            gr.replay()
        ts = []
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            gr.replay()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1000 / 20)
        res[f"{tj} (C={sk.query('tile_chars')})"] = round(statistics.median(ts), 2)
    print(f"hum32 x {n}: us per launch", res, flush=True)
