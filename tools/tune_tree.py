#!/usr/bin/env python
"""Tuning aid: tree1024 at C5 size under the chunked kernel's stage / S-buffer /
anchor-buffer / chunking options (CUDA-event median of 10)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hsgen  # noqa: E402
import paper_2505_06703_b200 as hs  # noqa: E402

n = 333_333
par = hsgen.skeleton("tree1024")
J = len(par)
x = torch.empty((n, J, 3, 4), device="cuda")
hsgen.lib_cuda().hsg_cuda_local_poses(5, 2, J, 0, n, x.data_ptr(), torch.cuda.current_stream().cuda_stream)
g, s = torch.empty_like(x), torch.empty_like(x)


def timed(fn):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return round(statistics.median(ts), 3)


for opts in [{}, dict(stages=2, sbufs=2), dict(stages=2, sbufs=1), dict(stages=3, sbufs=1, pbuf=1),
             dict(stages=3, sbufs=2, pbuf=1), dict(chunking=2), dict(chunking=1)]:
    try:
        sk = hs.Skeleton(par, hsgen.inv_bind(4, J), **opts)
        q = {k: sk.query(k) for k in ("stages", "sbufs", "pbufs", "chunking", "smem_bytes")}
        print(opts, q, timed(lambda: sk.scan_into(x, g, s)), flush=True)
    except hs.HSError as e:
        print(opts, "ERR", e, flush=True)
