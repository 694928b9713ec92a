#!/usr/bin/env python
"""Tuning aid: host-buffer pipeline over C5's types, per-type hs_scan_host calls vs one
hs_scan_host_batch (1/8 sample, pinned buffers, wall clock over 3 steps)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hsgen  # noqa: E402
import paper_2505_06703_b200 as hs  # noqa: E402

items, joints = [], 0
for name, n, seed, type_, ib_seed in hsgen.CONFIGS[5]:
    par = hsgen.skeleton(name)
    J = len(par)
    m = n // 8
    hl = torch.from_numpy(hsgen.local_poses(seed, J, m, type_=type_)).pin_memory()
    items.append((hs.Skeleton(par, hsgen.inv_bind(ib_seed, J)), hl, torch.empty_like(hl).pin_memory(),
                  torch.empty_like(hl).pin_memory()))
    joints += m * J
for batch_mb in (256, 64):
    pl = hs.Pipeline(batch_bytes=batch_mb << 20)
    for label, fn in (("per-type", lambda: [pl.scan_host(*it) for it in items]),
                      ("batch", lambda: pl.scan_host_batch(items))):
        fn()
        t0 = time.perf_counter()
        for _ in range(3):
            fn()
        dt = (time.perf_counter() - t0) / 3
        print(f"{batch_mb} MiB {label}: {joints / dt / 1e8:.2f}e8 joints/s", flush=True)
    pl.close()
