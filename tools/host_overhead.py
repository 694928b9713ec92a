#!/usr/bin/env python
"""Tuning aid: host-side cost per hs_scan_ex call (enqueue only, fewer calls than the
launch queue holds) through ctypes, against a bare ctypes call, for a tiny crowd."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hsgen  # noqa: E402
import paper_2505_06703_b200 as hs  # noqa: E402

L = hs.lib()
for name in ("hum64", "tree1024"):
    par = hsgen.skeleton(name)
    J = len(par)
    sk = hs.Skeleton(par, hsgen.inv_bind(2, J))
    x = torch.from_numpy(hsgen.local_poses(1, J, 4)).cuda()
    g, s = torch.empty_like(x), torch.empty_like(x)
    st = torch.cuda.current_stream().cuda_stream
    opts = hs._ScanOpts(0, -1, 0)
    args = (sk.handle, x.data_ptr(), 1, g.data_ptr(), s.data_ptr(), st, ctypes.byref(opts))
    for reps in (1, 2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(200):
            L.hs_scan_ex(*args)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        for _ in range(200):
            L.hs_last_error()
        t3 = time.perf_counter()
        print(f"{name}: hs_scan_ex host {1e6 * (t1 - t0) / 200:.2f} us/call, bare ctypes "
              f"{1e6 * (t3 - t2) / 200:.2f} us/call", flush=True)
