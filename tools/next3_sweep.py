#!/usr/bin/env python
"""NEXT-3 measurement: many skeleton types in one hs_scan_batch launch
vs one hs_scan per type, on crowds from a few hundred characters (launch fill/drain and
tail dominate) to bench size.  Each cell is checked bitwise against the per-type
launches; times are CUDA-event medians of 20 after 5 warm-ups."""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import hsgen  # noqa: E402
import paper_2505_06703_b200 as hs  # noqa: E402


def timed(fn, n=20):
    for _ in range(5):
        fn()
    ts = []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--types", type=int, default=8)
    ap.add_argument("--chars", default="64,512,4096,32768")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01d_next3_sweep.json"))
    args = ap.parse_args(argv)
    # 8 skeleton types: the templates plus SPEC random trees of 100-1000 joints
    pars = [hsgen.skeleton("hum32"), hsgen.skeleton("hum64"), hsgen.skeleton("chain256"),
            hsgen.skeleton("tree1024")]
    pars += [hsgen.random_tree(50 + i, J, d) for i, (J, d) in
             enumerate([(120, 15), (300, 40), (600, 90), (900, 30)])]
    pars = pars[:args.types]
    sks = [hs.Skeleton(p, hsgen.inv_bind(7, len(p))) for p in pars]
    rows = []
    for n in [int(c) for c in args.chars.split(",")]:
        items = []
        for i, (p, sk) in enumerate(zip(pars, sks)):
            x = torch.empty((n, len(p), 3, 4), device="cuda")
            assert hsgen.lib_cuda().hsg_cuda_local_poses(9, i, len(p), 0, n, x.data_ptr(),
                                                         torch.cuda.current_stream().cuda_stream) == 0
            items.append((sk, x, torch.empty_like(x), torch.empty_like(x)))
        ref = []
        for sk, x, g, s in items:
            sk.scan_into(x, g, s)
            ref.append((g.clone(), s.clone()))
        hs.scan_batch(items)
        torch.cuda.synchronize()
        same = all(torch.equal(g, rg) and torch.equal(s, rs) for (_, _, g, s), (rg, rs) in zip(items, ref))
        per_type = timed(lambda: [sk.scan_into(x, g, s) for sk, x, g, s in items])
        batch = timed(lambda: hs.scan_batch(items))
        joints = n * sum(len(p) for p in pars)
        row = {"chars_per_type": n, "types": len(pars), "joints": joints, "per_type_ms": per_type,
               "batch_ms": batch, "speedup": per_type / batch, "bitwise_equal": same}
        rows.append(row)
        print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in row.items()}),
              flush=True)
    json.dump({"experiment": "NEXT-3 heterogeneous single launch vs one launch per type, one B200",
               "skeletons": [len(p) for p in pars], "rows": rows}, open(args.out, "w"), indent=1)
    return 0


if __name__ == "__main__":
    sys.exit(main())
