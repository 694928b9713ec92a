#!/usr/bin/env python
"""Fig. 7-shaped depth sweep (Table 1).

The paper's only experiment: 10,000 characters x ~300 joints (3,000,000 joints per
frame), hierarchy depth swept 15 -> 120 layers, Hierarchy-Scan time of the paper's
method vs Gateau 2012 (Alg. 1, thread per joint walking every ancestor) and KIYA
2024 (thread per leaf filling its root path).  Fig. 7 itself is an image
placeholder in PAPER.md, so only its shape is reproducible: "when the number of
bone levels > 30, the performance of our solution is significantly better"
(PAPER.md:270).

Here, on one B200, every algorithm runs through the same C ABI (hs_scan_ex) on the
same seeded crowd: `chunked` (this build's kernel), `doubling` (Alg. 2 verbatim),
`blocked` (Alg. 3 literally: 64-joint blocks, clamped in-block doubling, then the
MaxParentOutBlock walk), `gateau` (Alg. 1), `leaf` (KIYA).  Skeletons: SPEC random_tree with
300 joints and max level = depth.  Each cell is checked against the fp64 oracle on
sampled characters, then timed with CUDA events (median of 20 after 5 warm-ups).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import hsgen  # noqa: E402
import oracle  # noqa: E402

ALGOS = ["chunked", "doubling", "blocked", "gateau", "leaf"]


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--chars", type=int, default=10_000)
    ap.add_argument("--joints", type=int, default=300)
    ap.add_argument("--depths", default="15,30,45,60,90,120")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01h_fig7_sweep.json"))
    args = ap.parse_args(argv)

    import torch
    import paper_2505_06703_b200 as hs

    rows = []
    for depth in [int(x) for x in args.depths.split(",")]:
        par = hsgen.random_tree(100 + depth, args.joints, depth)
        J = len(par)
        lev = np.zeros(J, int)
        for i in range(J):
            lev[i] = 1 if par[i] < 0 else lev[par[i]] + 1
        local = hsgen.local_poses(7, J, args.chars)
        ib = hsgen.inv_bind(7, J)
        x = torch.from_numpy(local).cuda()
        g = torch.empty_like(x)
        s = torch.empty_like(x)
        sk = hs.Skeleton(par, ib)
        idx = np.linspace(0, args.chars - 1, 16).astype(int)
        G, S = oracle.scan(par, local[idx], ib)
        row = {"depth": depth, "mean_level": float(lev.mean()), "joints": J, "chars": args.chars,
               "chunked_program": {"chunking": sk.query("chunking"), "anchors": sk.query("anchors"),
                                   "anchor_rounds": sk.query("anchor_rounds")}}
        for algo in ALGOS:
            a = "auto" if algo == "chunked" else algo
            sk.scan_into(x, g, s, algo=a)
            torch.cuda.synchronize()
            err = max(float(np.abs(g[idx].cpu().numpy() - G).max()),
                      float(np.abs(s[idx].cpu().numpy() - S).max()))
            for _ in range(5):
                sk.scan_into(x, g, s, algo=a)
            times = []
            for _ in range(args.iters):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                sk.scan_into(x, g, s, algo=a)
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1))
            ms = statistics.median(times)
            row[algo] = {"ms": ms, "joints_per_s": J * args.chars / (ms / 1e3),
                         "hbm_gbs": 144 * J * args.chars / (ms / 1e3) / 1e9, "max_err": err}
            assert err <= 1e-4, (depth, algo, err)
        rows.append(row)
        print(json.dumps({"depth": depth, "mean_level": round(row["mean_level"], 1),
                          **{al: round(row[al]["ms"], 4) for al in ALGOS}}), flush=True)
        sk.close()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump({"experiment": "Fig. 7 shape (PAPER.md:253-270), one B200",
               "workload": f"{args.chars} characters x {args.joints}-joint SPEC random_tree, depth swept",
               "timing": f"CUDA events, median of {args.iters} after 5 warm-ups; ms per frame (one launch)",
               "rows": rows}, open(args.out, "w"), indent=1)
    # markdown table next to the json
    with open(args.out.replace(".json", ".md"), "w") as f:
        f.write("# Fig. 7-shaped depth sweep on one B200 (ms per frame; lower is better)\n\n")
        f.write(f"{args.chars} characters x {args.joints} joints (SPEC random_tree, max level = depth), "
                "3x4 fp32 poses, G and S written; oracle parity checked per cell.\n\n")
        f.write("| depth | mean level | chunked (this build) | Alg. 2 doubling | Alg. 3 blocked | Gateau (Alg. 1) | KIYA leaf |\n")
        f.write("|---|---|---|---|---|---|---|\n")
        for r in rows:
            f.write(f"| {r['depth']} | {r['mean_level']:.1f} | " +
                    " | ".join(f"{r[a]['ms']:.3f}" for a in ALGOS) + " |\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())
