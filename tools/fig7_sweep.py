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
MaxParentOutBlock walk), `compressed` (Alg. 4 literally, the paper's final algorithm:
7 serial in-block composes, 7 stride-8 composes, the MaxParentOutBlock walk),
`gateau` (Alg. 1), `leaf` (KIYA).  Skeletons: SPEC random_tree with 300
joints and max level = depth.  Timed with CUDA events (median of 20 after 5 warm-ups).
Correctness per cell without the oracle (tools may not use it): on the exact-arithmetic
family every algorithm must equal the chunked kernel bit for bit, and on the timed
rigid crowd stay within 2e-4 of it (each is within 1e-4 of the oracle in
tests/test_gpu_parity.py::test_fig7_shape_depth_sweep).
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

ALGOS = ["chunked", "doubling", "blocked", "compressed", "gateau", "leaf"]
NAMES = {"chunked": "chunked (this build)", "doubling": "Alg. 2 doubling", "blocked": "Alg. 3 blocked",
         "compressed": "Alg. 4 compressed (paper's final)", "gateau": "Gateau (Alg. 1)", "leaf": "KIYA leaf"}


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--chars", type=int, default=10_000)
    ap.add_argument("--joints", type=int, default=300)
    ap.add_argument("--depths", default="15,30,45,60,90,120")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02b_fig7_sweep.json"))
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
        # exact family: every algorithm bitwise equal to the chunked kernel
        xe = torch.from_numpy(hsgen.exact_poses(9, J, 64)).cuda()
        ge_ref, se_ref = sk.scan(xe)
        g_ref, s_ref = sk.scan(x)
        row = {"depth": depth, "mean_level": float(lev.mean()), "joints": J, "chars": args.chars,
               "chunked_program": {"chunking": sk.query("chunking"), "anchors": sk.query("anchors"),
                                   "anchor_rounds": sk.query("anchor_rounds")}}
        for algo in ALGOS:
            a = "auto" if algo == "chunked" else algo
            ge, se = sk.scan(xe, algo=a)
            sk.scan_into(x, g, s, algo=a)
            torch.cuda.synchronize()
            assert torch.equal(ge, ge_ref) and torch.equal(se, se_ref), (depth, algo, "exact family")
            err = max(float((g - g_ref).abs().max()), float((s - s_ref).abs().max()))
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
                         "hbm_gbs": 144 * J * args.chars / (ms / 1e3) / 1e9, "max_diff_vs_chunked": err}
            assert err <= 2e-4, (depth, algo, err)
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
                "3x4 fp32 poses, G and S written; every cell bitwise equal to the chunked kernel on the "
                "exact family.\n\n")
        f.write("| depth | mean level | " + " | ".join(NAMES[a] for a in ALGOS) + " |\n")
        f.write("|---" * (len(ALGOS) + 2) + "|\n")
        for r in rows:
            f.write(f"| {r['depth']} | {r['mean_level']:.1f} | " +
                    " | ".join(f"{r[a]['ms']:.3f}" for a in ALGOS) + " |\n")
        f.write("\nSpeed-up of the paper's final algorithm (Alg. 4) and of this build's kernel over the "
                "comparison systems (time ratio; > 1 = faster), the shape PAPER.md:268-270 describes:\n\n")
        f.write("| depth | Gateau / Alg. 4 | KIYA / Alg. 4 | Gateau / chunked | KIYA / chunked | Alg. 4 / chunked |\n")
        f.write("|---|---|---|---|---|---|\n")
        for r in rows:
            c, g4 = r["chunked"]["ms"], r["compressed"]["ms"]
            f.write(f"| {r['depth']} | {r['gateau']['ms'] / g4:.2f} | {r['leaf']['ms'] / g4:.2f} | "
                    f"{r['gateau']['ms'] / c:.2f} | {r['leaf']['ms'] / c:.2f} | {g4 / c:.2f} |\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())
