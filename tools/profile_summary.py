"""Summarise a round's ncu captures (tools/round_artifacts.sh TAG -> gpurun_out/TAG/) into
profiles/: the launch list of the bench command (per-launch times, step shares), the
`--set full` summaries of the dominant launches, and profiles/ncu_traffic.json — the
DRAM bytes per launch bench.py reports as `roofline.traffic`, each entry tagged with the
library sources' hash the capture was taken on (bench.py reports it only on a match).

    python tools/profile_summary.py TAG [SOURCES_SHA]

SOURCES_SHA defaults to the current tree's `paper_2505_06703_b200.sources_sha256()`:
pass the hash the bench printed for the captured build when the tree changed since."""
from __future__ import annotations

import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
UNITS = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
        "launch__shared_mem_per_block_dynamic", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smsp__inst_executed.sum",
        "sm__cycles_elapsed.avg.per_second"]


def launches(csv_path, out_path, tag):
    recs, hdr = [], None
    for r in csv.reader(open(csv_path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                recs.append((int(d["ID"]), d["Kernel Name"],
                             float(d["Metric Value"].replace(",", "")) * UNITS[d["Metric Unit"]]))
    ours = [x for x in recs if "hs::" in x[1] or "chunked_kernel" in x[1] or "seq_kernel" in x[1]]
    with open(out_path, "w") as f:
        f.write(f"# Launch list ({tag}): ncu --metrics gpu__time_duration.sum --clock-control none -c 400\n")
        f.write("#   python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-configs   (C5, 1 GPU)\n")
        f.write("# Cold-cache, serialised launches: compare SHARES of the step, not absolutes.\n")
        f.write("# id  duration_us  kernel\n")
        for i, k, us in recs:
            f.write(f"{i:4d} {us:12.1f}  {k[:110]}\n")
        step = [x for x in ours if "chunked_kernel" in x[1]][-3:]   # the last timed step: 3 launches
        tot = sum(us for _, _, us in step)
        f.write("\n# last timed step (3 chunked_kernel launches: hum64, chain256, tree1024): share of the step\n")
        for (_, k, us), nm in zip(step, ["hum64", "chain256", "tree1024"]):
            f.write(f"#   {nm:9s} {us:9.1f} us  {100 * us / tot:5.1f}%\n")


def capture(rep, out_path, title, alg_bytes):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    res = {k: (v[h.index(k)], u[h.index(k)]) for k in KEYS if k in h}
    rd = float(res["dram__bytes_read.sum"][0]) * SCALE[res["dram__bytes_read.sum"][1]]
    wr = float(res["dram__bytes_write.sum"][0]) * SCALE[res["dram__bytes_write.sum"][1]]
    lines = [f"# {title}", f"# kernel: {v[h.index('Kernel Name')] if 'Kernel Name' in h else '?'}",
             f"# DRAM traffic per launch = {rd / 1e9:.3f} GB read + {wr / 1e9:.3f} GB write = {(rd + wr) / 1e9:.3f} GB",
             f"# algorithmic bytes = {alg_bytes / 1e9:.3f} GB  (traffic / algorithmic = {(rd + wr) / alg_bytes:.4f})", ""]
    lines += [f"{k:75s} {res[k][0]:>18s} {res[k][1]}" for k in KEYS if k in res]
    lines += ["", "# warp stall reasons (warps stalled per issued instruction)"]
    stalls = sorted(((h[i], float(v[i])) for i in range(len(h))
                     if "average_warps_issue_stalled" in h[i] and "per_issue_active" in h[i]), key=lambda z: -z[1])
    lines += [f"{k:75s} {x:8.3f}" for k, x in stalls if x > 0.01]
    open(out_path, "w").write("\n".join(lines) + "\n")
    return rd, wr


def main():
    tag = sys.argv[1]
    src = f"{ROOT}/gpurun_out/{tag}"
    import paper_2505_06703_b200 as hs
    sha = sys.argv[2] if len(sys.argv) > 2 else hs.sources_sha256()
    entries = []
    if os.path.exists(f"{src}/launches.csv"):
        launches(f"{src}/launches.csv", f"{ROOT}/profiles/{tag}_launches.txt", tag)
    if os.path.exists(f"{src}/prof_tree1024.ncu-rep"):
        alg = 333_333 * 1024 * 144
        rd, wr = capture(f"{src}/prof_tree1024.ncu-rep", f"{ROOT}/profiles/{tag}_ncu_tree1024.txt",
                         f"{tag}: ncu --set full, the C5 tree1024 launch (bench.py --profile)", alg)
        entries.append({"workload": "C5 1,000,000 mixed hum64/chain256/tree1024 per GPU",
                        "kernel": "chunked_kernel (tree1024 launch)", "dram_bytes_per_launch": rd + wr,
                        "dram_read": rd, "dram_write": wr, "algorithmic_bytes_per_launch": alg,
                        "source": f"profiles/{tag}_ncu_tree1024.txt", "sources_sha256": sha})
    if os.path.exists(f"{src}/prof_seq_c6.ncu-rep"):
        alg = 2000 * 16384 * 144
        rd, wr = capture(f"{src}/prof_seq_c6.ncu-rep", f"{ROOT}/profiles/{tag}_ncu_seq_c6.txt",
                         f"{tag}: ncu --set full, the C6 multi-tile launch (tools/tiles_one.py)", alg)
        entries.append({"workload": "C6 2,000 x tree16384 (L=1024, beyond one CTA: multi-tile path)",
                        "kernel": "seq_kernel (multi-tile path, tree16384 launch)", "dram_bytes_per_launch": rd + wr,
                        "dram_read": rd, "dram_write": wr, "algorithmic_bytes_per_launch": alg,
                        "source": f"profiles/{tag}_ncu_seq_c6.txt", "sources_sha256": sha})
    if os.path.exists(f"{src}/prof_seq_c7.ncu-rep"):
        alg = 2000 * 16384 * 144
        rd, wr = capture(f"{src}/prof_seq_c7.ncu-rep", f"{ROOT}/profiles/{tag}_ncu_seq_c7.txt",
                         f"{tag}: ncu --set full, the C7 multi-tile launch (tools/tiles_one.py --dfs)", alg)
        entries.append({"workload": "C7 2,000 x tree16384, depth-first labels (multi-tile path)",
                        "kernel": "seq_kernel (multi-tile path, tree16384dfs launch)", "dram_bytes_per_launch": rd + wr,
                        "dram_read": rd, "dram_write": wr, "algorithmic_bytes_per_launch": alg,
                        "source": f"profiles/{tag}_ncu_seq_c7.txt", "sources_sha256": sha})
    if os.path.exists(f"{src}/prof_stage1.ncu-rep"):
        capture(f"{src}/prof_stage1.ncu-rep", f"{ROOT}/profiles/{tag}_ncu_stage1_streaming_kernel.txt",
                f"{tag}: ncu --set full, stage1_kernel (two-pass hs_animate, tree1024 x 50,000, 2 layers; "
                "the captured launch is a full 1 GiB workspace batch: 21,845 characters)",
                21_845 * (1024 * 48 + 32))
    json.dump(entries, open(f"{ROOT}/profiles/ncu_traffic.json", "w"), indent=1)
    for e in entries:
        print(e["kernel"], e["dram_bytes_per_launch"] / e["algorithmic_bytes_per_launch"])


if __name__ == "__main__":
    main()
