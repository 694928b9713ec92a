"""Summarise a round's ncu captures into profiles/ (launch list + full capture of the
dominant kernel) and refresh profiles/ncu_traffic.json for bench.py's roofline."""
from __future__ import annotations

import csv
import json
import subprocess
import sys

LAUNCH_ROLES = ["gen hum64", "gen chain256", "gen tree1024", "scan hum64 (check step)",
                "scan chain256 (check step)", "scan tree1024 (check step)", "scan hum64 (timed step)",
                "scan chain256 (timed step)", "scan tree1024 (timed step)"]
UNITS = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}


def launches(csv_path, out_path, tag):
    rows = list(csv.reader(open(csv_path)))
    hdr, recs = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                recs.append((int(d["ID"]), d["Kernel Name"],
                             float(d["Metric Value"].replace(",", "")) * UNITS[d["Metric Unit"]]))
    with open(out_path, "w") as f:
        f.write(f"# Launch list ({tag}): ncu --metrics gpu__time_duration.sum --clock-control none\n")
        f.write("#   python bench.py --profile --steps 1 --warmup 0   (config C5, 1 GPU)\n")
        f.write("# Cold-cache, serialised launches: compare SHARES, not absolutes.\n")
        f.write("# id  duration_us  role  kernel\n")
        for (i, k, us), nm in zip(recs, LAUNCH_ROLES):
            f.write(f"{i:3d} {us:12.1f}  {nm:28s} {k}\n")
        step = [us for (_, _, us) in recs[6:9]]
        f.write("\n# timed step (3 chunked_kernel launches): share of step time\n")
        for nm, us in zip(["hum64", "chain256", "tree1024"], step):
            f.write(f"#   {nm:9s} {us:9.1f} us  {100 * us / sum(step):5.1f}%\n")
    return recs


def full_capture(rep, out_path, tag, n_joints, workload):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__block_size", "launch__grid_size", "launch__shared_mem_per_block_dynamic",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
            "sm__cycles_elapsed.avg.per_second"]
    res = {}
    for i, k in enumerate(h):
        if k in want or ("average_warps_issue_stalled" in k and "per_issue_active" in k):
            res[k] = (v[i], u[i])
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
    rd = float(res["dram__bytes_read.sum"][0]) * scale[res["dram__bytes_read.sum"][1]]
    wr = float(res["dram__bytes_write.sum"][0]) * scale[res["dram__bytes_write.sum"][1]]
    alg = n_joints * 144
    lines = [f"# {tag}: ncu --set full --clock-control none --import-source on -k regex:chunked_kernel -s 2 -c 1",
             "#   python bench.py --profile --steps 1 --warmup 0   (the C5 tree1024 launch)",
             f"# DRAM traffic per launch = {rd / 1e9:.3f} GB read + {wr / 1e9:.3f} GB write = {(rd + wr) / 1e9:.3f} GB",
             f"# algorithmic bytes (144 B/joint x {n_joints / 1e6:.2f} M joints) = {alg / 1e9:.3f} GB"
             f"  (ratio {(rd + wr) / alg:.4f})", ""]
    for k in want:
        if k in res:
            lines.append(f"{k:75s} {res[k][0]:>18s} {res[k][1]}")
    lines += ["", "# warp stall reasons (warps stalled per issued instruction)"]
    stalls = sorted(((k, float(res[k][0])) for k in res if "stalled" in k), key=lambda z: -z[1])
    lines += [f"{k:75s} {x:8.3f}" for k, x in stalls if x > 0.01]
    open(out_path, "w").write("\n".join(lines) + "\n")
    json.dump({"workload": workload, "kernel": "chunked_kernel (tree1024 launch)",
               "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
               "algorithmic_bytes_per_launch": alg, "source": f"{out_path} (ncu --set full, {tag})"},
              open("profiles/ncu_traffic.json", "w"), indent=1)


def kernel_summary(rep, out_path, title, alg_bytes):
    """Key counters of one captured launch (no ncu_traffic.json update)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "lts__t_sectors_srcunit_tex_op_read.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__shared_mem_per_block_dynamic", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smsp__inst_executed.sum"]
    lines = [f"# {title}", f"# algorithmic HBM bytes per launch: {alg_bytes / 1e9:.3f} GB", ""]
    for k in keys:
        if k in h:
            i = h.index(k)
            lines.append(f"{k:75s} {v[i]:>18s} {u[i]}")
    stalls = sorted(((h[i], float(v[i])) for i in range(len(h))
                     if "average_warps_issue_stalled" in h[i] and "per_issue_active" in h[i]),
                    key=lambda z: -z[1])
    lines += ["", "# warp stall reasons (warps stalled per issued instruction)"]
    lines += [f"{k:75s} {x:8.3f}" for k, x in stalls if x > 0.01]
    open(out_path, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    tag = sys.argv[1]
    if len(sys.argv) > 2 and sys.argv[2] == "stage1":
        kernel_summary(f"gpurun_out/prof_stage1_{tag}.ncu-rep", f"profiles/{tag}_ncu_stage1_tree1024.txt",
                       f"{tag}: ncu --set full, hs_animate tree1024 x 50,000 characters, 2 layers "
                       "(tools/stage1_one.py, 3rd launch)", 50_000 * (1024 * 96 + 32))
        sys.exit(0)
    if len(sys.argv) > 2 and sys.argv[2] == "lbs":
        kernel_summary(f"gpurun_out/prof_lbs_{tag}.ncu-rep", f"profiles/{tag}_ncu_lbs_tree1024.txt",
                       f"{tag}: ncu --set full, hs_scan_skin tree1024 x 20,000 characters, 1000-vertex "
                       "mesh (tools/lbs_one.py, 3rd launch)", 20_000 * (1024 * 144 + 1000 * 12))
        sys.exit(0)
    launches(f"gpurun_out/launches_{tag}.csv", f"profiles/{tag}_launches.txt", tag)
    full_capture(f"gpurun_out/prof_tree_{tag}.ncu-rep", f"profiles/{tag}_ncu_tree1024.txt", tag,
                 333333 * 1024, "C5 1,000,000 mixed hum64/chain256/tree1024 per GPU")
    print(open(f"profiles/{tag}_launches.txt").read())
    print(open(f"profiles/{tag}_ncu_tree1024.txt").read())
