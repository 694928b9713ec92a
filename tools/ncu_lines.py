#!/usr/bin/env python
"""Per-source-line warp-stall summary of an ncu report (needs -lineinfo):
python tools/ncu_lines.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


fname, agg, tot = "?", [], 0.0
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or not r or not r[0].isdigit():
        continue
    ci = hdr.index("Warp Stall Sampling (All Samples)")
    ie = hdr.index("Instructions Executed")
    st = collections.Counter()
    for k, name in enumerate(hdr):
        if name.startswith("stall_") and "(Not" not in name:
            v = num(r[k])
            if v:
                st[name[6:]] += v
    s = num(r[ci])
    tot += s
    agg.append((s, fname, int(r[0]), r[1][:70], num(r[ie]), st))
print(f"total samples {tot:.0f}")
for s, f, ln, src, ins, st in sorted(agg, key=lambda x: -x[0])[:top]:
    print(f"{s / tot * 100:5.1f}% {f}:{ln:<5d} inst {ins:9.3g}  {src:70s} {st.most_common(2)}")
