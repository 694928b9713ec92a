#!/usr/bin/env python
"""Print the key fields of bench.py JSON lines (one file per argument)."""
import json
import sys

for f in sys.argv[1:]:
    for ln in open(f):
        ln = ln.strip()
        if not ln.startswith("{"):
            continue
        d = json.loads(ln)
        if "value" not in d:
            print(f, d)
            continue
        r = d.get("roofline") or {}
        p = d.get("parity") or {}
        print(f"{f}: {d['value'] / 1e9:.2f} G{d['unit']} ms/step {d['ms_per_step']:.3f} "
              f"frac {r.get('frac', 0):.3f} ({r.get('achieved', 0):.0f} GB/s) "
              f"per_launch {d['config'].get('per_launch_ms')} worst {p.get('worst')} "
              f"e2e {(d.get('e2e') or {}).get('value')} clocks {d.get('clocks')}")
