#!/bin/bash
# usage: sweep.sh "label|args" ...
for spec in "$@"; do
  label="${spec%%|*}"; args="${spec#*|}"
  timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-check $args > gpurun_out/sw_$label.log 2>&1
  python - "$label" <<'PY'
import json,sys
lab=sys.argv[1]
try:
    d=json.loads(open(f"gpurun_out/sw_{lab}.log").read().strip().splitlines()[-1])
    c=d["config"]
    print(lab, round(d["value"]/1e9,2), {k:round(v,3) for k,v in c["per_launch_ms"].items()}, c.get("stages"), c.get("sbufs"), c.get("pbufs"), round(d["roofline"]["frac"],3), d["clocks"]["sm_mhz"])
except Exception as e:
    print(lab, "FAILED", open(f"gpurun_out/sw_{lab}.log").read()[-800:])
PY
done
