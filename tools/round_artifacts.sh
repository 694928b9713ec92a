#!/bin/bash
# usage (on the GPU box): tools/round_artifacts.sh TAG  -> gpurun_out/TAG/
# The round's evidence set: GPU test log, the bench lines (scan, LBS, whole pipeline,
# Stage 1), then the ncu launch list of the bench command (after it exited 0 without ncu).
tag=${1:?tag}
out=gpurun_out/$tag
mkdir -p "$out"
python -m pytest tests -q -m gpu -rA > "$out/pytest_gpu.log" 2>&1; echo "pytest rc=$?"
tail -1 "$out/pytest_gpu.log"
python bench.py > "$out/bench_c5.json" 2> "$out/bench_c5.err"; echo "bench rc=$?"
python bench.py --stage1 > "$out/bench_c5_stage1.json" 2> "$out/bench_c5_stage1.err"; echo "stage1 rc=$?"
python bench.py --skin-mesh 1000 --no-e2e > "$out/bench_c5_lbs1000.json" 2> "$out/bench_c5_lbs1000.err"; echo "lbs rc=$?"
python bench.py --stage1 --skin-mesh 1000 > "$out/bench_c5_pipeline.json" 2> "$out/bench_c5_pipeline.err"; echo "pipeline rc=$?"
python bench.py --impl reference --steps 3 --warmup 3 > "$out/bench_reference.json" 2> "$out/bench_reference.err"; echo "reference rc=$?"
if python bench.py --steps 2 --warmup 1 > "$out/bench_short.json" 2>&1; then
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file "$out/launches.csv" \
      python bench.py --steps 2 --warmup 1 > "$out/ncu.log" 2>&1; echo "ncu rc=$?"
fi
