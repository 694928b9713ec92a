#!/bin/bash
# usage (on the GPU box, from the repo root): tools/round_artifacts.sh TAG -> gpurun_out/TAG/
# The round's evidence set: the GPU test log; the bench lines (default C5 with the
# per-config object, C6 multi-tile, Stage 1, LBS, the whole pipeline, the reference
# arm); the Fig. 7 sweep, the HBM speed-of-light probe, the NEXT-3 timing; then, after
# the bench command exited 0 without ncu, the ncu launch list of that command and
# --set full captures of the dominant launches.
tag=${1:?tag}
out=gpurun_out/$tag
mkdir -p "$out"
python -c "import __graft_entry__ as g; g.build()" > "$out/build.log" 2>&1 || { echo "build failed"; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu -rA > "$out/pytest_gpu.log" 2>&1; echo "pytest rc=$?"
tail -1 "$out/pytest_gpu.log"
python bench.py > "$out/bench_c5.json" 2> "$out/bench_c5.err"; echo "bench rc=$?"
python bench.py --config 6 > "$out/bench_c6.json" 2> "$out/bench_c6.err"; echo "bench c6 rc=$?"
python bench.py --config 7 > "$out/bench_c7.json" 2> "$out/bench_c7.err"; echo "bench c7 rc=$?"
python bench.py --stage1 > "$out/bench_c5_stage1.json" 2> "$out/bench_c5_stage1.err"; echo "stage1 rc=$?"
python bench.py --skin-mesh 1000 --no-e2e > "$out/bench_c5_lbs1000.json" 2> "$out/bench_c5_lbs1000.err"; echo "lbs rc=$?"
python bench.py --stage1 --skin-mesh 1000 > "$out/bench_c5_pipeline.json" 2> "$out/bench_c5_pipeline.err"; echo "pipeline rc=$?"
python bench.py --impl reference --steps 3 --warmup 3 > "$out/bench_reference.json" 2> "$out/bench_reference.err"; echo "reference rc=$?"
python tools/fig7_sweep.py --out "$out/fig7_sweep.json" > "$out/fig7.log" 2>&1; echo "fig7 rc=$?"
python tools/sol_stream.py --out "$out/sol_stream.json" > "$out/sol_stream.log" 2>&1; echo "sol rc=$?"
python tools/time_varied.py > "$out/time_varied.log" 2>&1; echo "varied rc=$?"
if python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-configs > "$out/bench_short.json" 2>&1; then
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file "$out/launches.csv" \
      python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-configs > "$out/ncu_launches.log" 2>&1; echo "ncu list rc=$?"
fi
# --set full of the dominant C5 launch (tree1024: the 3rd chunked launch of the profile pass)
ncu --set full --clock-control none --import-source on -k regex:chunked_kernel -s 5 -c 1 \
    -o "$out/prof_tree1024" -f python bench.py --profile --steps 1 --warmup 1 > "$out/ncu_tree.log" 2>&1; echo "ncu tree rc=$?"
ncu --set full --clock-control none --import-source on -k regex:seq_kernel -s 2 -c 1 \
    -o "$out/prof_seq_c6" -f python tools/tiles_one.py > "$out/ncu_seq.log" 2>&1; echo "ncu seq rc=$?"
ncu --set full --clock-control none --import-source on -k regex:seq_kernel -s 2 -c 1 \
    -o "$out/prof_seq_c7" -f python tools/tiles_one.py --dfs > "$out/ncu_seq7.log" 2>&1; echo "ncu seq7 rc=$?"
HS_ANIMATE_MODE=two_pass ncu --set full --clock-control none --import-source on -k regex:stage1_kernel -s 3 -c 1 \
    -o "$out/prof_stage1" -f python tools/stage1_one.py > "$out/ncu_stage1.log" 2>&1; echo "ncu stage1 rc=$?"
