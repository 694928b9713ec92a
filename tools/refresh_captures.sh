#!/bin/bash
# usage (on the GPU box): tools/refresh_captures.sh TAG -> gpurun_out/TAG/
# After a library change that leaves the hot kernels alone: the GPU test log, the NEXT-3
# timing, the default bench line and fresh --set full captures of the dominant launches
# (so profiles/ncu_traffic.json matches the committed sources).
tag=${1:?tag}
out=gpurun_out/$tag
mkdir -p "$out"
python -c "import __graft_entry__ as g; g.build()" > "$out/build.log" 2>&1 || { echo "build failed"; exit 1; }
if [ -z "$CAPTURES_ONLY" ]; then   # CAPTURES_ONLY=1: a comment-only source change
  timeout 1800 python -m pytest tests -q -m gpu -rA > "$out/pytest_gpu.log" 2>&1; echo "pytest rc=$?"
  tail -1 "$out/pytest_gpu.log"
  python tools/time_varied.py > "$out/time_varied.log" 2>&1; echo "varied rc=$?"
  python bench.py > "$out/bench_c5.json" 2> "$out/bench_c5.err"; echo "bench rc=$?"
fi
ncu --set full --clock-control none --import-source on -k regex:chunked_kernel -s 5 -c 1 \
    -o "$out/prof_tree1024" -f python bench.py --profile --steps 1 --warmup 1 > "$out/ncu_tree.log" 2>&1; echo "ncu tree rc=$?"
ncu --set full --clock-control none --import-source on -k regex:seq_kernel -s 2 -c 1 \
    -o "$out/prof_seq_c6" -f python tools/tiles_one.py > "$out/ncu_seq.log" 2>&1; echo "ncu seq rc=$?"
ncu --set full --clock-control none --import-source on -k regex:seq_kernel -s 2 -c 1 \
    -o "$out/prof_seq_c7" -f python tools/tiles_one.py --dfs > "$out/ncu_seq7.log" 2>&1; echo "ncu seq7 rc=$?"
