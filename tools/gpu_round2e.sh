set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2e_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -s -k "multi_tile or large_skeleton or forced_split" > gpurun_out/r2e_pytest_tiles.log 2>&1; echo "tiles rc=$?"
timeout 300 python tools/time_tiles.py > gpurun_out/r2e_time_tiles.log 2>&1; echo "time rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:seq_kernel -s 2 -c 1 -o gpurun_out/r2e_prof_seq -f python tools/tiles_one.py > gpurun_out/r2e_ncu_seq.log 2>&1
timeout 600 python -m pytest tests/test_gpu_stage1.py -x -q -s > gpurun_out/r2e_pytest_stage1.log 2>&1; echo "stage1 rc=$?"
