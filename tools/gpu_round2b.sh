set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2b_build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -s -k "multi_tile or large_skeleton or forced_split" > gpurun_out/r2b_pytest_tiles.log 2>&1; echo "tiles rc=$?"
timeout 300 python -m pytest tests/test_gpu_stage1_budget.py tests/test_gpu_stage1.py -x -q -s > gpurun_out/r2b_pytest_stage1.log 2>&1; echo "stage1 rc=$?"
timeout 300 python tools/time_tiles.py > gpurun_out/r2b_time_tiles.log 2>&1; echo "time rc=$?"
