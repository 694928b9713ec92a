set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2w_build.log 2>&1
timeout 300 python tools/prof_tiles.py > gpurun_out/r2w_prof_tiles.log 2>&1; echo "prof rc=$?"
timeout 600 python tools/tune_tiles.py > gpurun_out/r2w_tune_tiles.log 2>&1; echo "tune rc=$?"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -s -k "multi_tile or large_skeleton" > gpurun_out/r2w_pytest_tiles.log 2>&1; echo "tiles rc=$?"
