set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2k_build.log 2>&1
timeout 300 python tools/prof_tiles.py > gpurun_out/r2k_prof_tiles.log 2>&1; echo "prof rc=$?"
timeout 600 python tools/tune_tiles.py > gpurun_out/r2k_tune_tiles.log 2>&1; echo "tune rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:seq_kernel -s 2 -c 1 -o gpurun_out/r2k_prof_seq -f python tools/tiles_one.py > gpurun_out/r2k_ncu_seq.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -s -k "multi_tile or large_skeleton" > gpurun_out/r2k_pytest_tiles.log 2>&1; echo "tiles rc=$?"
