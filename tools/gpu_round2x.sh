set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2x_build.log 2>&1
timeout 300 python tools/prof_tiles.py > gpurun_out/r2x_prof_tiles.log 2>&1; echo "prof rc=$?"
timeout 600 python tools/tune_tiles.py > gpurun_out/r2x_tune_tiles.log 2>&1; echo "tune rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:seq_kernel -s 2 -c 1 -o gpurun_out/r2x_prof_seq -f python tools/tiles_one.py > gpurun_out/r2x_ncu_seq.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lbs.py tests/test_gpu_stage1_budget.py -x -q -s -k "multi_tile or large_skeleton or multi_cta or budget" > gpurun_out/r2x_pytest.log 2>&1; echo "tests rc=$?"
timeout 300 python tools/time_stage1.py > gpurun_out/r2x_time_stage1.log 2>&1; echo "s1 rc=$?"
