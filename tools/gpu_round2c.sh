set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2c_build.log 2>&1
python -c "import paper_2505_06703_b200 as hs; hs.build_variant('libhs_s1f64.so', ['-DHS_S1_F64=1'])"
timeout 300 python -m pytest tests/test_gpu_stage1_budget.py -q -s > gpurun_out/r2c_budget_f32.log 2>&1
HS_LIB=build/libhs_s1f64.so timeout 300 python -m pytest tests/test_gpu_stage1_budget.py -q -s > gpurun_out/r2c_budget_f64.log 2>&1
timeout 300 python tools/time_stage1.py > gpurun_out/r2c_time_stage1_f32.log 2>&1
HS_LIB=build/libhs_s1f64.so timeout 300 python tools/time_stage1.py > gpurun_out/r2c_time_stage1_f64.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:seq_kernel -s 2 -c 1 -o gpurun_out/r2c_prof_seq -f python tools/tiles_one.py > gpurun_out/r2c_ncu_seq.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi_rank.py tests/test_gpu_parity.py -q -s -x -k "two_ranks or comparison or single_joint or fig7" > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc=$?"
timeout 600 python tools/fig7_sweep.py > gpurun_out/r2c_fig7.log 2>&1; echo "fig7 rc=$?"
cp profiles/r02_fig7_sweep.* gpurun_out/ 2>/dev/null
