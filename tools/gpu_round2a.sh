set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2a_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -rA -s > gpurun_out/r2a_pytest_gpu.log 2>&1; echo "pytest rc=$?"
HS_LIB=build/libhs_s1approx.so timeout 300 python -m pytest tests/test_gpu_stage1_budget.py -q -s > gpurun_out/r2a_budget_approx.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "bench rc=$?"
