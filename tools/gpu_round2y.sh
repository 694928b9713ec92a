set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2y_build.log 2>&1
python -c "import paper_2505_06703_b200 as hs; hs.build_variant('libhs_hints.so', ['-DHS_STREAM_HINTS=1'])"
for i in 1 2; do
timeout 300 python tools/time_scan.py > gpurun_out/r2y_time_scan_default_$i.log 2>&1
HS_LIB=build/libhs_hints.so timeout 300 python tools/time_scan.py > gpurun_out/r2y_time_scan_hints_$i.log 2>&1
done
timeout 300 python tools/prof_tiles.py > gpurun_out/r2y_prof_tiles.log 2>&1; echo "prof rc=$?"
timeout 600 python tools/tune_tiles.py > gpurun_out/r2y_tune_tiles.log 2>&1; echo "tune rc=$?"
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2y_pytest_gpu.log 2>&1; echo "pytest rc=$?"
