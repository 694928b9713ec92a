set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2f_build.log 2>&1
timeout 300 python tools/prof_tiles.py > gpurun_out/r2f_prof_tiles.log 2>&1; echo "prof rc=$?"
timeout 600 python tools/tune_tiles.py > gpurun_out/r2f_tune_tiles.log 2>&1; echo "tune rc=$?"
