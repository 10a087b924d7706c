cd $GRAFT_REPO_ROOT
nproc > gpurun_out/r2_nproc.txt; lscpu | head -20 >> gpurun_out/r2_nproc.txt
timeout 1500 python -m pytest tests -m gpu -x -q -rA --durations=25 > gpurun_out/r2_gputest1.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_gputest1.log
timeout 300 python bench.py > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err
