cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-pstep}
mkdir -p $out
timeout 600 python -m pytest tests/test_invariants_gpu.py tests/test_parity_gpu.py -x -q > $out/tests.log 2>&1
timeout 300 python tools/small_grid_sweep.py > $out/sweep.jsonl 2>&1
