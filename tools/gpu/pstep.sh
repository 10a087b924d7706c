cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-pstep}
mkdir -p $out
timeout 600 python -m pytest tests/test_invariants_gpu.py -x -q -k "persistent or band" > $out/tests.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > $out/parity.log 2>&1
timeout 300 python tools/small_grid_sweep.py > $out/sweep.jsonl 2>&1
PF_PERSIST_STEP=0 timeout 300 python tools/small_grid_sweep.py > $out/sweep_old.jsonl 2>&1
