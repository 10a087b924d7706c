# persistent step kernel: neighbour flags (default) vs a grid barrier per step (PF_STEP_FLAGS=0)
cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-flags}
mkdir -p $out
for rep in 1 2; do
timeout 120 python tools/step_sweep.py >> $out/sweep_flags.jsonl 2>> $out/err.log
PF_STEP_FLAGS=0 timeout 120 python tools/step_sweep.py >> $out/sweep_gridsync.jsonl 2>> $out/err.log
done
timeout 900 python -m pytest tests/test_invariants_gpu.py tests/test_parity_gpu.py tests/test_checked_build_gpu.py -x -q > $out/tests.log 2>&1
echo "rc=$?" >> $out/tests.log
