cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-bench}
mkdir -p $out
timeout 600 python -m pytest tests/test_nccl_gpu.py tests/test_invariants_gpu.py -q -rs > $out/tests.log 2>&1
timeout 600 python bench.py > $out/bench.json 2> $out/bench.err
