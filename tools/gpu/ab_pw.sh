# A/B of the pair kernel with / without the producer warp (PF_PAIR_PW), then the invariant tests
cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-ab}
mkdir -p $out
for cfg in 3 4 5; do
  for pw in 0 1; do
    PF_PAIR_PW=$pw timeout 120 python tools/kbench.py --config $cfg --steps 100 > $out/kb_c${cfg}_pw${pw}.json 2>&1
  done
done
timeout 900 python -m pytest tests/test_invariants_gpu.py tests/test_parity_gpu.py -x -q > $out/tests.log 2>&1
timeout 300 python bench.py --no-cpu-baseline > $out/bench.json 2> $out/bench.err
