cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-f32}
mkdir -p $out
timeout 900 python -m pytest tests/test_invariants_gpu.py tests/test_parity_full_gpu.py -q -x -k "fp32 or cfg5 or tile_stream" > $out/tests.log 2>&1
for rep in 1 2; do for cfg in 5 3; do
  timeout 120 python tools/kbench.py --config $cfg --steps 100 >> $out/kb_c${cfg}.json 2>&1
done; done
