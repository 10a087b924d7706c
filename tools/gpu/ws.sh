# ws kernel (kernel_path 5) packed vs unpacked (libpf_ws0), pair kernel reference, small-grid
# default check, and the ws / persistent bitwise tests.
cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-ws}
mkdir -p $out
for rep in 1 2; do
for cfg in 3 4 5; do
  timeout 60 python tools/kbench.py --config $cfg --path 5 --steps 100 >> $out/kb_ws_c$cfg.json 2>&1
  PF_LIB=$PWD/paper_2312_05410_b200/_variants/libpf_ws0.so timeout 60 python tools/kbench.py --config $cfg --path 5 --steps 100 >> $out/kb_ws0_c$cfg.json 2>&1
done
done
timeout 60 python tools/kbench.py --config 3 --steps 100 >> $out/kb_pair_c3.json 2>&1
timeout 120 python tools/step_sweep.py >> $out/sweep.jsonl 2>> $out/err.log
timeout 600 python -m pytest tests/test_invariants_gpu.py tests/test_parity_gpu.py -x -q > $out/tests.log 2>&1
echo "rc=$?" >> $out/tests.log
