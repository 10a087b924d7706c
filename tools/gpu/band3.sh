# band kernel: st.async + mbarrier halos (default) vs cluster barrier per stage (libpf_band0).
cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-band3}
mkdir -p $out
for rep in 1 2; do
timeout 120 python tools/step_sweep.py >> $out/sweep.jsonl 2>> $out/err.log
PF_LIB=$PWD/paper_2312_05410_b200/_variants/libpf_band0.so timeout 120 python tools/step_sweep.py >> $out/sweep.jsonl 2>> $out/err.log
done
timeout 600 python -m pytest tests/test_invariants_gpu.py tests/test_parity_gpu.py -x -q > $out/tests.log 2>&1
echo "rc=$?" >> $out/tests.log
for c in 3 4; do PF_WS_NCW=2 timeout 60 python tools/kbench.py --config $c --path 5 --steps 100 >> $out/kb_ws_ncw2_c$c.json 2>&1; done
