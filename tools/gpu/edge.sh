# Edge-store rewrite: A/B vs HEAD build, block-span trace, invariants + parity tests.
cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-edge}
mkdir -p $out
TAG=${TAG:-edge} CFGS="3 4 5" bash tools/gpu/ab_libs.sh
for cfg in 3 4; do
  PF_LIB=$PWD/paper_2312_05410_b200/_variants/libpf_trace.so timeout 120 python tools/trace_stage1.py $cfg > $out/trace_c$cfg.json 2>> $out/trace.err
done
for cfg in 3 4; do
  PF_STREAM_NOGROUP=1 timeout 120 python tools/kbench.py --config $cfg --steps 100 >> $out/kb_c${cfg}_nogroup.json 2>&1
done
timeout 900 python -m pytest tests/test_invariants_gpu.py tests/test_parity_gpu.py tests/test_parity_full_gpu.py -x -q > $out/tests.log 2>&1
echo tests rc=$? >> $out/tests.log
