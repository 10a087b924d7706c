# Step-kernel tile / unroll sweep (variants libpf_stu2 = unroll 2 + tile knob, libpf_stt6 = tile knob).
cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-step}
mkdir -p $out
timeout 120 python tools/step_sweep.py >> $out/sweep.jsonl 2>> $out/err.log
for v in stu2 stt6; do
  for tby in 4 6 8; do
    PF_LIB=$PWD/paper_2312_05410_b200/_variants/libpf_$v.so PF_STEP_TBY=$tby timeout 120 python tools/step_sweep.py >> $out/sweep.jsonl 2>> $out/err.log
  done
done
PF_LIB=$PWD/paper_2312_05410_b200/_variants/libpf_stu2.so timeout 600 python -m pytest tests/test_invariants_gpu.py -x -q -k "persistent or band or small" > $out/tests_stu2.log 2>&1
echo "rc=$?" >> $out/tests_stu2.log
