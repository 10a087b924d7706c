# Step-kernel tile-shape sweep (variant libpf_stt: PF_STEP_TBY selects the tile shape:
# 8 = 32x8/512 threads (default), 9 = 32x8/544, 12 = 32x12/704, 16 = 32x16/1024).
cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-step}
mkdir -p $out
for tby in 8 9 12 16; do
  PF_LIB=$PWD/paper_2312_05410_b200/_variants/libpf_stt.so PF_STEP_TBY=$tby timeout 120 python tools/step_sweep.py >> $out/sweep.jsonl 2>> $out/err.log
done
for tby in 12 16; do
PF_LIB=$PWD/paper_2312_05410_b200/_variants/libpf_stt.so PF_STEP_TBY=$tby timeout 600 python -m pytest tests/test_invariants_gpu.py tests/test_parity_gpu.py -x -q -k "persistent or cfg2 or cfg1" > $out/tests_stt_$tby.log 2>&1
echo "rc=$?" >> $out/tests_stt_$tby.log
done
