#!/bin/bash
# band kernel: border-row pushes before the own-row stores (libpf_vec0) vs default.
cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-s3d}
mkdir -p $out
for rep in 1 2 3; do
timeout 120 python tools/small_grid_sweep.py --only-configs >> $out/sweep_default.jsonl 2>> $out/err.log
PF_LIB=$PWD/paper_2312_05410_b200/_variants/libpf_vec0.so timeout 120 python tools/small_grid_sweep.py --only-configs >> $out/sweep_vec0.jsonl 2>> $out/err.log
done
PF_LIB=$PWD/paper_2312_05410_b200/_variants/libpf_vec0.so timeout 600 python -m pytest tests/test_invariants_gpu.py -k band -x -q > $out/tests.log 2>&1
echo "rc=$?" >> $out/tests.log
timeout 600 python -m pytest tests/test_invariants_gpu.py -k band -x -q > $out/tests_default.log 2>&1
echo "rc=$?" >> $out/tests_default.log
