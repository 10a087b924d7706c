# Packed pair blocks: A/B (default = fp64 packed, wg0 = off, wg2 = fp64 + fp32 packed), then the
# invariants / parity suites on the default build and the fp32 invariants on wg2.
cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-wg}
mkdir -p $out
TAG=${TAG:-wg} CFGS="3 4 5" bash tools/gpu/ab_libs.sh
timeout 600 python -m pytest tests/test_invariants_gpu.py tests/test_parity_gpu.py tests/test_parity_full_gpu.py -x -q > $out/tests_default.log 2>&1
echo "rc=$?" >> $out/tests_default.log
PF_LIB=$PWD/paper_2312_05410_b200/_variants/libpf_wg2.so timeout 300 python -m pytest tests/test_invariants_gpu.py -x -q -k "f32 or fp32 or float" > $out/tests_wg2.log 2>&1
echo "rc=$?" >> $out/tests_wg2.log
