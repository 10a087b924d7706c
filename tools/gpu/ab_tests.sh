# A/B of variant builds plus the invariants / parity suites on each variant.
# usage: TAG=... CFGS="3 4" bash tools/gpu/ab_tests.sh
cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-abt}
mkdir -p $out
TAG=${TAG:-abt} CFGS="${CFGS:-3 4 5}" bash tools/gpu/ab_libs.sh
for f in paper_2312_05410_b200/_variants/libpf_*.so; do
  n=$(basename $f .so)
  [ "$n" = "libpf_checked" ] && continue
  PF_LIB=$PWD/$f timeout 600 python -m pytest tests/test_invariants_gpu.py tests/test_parity_gpu.py -x -q > $out/tests_$n.log 2>&1
  echo "rc=$?" >> $out/tests_$n.log
done
