# A/B of variant builds (paper_2312_05410_b200/_variants/libpf_*.so, not the checked one) with
# tools/kbench.py.  usage: TAG=... CFGS="3 4" TESTS="tests/..." bash tools/gpu/ab_libs.sh
cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-ab}
mkdir -p $out
for rep in 1 2; do
for cfg in ${CFGS:-3 4}; do
  timeout 60 python tools/kbench.py --config $cfg --steps 100 >> $out/kb_c${cfg}_default.json 2>&1
  for f in paper_2312_05410_b200/_variants/libpf_*.so; do
    n=$(basename $f .so)
    [ "$n" = "libpf_checked" ] && continue
    PF_LIB=$PWD/$f timeout 60 python tools/kbench.py --config $cfg --steps 100 >> $out/kb_c${cfg}_$n.json 2>&1
  done
done
done
if [ -n "$TESTS" ]; then timeout 900 python -m pytest $TESTS -x -q > $out/tests.log 2>&1; fi
