cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-checked}
mkdir -p $out
timeout 900 python -m pytest tests/test_checked_build_gpu.py -q -rA > $out/checked.log 2>&1
for case in band persistent pair loopback ws tile; do
  PF_LIB=$PWD/paper_2312_05410_b200/_variants/libpf_checked.so timeout 300 python tools/sanitize_case.py $case >> $out/cases.log 2>&1
done
