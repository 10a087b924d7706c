cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-san}
mkdir -p $out
for tool in memcheck racecheck synccheck; do
  for case in band persistent pair loopback ws; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py $case > $out/${tool}_${case}.log 2>&1
    echo "$tool $case rc=$?" >> $out/summary.txt
  done
done
