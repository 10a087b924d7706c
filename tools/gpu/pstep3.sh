cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-pstep}
mkdir -p $out
timeout 300 python tools/small_grid_sweep.py > $out/sweep.jsonl 2>&1
for f in paper_2312_05410_b200/_variants/libpf_n*.so; do n=$(basename $f .so)
PF_LIB=$PWD/$f timeout 300 python tools/small_grid_sweep.py > $out/sweep_$n.jsonl 2>&1
done
