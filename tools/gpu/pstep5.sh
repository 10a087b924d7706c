cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-pstep}
mkdir -p $out
timeout 300 python tools/small_grid_sweep.py > $out/sweep.jsonl 2>&1
PF_LIB=$PWD/paper_2312_05410_b200/_variants/libpf_t4.so timeout 300 python tools/small_grid_sweep.py > $out/sweep_t4.jsonl 2>&1
