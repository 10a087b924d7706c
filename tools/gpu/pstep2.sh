cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-pstep}
mkdir -p $out
timeout 600 python -m pytest tests/test_invariants_gpu.py -x -q -k "persistent or band or default" > $out/tests.log 2>&1
timeout 300 python tools/small_grid_sweep.py > $out/sweep.jsonl 2>&1
PF_LIB=$PWD/paper_2312_05410_b200/_variants/libpf_t8.so timeout 300 python tools/small_grid_sweep.py > $out/sweep_t8.jsonl 2>&1
