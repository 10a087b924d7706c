cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-traj}
mkdir -p $out
timeout 900 python -m pytest tests/test_trajectory_gpu.py tests/test_abi.py -q -rA > $out/tests.log 2>&1
timeout 300 python tools/dataset_bench.py > $out/dataset_bench.jsonl 2>&1
