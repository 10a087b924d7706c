cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-unet}
mkdir -p $out
timeout 900 python -m pytest tests/test_unet_gpu.py tests/test_abi.py tests/test_unet_abi.py -q > $out/tests.log 2>&1
timeout 600 python tools/unet_bench.py --no-cpu > $out/unet_bench.json 2> $out/unet_bench.err
timeout 600 python tools/hybrid_bench.py > $out/hybrid_bench.json 2> $out/hybrid_bench.err
