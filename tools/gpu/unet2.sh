cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-unet}
mkdir -p $out
timeout 900 python -m pytest tests/test_unet_gpu.py -q -x > $out/tests.log 2>&1
timeout 600 python tools/unet_bench.py --no-cpu > $out/unet_bench.json 2> $out/unet_bench.err
CMD="python tools/unet_bench.py --no-cpu --iters 2 --warmup 1"
$CMD > $out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/unet_launches.csv $CMD > $out/ncu.log 2>&1
python tools/launch_table.py $out/unet_launches.csv 29 > $out/launch_table.txt 2>&1
