# U-Net: GPU parity tests, the bench line and the launch table; the MMA issue microbenchmark.
cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-unet3}
mkdir -p $out
UN_DEBUG_LAUNCH=1 timeout 60 python tools/unet_probe.py conv 8 80 128 64 16 > $out/probe.log 2>&1 || exit 1
UN_DEBUG_LAUNCH=1 UN_NO_GRAPH=1 timeout 60 python tools/unet_probe.py fwd 64 256 256 >> $out/probe.log 2>&1
timeout 400 python -m pytest tests/test_unet_gpu.py -x -q > $out/tests.log 2>&1
echo "rc=$?" >> $out/tests.log
timeout 120 python tools/unet_bench.py --no-cpu > $out/unet_bench.json 2> $out/unet_bench.err
CMD="python tools/unet_bench.py --no-cpu --iters 1 --warmup 1"
timeout 240 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv $CMD > $out/ncu_launch.log 2>&1
python tools/launch_table.py $out/launches.csv > $out/launch_table.txt 2>&1
TAG=$(basename $out) bash tools/gpu/untrace.sh
