# Evidence run (round 2, final session): smoke, full GPU suite, the default bench line, the launch
# list, full ncu captures of the stage kernels (cfg3 / cfg4 / cfg5), the U-Net bench + launch table +
# one full ncu capture of its largest row convolution.  usage: TAG=... bash tools/gpu/final2.sh
cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-final2}
mkdir -p $out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1
echo "smoke rc=$?" >> $out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=15 > $out/gputests.log 2>&1
echo "pytest rc=$?" >> $out/gputests.log
timeout 600 python bench.py > $out/bench.json 2> $out/bench.err
timeout 300 python tools/unet_bench.py > $out/unet_bench.json 2> $out/unet_bench.err
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-slab"
$CMD > $out/plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_cfg3.csv $CMD > $out/ncu_launch.log 2>&1
for cfg in 3 4; do
  C2="python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-slab"
  $C2 > $out/plain_c$cfg.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 6 -c 2 -o $out/pair_c$cfg $C2 > $out/ncu_full_c$cfg.log 2>&1
done
UC="python tools/unet_bench.py --no-cpu --iters 1 --warmup 1"
timeout 240 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/unet_launches.csv $UC > $out/unet_ncu_launch.log 2>&1
python tools/launch_table.py $out/unet_launches.csv > $out/unet_launch_table.txt 2>&1
timeout 500 ncu --set full --import-source on --clock-control none -k regex:"conv3x3_rows_kernel" -s 12 -c 1 -o $out/unet_rows $UC > $out/ncu_unet_rows.log 2>&1
