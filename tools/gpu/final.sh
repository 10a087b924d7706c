# Evidence run: full GPU suite, the default bench line, the launch list and full ncu captures of the
# stage kernels (cfg3 / cfg4 / cfg5) for profiles/.  usage: TAG=... bash tools/gpu/final.sh
cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-final}
mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=15 > $out/gputests.log 2>&1
echo "pytest rc=$?" >> $out/gputests.log
timeout 600 python bench.py > $out/bench.json 2> $out/bench.err
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-slab"
$CMD > $out/plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_cfg3.csv $CMD > $out/ncu_launch.log 2>&1
for cfg in 3 4 5; do
  C2="python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-slab"
  $C2 > $out/plain_c$cfg.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 6 -c 2 -o $out/pair_c$cfg $C2 > $out/ncu_full_c$cfg.log 2>&1
done
