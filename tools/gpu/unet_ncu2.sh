cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-unetncu}
mkdir -p $out
CMD="python tools/unet_bench.py --no-cpu --iters 1 --warmup 1"
timeout 500 ncu --set full --import-source on --clock-control none -k regex:"conv3x3_rows_kernel" -s 8 -c 1 -o $out/rows $CMD > $out/ncu_rows.log 2>&1
