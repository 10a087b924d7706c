cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-unet}
mkdir -p $out
CMD="python tools/unet_bench.py --no-cpu --iters 1 --warmup 1"
$CMD > $out/plain2.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:"conv3x3_rows_kernel" -s 5 -c 3 -o $out/rows $CMD > $out/ncu_full.log 2>&1
