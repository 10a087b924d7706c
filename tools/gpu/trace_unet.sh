# Step-kernel phase timeline (PF_TRACE variant) on configs[1] / 128^2 / configs[0], and a full ncu
# capture of the U-Net row convolutions.  usage: TAG=... bash tools/gpu/trace_unet.sh
cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-traceu}
mkdir -p $out
export PF_LIB=$PWD/paper_2312_05410_b200/_variants/libpf_trace.so
timeout 120 python tools/trace_step.py 2 > $out/trace_step.jsonl 2>&1
timeout 120 python tools/trace_step.py 2 128 >> $out/trace_step.jsonl 2>&1
timeout 120 python tools/trace_step.py 1 >> $out/trace_step.jsonl 2>&1
unset PF_LIB
timeout 60 ./tools/mma_bench > $out/mma_bench.jsonl 2>&1
CMD="python tools/unet_bench.py --no-cpu --iters 1 --warmup 1"
$CMD > $out/unet_plain.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:"conv3x3_rows_kernel" -s 5 -c 3 -o $out/rows $CMD > $out/ncu_rows.log 2>&1
