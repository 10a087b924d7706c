cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-untrace}
mkdir -p $out
export PF_LIB=$PWD/paper_2312_05410_b200/_variants/libpf_untrace.so
for a in "64 256 256 32 16" "64 256 256 16 16" "64 128 128 64 16" "64 128 128 16 32"; do
  timeout 60 python tools/unet_trace.py $a >> $out/trace.jsonl 2>&1
done
