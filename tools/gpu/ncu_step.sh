# ncu of the small-grid kernels: persistent step kernel on configs[1] (256^2), band kernel on
# configs[0]; plus kbench of the ws kernel (kernel_path 5) against the pair kernel.
cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-ncustep}
mkdir -p $out
cat > /tmp/small_run.py <<'PY'
import sys; sys.path.insert(0, '.')
from paper_2312_05410_b200 import pf
p = pf.pf_default_params(int(sys.argv[1])).replace(kernel_path=int(sys.argv[2]))
with pf.Simulation(p) as s:
    s.step(200)
PY
python /tmp/small_run.py 2 7 > $out/plain.log 2>&1 && \
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"persistent_step" -s 1 -c 1 -o $out/step python /tmp/small_run.py 2 7 > $out/ncu.log 2>&1
python /tmp/small_run.py 1 6 >> $out/plain.log 2>&1 && \
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"band_kernel" -s 1 -c 1 -o $out/band python /tmp/small_run.py 1 6 >> $out/ncu.log 2>&1
for cfg in 3 4 5; do
  timeout 60 python tools/kbench.py --config $cfg --path 5 --steps 100 >> $out/kb_ws_c$cfg.json 2>&1
done
