cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-ncustep2}
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
