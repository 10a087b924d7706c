cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-ncupair}
mkdir -p $out
cat > /tmp/pair_run.py <<'PY'
import sys; sys.path.insert(0, '.')
from paper_2312_05410_b200 import pf
p = pf.pf_default_params(int(sys.argv[1])).replace(check_every=1000)
with pf.Simulation(p) as s:
    s.step(4)
PY
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"pair_kernel" -s 2 -c 2 -o $out/pair python /tmp/pair_run.py 3 > $out/ncu.log 2>&1
