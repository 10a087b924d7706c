cd $GRAFT_REPO_ROOT
out=gpurun_out/${TAG:-band}
mkdir -p $out
timeout 600 python -m pytest tests/test_invariants_gpu.py -x -q -k "band or persistent" > $out/tests.log 2>&1
timeout 300 python tools/small_grid_sweep.py > $out/sweep.jsonl 2>&1
cat > /tmp/band_run.py <<'PY'
import sys; sys.path.insert(0, '.')
from paper_2312_05410_b200 import pf
p = pf.pf_default_params(int(sys.argv[1])).replace(kernel_path=int(sys.argv[2]))
with pf.Simulation(p) as s:
    s.step(200)
PY
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"band_kernel" -c 1 -o $out/band python /tmp/band_run.py 1 6 > $out/ncu.log 2>&1
