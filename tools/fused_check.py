import sys, numpy as np
sys.path.insert(0, '.')
from paper_2312_05410_b200 import pf
def run(p, n):
    with pf.Simulation(p) as s:
        s.step(n)
        return [s.fields(m) for m in range(p.n_members)]
ok = True
for (nx, ny, mem, extra) in [(128, 40, 2, {}), (512, 72, 2, {}), (96, 64, 3, dict(noise_rho=0.2)), (1000, 24, 1, {}), (4096, 12, 1, {})]:
    p = pf.pf_default_params(2).replace(nx=nx, ny=ny, ic_height=ny/4, n_members=mem, graph_steps=0, seed=21,
                                       theta_deg=71.0, M_A_bulk=12.0, M_B_bulk=6.0, M_A_surf=9.0, M_B_surf=3.0, **extra)
    a = run(p.replace(kernel_path=3), 7)
    b = run(p.replace(kernel_path=int(sys.argv[1]) if len(sys.argv) > 1 else 4), 7)
    for m in range(mem):
        eq = all(np.array_equal(x, y) for x, y in zip(a[m], b[m]))
        err = max(float(np.abs(x - y).max()) for x, y in zip(a[m], b[m]))
        print(nx, ny, m, "bitwise" if eq else f"DIFF max {err:.3e}")
        ok &= eq
print("ALL OK" if ok else "MISMATCH")
