"""Parity report (run on a GPU box): the measured GPU-vs-oracle errors behind BASELINE.md 6, with the
same inputs, horizons and metrics as tests/test_parity_gpu.py and tests/test_parity_full_gpu.py.

    python tests/parity_report.py > parity.json
"""
import json
import os
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as ora  # noqa: E402  (test infrastructure)
from paper_2312_05410_b200 import pf  # noqa: E402
from tests._maps import oracle_member, normwise  # noqa: E402
from tests.test_parity_full_gpu import _window, _window_err  # noqa: E402

POOL = ThreadPoolExecutor(max_workers=max(2, min(8, os.cpu_count() or 2)))


def diag_rel(d, dref):
    return max(abs(d[q] - dref[q]) / abs(dref[q]) for q in (0, 3))


def main():
    ora.build()
    out = {}
    # cfg1: 1 and 1000 steps
    p = pf.pf_default_params(1)
    m, ic = oracle_member(ora, p, 0)
    u0 = ora.initial_fields(ic, 64, 64, 0)
    with pf.Simulation(p) as s:
        s.step(1); e1 = normwise(s.fields(0), ora.step(m, *u0, 1))
        s.step(999); ref = ora.step(m, *u0, 1000); e = normwise(s.fields(0), ref)
        dr = diag_rel(s.diagnostics(0), ora.diagnostics(m, *ref))
    out["cfg1"] = {"step1": e1, "step1000": e, "diag_rel_step1000": dr}
    # cfg2: 1000 steps
    p = pf.pf_default_params(2)
    m, ic = oracle_member(ora, p, 0)
    u0 = ora.initial_fields(ic, 256, 256, 0)
    f = POOL.submit(ora.step, m, *u0, 1000)
    with pf.Simulation(p) as s:
        s.step(1); e1 = normwise(s.fields(0), ora.step(m, *u0, 1))
        s.step(999); g = s.fields(0); d = s.diagnostics(0)
    ref = f.result()
    out["cfg2"] = {"step1": e1, "step1000": normwise(g, ref), "diag_rel_step1000": diag_rel(d, ora.diagnostics(m, *ref))}
    # cfg3: all members 1 step, 4 members 400 steps
    p = pf.pf_default_params(3)
    with pf.Simulation(p) as s:
        s.step(1); g1 = s.fields(-1)
        s.step(399); g400 = {k: s.fields(k) for k in (0, 21, 42, 63)}

    def one(k):
        m, ic = oracle_member(ora, p, k)
        return normwise([g1[0][k], g1[1][k], g1[2][k]], ora.step(m, *ora.initial_fields(ic, 512, 512, k), 1))

    def long(k):
        m, ic = oracle_member(ora, p, k)
        return normwise(g400[k], ora.step(m, *ora.initial_fields(ic, 512, 512, k), 400))
    out["cfg3"] = {"step1_max_over_64_members": max(POOL.map(one, range(64))),
                   "step400_max_over_members_0_21_42_63": max(POOL.map(long, (0, 21, 42, 63)))}
    # cfg4: full grid 1 step; windows at 100 steps
    p = pf.pf_default_params(4)
    m, ic = oracle_member(ora, p, 0)
    wins = [(1000, 0, 1024, 1024), (3000, 100, 1024, 1024)]
    futs = [POOL.submit(_window, ora, m, ic, 0, 4096, 4096, i0, j0, W, H, 100) for i0, j0, W, H in wins]
    with pf.Simulation(p) as s:
        s.step(1); g1 = s.fields(0)
        s.step(99); g100 = s.fields(0)
    e1 = normwise(g1, ora.step(m, *ora.initial_fields(ic, 4096, 4096, 0), 1))
    ew = [_window_err(g100, j0, H, cols, ref, valid) for (i0, j0, W, H), (ref, valid, cols) in
          zip(wins, [f.result() for f in futs])]
    out["cfg4"] = {"step1_full_grid": e1, "step100_windows": ew}
    # cfg5: fp32 windows at 100 steps
    p = pf.pf_default_params(5)
    m, ic = oracle_member(ora, p, 0)
    wins = [(2000, 3584, 1024, 1024), (6000, 0, 1024, 1024)]
    futs = [POOL.submit(_window, ora, m, ic, 0, 8192, 8192, i0, j0, W, H, 100) for i0, j0, W, H in wins]
    with pf.Simulation(p) as s:
        s.step(100); g = s.fields(0)
    ew = [_window_err(g, j0, H, cols, ref, valid) for (i0, j0, W, H), (ref, valid, cols) in
          zip(wins, [f.result() for f in futs])]
    out["cfg5_fp32"] = {"step100_windows": ew}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
