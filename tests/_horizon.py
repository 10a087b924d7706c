"""Background oracle jobs for the full-horizon parity tests.

The full horizons -- configs[1] to 10,000 steps and configs[2] members 0, 21, 42, 63 to 5,000 steps
-- cost the single-threaded oracle several minutes each.  conftest.py starts them in a thread pool
(one job per member; ctypes releases the GIL, each oracle call stays single-threaded) as soon as
collection shows that tests/test_zz_full_horizon_gpu.py will run, so they overlap the rest of the
GPU suite; the tests there collect the results.  Test glue only: no arithmetic of the method."""
import os
from concurrent.futures import ThreadPoolExecutor

CFG2_STEPS = 10000
CFG3_STEPS = 5000
CFG3_MEMBERS = (0, 21, 42, 63)

_pool = None
_jobs = {}


def _cfg2(ora):
    from paper_2312_05410_b200 import pf
    from tests._maps import oracle_member
    p = pf.pf_default_params(2)
    m, ic = oracle_member(ora, p, 0)
    return ora.step(m, *ora.initial_fields(ic, p.nx, p.ny, 0), CFG2_STEPS)


def _cfg3(ora, k):
    from paper_2312_05410_b200 import pf
    from tests._maps import oracle_member
    p = pf.pf_default_params(3)
    m, ic = oracle_member(ora, p, k)
    return ora.step(m, *ora.initial_fields(ic, p.nx, p.ny, k), CFG3_STEPS)


def start():
    """Submit every full-horizon oracle job (idempotent)."""
    global _pool
    if _pool is not None:
        return
    from oracle import oracle as ora
    ora.build()
    _pool = ThreadPoolExecutor(max_workers=max(1, min(1 + len(CFG3_MEMBERS), os.cpu_count() or 1)))
    _jobs["cfg2"] = _pool.submit(_cfg2, ora)
    for k in CFG3_MEMBERS:
        _jobs[("cfg3", k)] = _pool.submit(_cfg3, ora, k)


def result(key):
    start()
    return _jobs[key].result()
