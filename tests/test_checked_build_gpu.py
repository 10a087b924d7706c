"""The checked build (paper_2312_05410_b200/_variants/libpf_checked.so: every kernel with device-side
bounds checks that trap, 64 KiB guard zones around every state buffer) runs each kernel path on a
small case without a trap and with every guard byte intact.  This stands in for compute-sanitizer
memcheck, which the GPU pool does not allow; races are covered by the bitwise
run-to-run and cross-path invariants (tests/test_invariants_gpu.py)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def checked_lib():
    from paper_2312_05410_b200 import build
    return build.build_checked()


@pytest.mark.parametrize("case", ["band", "persistent", "pair", "loopback", "peer", "nccl_self", "ws", "tile"])
def test_checked_build_case(checked_lib, case):
    env = dict(os.environ, PF_LIB=checked_lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_case.py"), case], env=env,
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-3000:])
    assert "guard zones of 65536 B intact" in r.stdout, r.stdout
