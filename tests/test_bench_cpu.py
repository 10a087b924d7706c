"""The reference arm of bench.py (the oracle) runs on the host alone and prints one
contract JSON line whose per-step time is measured, not extrapolated."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                        "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "cell-updates/s"
    assert line["steps"] == 2 and line["warmup"] == 3 and line["value"] > 0
    procs = line["cpu_baseline"]["cores"]
    assert 1 <= procs <= min(os.cpu_count() or 1, 64)
    # value = cells of the sample (one 512^2 member per process) x steps / measured wall time
    assert abs(line["value"] * line["ms_per_step"] * 1e-3 - procs * 512 * 512) <= 1e-6 * procs * 512 * 512
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["scaling"] == "weak" and line["higher_is_better"] is True
