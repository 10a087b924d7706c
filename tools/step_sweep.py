"""Cell-steps/s of the persistent small-grid step kernel (kernel_path 7) on configs[1] (256^2) and
128^2 / 512^2 variants under the current library (PF_LIB) and environment (PF_STEP_TBY).
One JSON line per grid."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from small_grid_sweep import _try  # noqa: E402


def main():
    from paper_2312_05410_b200 import pf
    tag = {"lib": os.path.basename(os.environ.get("PF_LIB", "default")), "tby": os.environ.get("PF_STEP_TBY", "auto")}
    p = pf.pf_default_params(2)
    print(json.dumps(dict(tag, config=2, persistent_G=_try(p.replace(kernel_path=7), 2000))), flush=True)
    p1 = pf.pf_default_params(1)
    print(json.dumps(dict(tag, config=1, band_G=_try(p1.replace(kernel_path=6), 1000),
                          persistent_G=_try(p1.replace(kernel_path=7), 1000))), flush=True)
    for n in (128, 512):
        q = p.replace(nx=n, ny=n, ic_height=n / 8, check_every=100)
        print(json.dumps(dict(tag, nx=n, persistent_G=_try(q.replace(kernel_path=7), 400))), flush=True)


if __name__ == "__main__":
    main()
