"""paper_2312_05410_b200 -- B200-native explicit-midpoint step of the PVD phase-field model
of arXiv 2312.05410 (C-ABI library libpf.so + thin ctypes binding).  See DESIGN.md."""
from .pf import *  # noqa: F401,F403
from .pf import Simulation, PfError, lib  # noqa: F401
