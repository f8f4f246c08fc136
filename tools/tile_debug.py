"""Tiny tile-kernel probe: one phase of each kernel variant on a forced-tiled 32x16x16 level."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2312_10615_b200 as smg

which = sys.argv[1] if len(sys.argv) > 1 else "fwd"
s = smg.Solver(32, 16, 16, h=1 / 16, levels=2, tile_min=1)
n = s.ndof()
x = np.random.default_rng(1).uniform(-1, 1, n)
b = np.random.default_rng(2).uniform(-1, 1, n)
ph = 0 if which == "fwd" else 10
try:
    y = s.smoother(smg.OP_DGS_PHASE, x, b, arg=ph)
    print(which, "ok", float(np.abs(y - x).max()))
except Exception as e:
    print(which, "FAILED", e)
