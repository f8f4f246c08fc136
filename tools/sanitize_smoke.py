"""Small end-to-end solves for compute-sanitizer (memcheck / racecheck / synccheck):
exercises every kernel family: cluster + grid cooperative sweeps, shared-memory
smoother, per-phase DGS, ping-pong Vanka, transfers, coarse GEMV, SQMR graph,
and the z-slab path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2312_10615_b200 as smg  # noqa: E402

b = smg.forcing(64, seed=1)
s = smg.Solver(64, levels=4)
x, h, _, st = s.sqmr(b, 1e-6, 50)
assert st == smg.SMG_CONVERGED, st
s2 = smg.Solver(64, levels=4, devices=[0, 0])
x2, h2, _, _ = s2.sqmr(b, 1e-6, 50)
assert np.array_equal(x, x2)
s3 = smg.Solver(32, levels=3, cycle=1)
s3.mg_solve(smg.forcing(32, seed=2), 1e-6, 20)
print("sanitize smoke ok", len(h))
