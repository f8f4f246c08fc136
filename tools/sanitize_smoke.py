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
# tile-ordered DGS (TMA-staged tiles) on a small level, and a labelled domain (masked kernels)
s4 = smg.Solver(32, 16, 16, h=1 / 16, levels=2, tile_min=1)
assert s4.dgs_tiled(0)
s4.sqmr(smg.forcing(32, 16, 16, h=1 / 16, seed=3), 1e-6, 30)
from paper_2312_10615_b200 import scenarios  # noqa: E402

lab = scenarios.porous3d(32, 16, 16, seed=3)
s5 = smg.Solver.from_labels(lab, h=1 / 16, levels=3)
_, h5, _, st5 = s5.sqmr(smg.forcing_labels(lab, 1 / 16, 0, 4), 1e-8, 60)
assert st5 == smg.SMG_CONVERGED
print("sanitize smoke (tiles, labelled) ok", len(h5))
