"""MG-SQMR on a large labelled domain (cylinder channel / porous slab): device-resident solve time,
iterations, and the same grid size as a walled box for comparison."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2312_10615_b200 as smg  # noqa: E402
from paper_2312_10615_b200 import scenarios  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nx", type=int, default=256)
ap.add_argument("--ny", type=int, default=128)
ap.add_argument("--nz", type=int, default=128)
ap.add_argument("--levels", type=int, default=5)
ap.add_argument("--scenario", default="cylinder")
ap.add_argument("--tol", type=float, default=1e-6)
ap.add_argument("--no-box", action="store_true")
a = ap.parse_args()
mk = {"cylinder": scenarios.cylinder3d, "porous": scenarios.porous3d, "brancher": scenarios.brancher3d,
      "hollow": scenarios.hollow_square3d}[a.scenario]
lab = mk(a.nx, a.ny, a.nz)
h = 1.0 / a.ny
t0 = time.time()
s = smg.Solver.from_labels(lab, h=h, levels=a.levels)
b = smg.forcing_labels(lab, h, smg.FORCE_CHANNEL, 4)
print(f"{a.scenario} {a.nx}x{a.ny}x{a.nz}: N = {s.ndof(0)}, setup {time.time() - t0:.1f} s", flush=True)
s.set_rhs(b)
for rep in range(3):
    hist, st = s.solve_resident(a.tol, 300)
    t = s.timing()
    print(f"  labelled: status {st}, {len(hist)} iterations, {t['solve_ms']:.1f} ms, "
          f"{s.ndof(0) * len(hist) / t['solve_ms'] / 1e6:.2f} GDOF/s, {t['kernel_launches']} launches, rel {hist[-1]:.2e}", flush=True)
xm, hm, _, stm = s.mg_solve(b, a.tol, 30)  # pure multigrid on L~ (PAPER section 6: the robustness split)
print(f"  pure MG (30 cycles max): status {stm}, {len(hm)} cycles, rel {hm[-1]:.2e}", flush=True)
s.close()
if a.no_box:
    sys.exit(0)
sb = smg.Solver(a.nx, a.ny, a.nz, h=h, levels=a.levels, tile_min=-1)
sb.set_rhs(smg.forcing(a.nx, a.ny, a.nz, h=h, kind=smg.FORCE_CHANNEL, seed=4))
for rep in range(2):
    hist, st = sb.solve_resident(a.tol, 300)
    t = sb.timing()
    print(f"  box (untiled): status {st}, {len(hist)} iterations, {t['solve_ms']:.1f} ms, "
          f"{sb.ndof(0) * len(hist) / t['solve_ms'] / 1e6:.2f} GDOF/s, {t['kernel_launches']} launches", flush=True)
