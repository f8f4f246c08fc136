"""Profiling driver for the labelled-domain path: one warm MG-SQMR solve of the cylinder channel,
then a profiler-bracketed region of `--iters` SQMR iterations (ncu --profile-from-start off)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_10615_b200 as smg  # noqa: E402
from paper_2312_10615_b200 import scenarios  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=1)
a = ap.parse_args()
nx, ny, nz, lv = 256, 128, 128, 5
lab = scenarios.cylinder3d(nx, ny, nz)
s = smg.Solver.from_labels(lab, h=1.0 / ny, levels=lv)
s.set_rhs(smg.forcing_labels(lab, 1.0 / ny, smg.FORCE_CHANNEL, 4))
s.solve_resident(1e-6, 500)
smg.lib().smg_profiler_range(1)
hist, st = s.solve_resident(1e-300, a.iters)
smg.lib().smg_profiler_range(0)
print("labelled cylinder", nx, ny, nz, "profiled iterations:", len(hist), "launches:", s.timing()["kernel_launches"])
s.close()
