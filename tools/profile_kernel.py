"""Profiler-bracketed single component launch (for ncu --profile-from-start off).

  python tools/profile_kernel.py --config 1 --which 4 --level 3
which: see smg_time_kernel in include/smg.h (2 DGS sweep, 4 Vanka sweep, 11 SQMR iteration graph, ...).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2312_10615_b200 as smg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--which", type=int, default=4)
ap.add_argument("--level", type=int, default=0)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
nx, ny, nz, h, lv, kind, seed, tol, name = bench.CONFIGS[a.config]
s = smg.Solver(nx, ny, nz, h=h, levels=lv)
s.set_rhs(smg.forcing(nx, ny, nz, h=h, kind=kind, seed=seed))
s.solve_resident(tol, 500)
s.time_kernel(a.which, 2, a.level)  # warm
smg.lib().smg_profiler_range(1)
ms = s.time_kernel(a.which, a.reps, a.level)
smg.lib().smg_profiler_range(0)
print(name, "which", a.which, "level", a.level, "ms", ms)
s.close()
