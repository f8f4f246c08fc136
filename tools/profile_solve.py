"""Profiling driver: one warm MG-SQMR solve, then a profiler-bracketed region of
`--iters` SQMR iterations, for `ncu --profile-from-start off`.

  python tools/profile_solve.py --config 1 --iters 1
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2312_10615_b200 as smg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--iters", type=int, default=1)
a = ap.parse_args()
nx, ny, nz, h, lv, kind, seed, tol, name = bench.CONFIGS[a.config]
s = smg.Solver(nx, ny, nz, h=h, levels=lv)
s.set_rhs(smg.forcing(nx, ny, nz, h=h, kind=kind, seed=seed))
s.solve_resident(tol, 500)
smg.lib().smg_profiler_range(1)
hist, st = s.solve_resident(1e-300, a.iters)
smg.lib().smg_profiler_range(0)
print(name, "profiled iterations:", len(hist), "launches:", s.timing()["kernel_launches"])
s.close()
