"""CUDA-event time of the fine-level symmetric DGS sweep / Vanka sweep / smooth (cfg by id)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2312_10615_b200 as smg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
nx, ny, nz, h, lv, kind, seed, tol, name = bench.CONFIGS[a.config]
s = smg.Solver(nx, ny, nz, h=h, levels=lv)
s.set_rhs(smg.forcing(nx, ny, nz, h=h, kind=kind, seed=seed))
hist, st = s.solve_resident(tol, 500)
hist, st = s.solve_resident(tol, 500)
print(name.split(":")[0], "solve %.2f ms, %d iterations" % (s.timing()["solve_ms"], len(hist)))
for rep in range(2):
    print(name.split(":")[0], "dgs_sym %.4f  vanka_sym %.4f  smooth %.4f  apply %.4f ms" % (
        s.time_kernel(2, a.reps, 0), s.time_kernel(4, a.reps, 0), s.time_kernel(5, a.reps, 0), s.time_kernel(0, a.reps, 0)))
# as the V-cycle runs them: k_dgs_cb once per level visit, the sweep / smooth without it
print(name.split(":")[0], "k_dgs_cb %.4f  dgs_sym(cb ready) %.4f  smooth(cb ready) %.4f  L1 smooth %.4f  vcycle %.4f ms" % (
    s.time_kernel(12, a.reps, 0), s.time_kernel(13, a.reps, 0), s.time_kernel(14, a.reps, 0),
    s.time_kernel(5, a.reps, 1) if lv > 2 else 0.0, s.time_kernel(3, a.reps, 0)))
