"""Per-component CUDA-event timing of one MG-SQMR iteration (cfg by id)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2312_10615_b200 as smg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
nx, ny, nz, h, lv, kind, seed, tol, name = bench.CONFIGS[a.config]
s = smg.Solver(nx, ny, nz, h=h, levels=lv)
s.set_rhs(smg.forcing(nx, ny, nz, h=h, kind=kind, seed=seed))
s.solve_resident(tol, 500)
names = {0: "apply", 1: "residual", 2: "dgs_sym", 3: "vcycle_from", 4: "vanka_sym", 5: "smooth", 6: "restrict",
         7: "prolong", 8: "coarse", 9: "cdot2", 10: "axpy", 11: "sqmr_iter_graph"}
out = {"config": name, "coop_blocks_per_sm": os.environ.get("SMG_COOP_BLOCKS_PER_SM", "max")}
for l in range(lv):
    for w in (0, 1, 2, 3, 4, 5, 6, 7, 9):
        if l == lv - 1 and w in (2, 4, 5, 6, 7):
            continue
        out[f"L{l}_{names[w]}_ms"] = round(s.time_kernel(w, a.reps, l), 4)
out["coarse_ms"] = round(s.time_kernel(8, a.reps, lv - 1), 4)
out["sqmr_iter_graph_ms"] = round(s.time_kernel(11, a.reps, 0), 4)
print(json.dumps(out, indent=1))
