"""z-slab path emulated on ONE GPU (all parts on device 0, one stream): what the slab machinery costs on
top of the single-part solve -- extra launches, halo copies (device-local here, NVLink on a real box),
per-part kernels -- with the halo-volume reductions of round 2 on and off.  Not a scaling measurement
(one GPU does all the work); the parts' results are bit-identical to one part (tests/test_gpu_slabs.py).

  python tools/time_slabs.py [--config 2] [--parts 1,2,4,8]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2312_10615_b200 as smg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--parts", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=2)
    a = ap.parse_args()
    nx, ny, nz, h, lv, kind, seed, tol, name = bench.CONFIGS[a.config]
    b = smg.forcing(nx, ny, nz, h=h, kind=kind, seed=seed)
    for parts in [int(p) for p in a.parts.split(",")]:
        for fr, ov in ((("0", "0"), ("1", "1")) if parts > 1 else (("1", "1"),)):
            os.environ["SMG_DIST_FRAMES"] = fr
            os.environ["SMG_DIST_OVERLAP"] = ov
            s = smg.Solver(nx, ny, nz, h=h, levels=lv, devices=[0] * parts) if parts > 1 else \
                smg.Solver(nx, ny, nz, h=h, levels=lv)
            s.set_rhs(b)
            s.solve_resident(tol, 500)
            ms = it = ln = 0
            for _ in range(a.steps):
                s.solve_resident(tol, 500)
                t = s.timing()
                ms += t["solve_ms"]
                it += t["iterations"]
                ln += t["kernel_launches"]
            print(json.dumps({"config": name, "parts": parts, "frames": int(fr), "overlap": int(ov),
                              "solve_ms": ms / a.steps, "iterations": it // a.steps,
                              "launches_per_solve": ln // a.steps}), flush=True)
            s.close()


if __name__ == "__main__":
    main()
