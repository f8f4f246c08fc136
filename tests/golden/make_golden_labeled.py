"""Oracle golden of a full-size labelled domain: the cylinder channel of PAPER section
6.2.2 at 256 x 128 x 128 cells (Dirichlet cylinder, Exterior outflow column; 16.2 M DOFs), 5 levels,
channel forcing seed 4 -- the workload `bench.py` reports under also.labelled_cylinder.  Holds the
first 4 MG-SQMR iterations: residual history, and per-field L2 norms / sha256 of the iterate (zeros
normalised to +0.0), so tests/test_gpu_fullsize.py can require the GPU's labelled-domain kernels to
reproduce the oracle bit for bit at full size.  Self-pinned like the box goldens (the reference pins
no residual history).

    python tests/golden/make_golden_labeled.py        # ~3 min on 8 threads, ~12 GB RAM
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402
from paper_2312_10615_b200 import scenarios  # noqa: E402  (host-side numpy label builder only)

NX, NY, NZ, LEVELS, SEED, MAXIT = 256, 128, 128, 5, 4, 4


def digest(x, cnt):
    out, o = {}, 0
    for k in ("nu", "nv", "nw", "np"):
        v = np.ascontiguousarray(x[o:o + cnt[k]] + 0.0)
        o += cnt[k]
        if k == "np":
            v = np.ascontiguousarray(v - v.mean() + 0.0)
        out[k] = {"l2": float(np.linalg.norm(v)), "sha256": hashlib.sha256(v.tobytes()).hexdigest()}
    return out


def main():
    oracle.set_threads(os.cpu_count() or 1)
    t0 = time.time()
    lab = scenarios.cylinder3d(NX, NY, NZ)
    h = 1.0 / NY
    o = oracle.Oracle(0, levels=LEVELS, labels=lab, h=h)
    b = o.forcing(oracle.FORCE_CHANNEL, SEED)
    x, hist, _, st = o.sqmr(b, tol=1e-30, maxit=MAXIT)
    rec = {"scenario": "cylinder3d", "grid": [NX, NY, NZ], "h": h, "levels": LEVELS, "forcing": oracle.FORCE_CHANNEL,
           "seed": SEED, "maxit": MAXIT, "eta": 1.0, "gamma": 1e-3, "nu": 1, "band_width": 1,
           "labels_sha256": hashlib.sha256(lab.tobytes()).hexdigest(), "counts": o.counts(0),
           "b_sha256": hashlib.sha256(np.ascontiguousarray(b).tobytes()).hexdigest(),
           "status": st, "history": [float(v) for v in hist], "fields": digest(x, o.counts(0)),
           "oracle_seconds": time.time() - t0, "oracle_threads": os.cpu_count()}
    with open(os.path.join(HERE, "labelled_cylinder_golden.json"), "w") as f:
        json.dump(rec, f, indent=1)
    print(st, hist, f"{time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
