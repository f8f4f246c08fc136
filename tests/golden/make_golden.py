"""Generate the oracle golden fixtures under tests/golden/ (committed).

The reference (arXiv 2312.10615) ships no solver and pins no residual history
(SPEC:624), so these fixtures are self-pinned by the oracle after it passed the
census / structural / direct-solve tests in tests/test_oracle_*.py.  They let
the GPU tests run on a box without the oracle's runtime, and pin the oracle
against accidental change.  Per config: the residual history, the iteration
count and status, and the solution -- per-field L2 norms and sha256 of u, v, w
and the mean-free p (zeros normalised to +0.0), so a GPU test can check the
whole solution vector bit for bit without storing it.

    python tests/golden/make_golden.py                 # cfg0, cfg1 (full), cfg2 (full solve)
    python tests/golden/make_golden.py cfg3 cfg4       # first 3 iterations (needs ~100 GB RAM;
                                                       # run on the GPU box's host)
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

CASES = {
    # name: (nx, ny, nz, h, levels, forcing kind, seed, tol, maxit) -- BASELINE.json configs 0-4
    "cfg0": (32, 32, 32, 1 / 32, 3, oracle.FORCE_UNIFORM, 0, 1e-6, 200),
    "cfg1": (128, 128, 128, 1 / 128, 5, oracle.FORCE_UNIFORM, 1, 1e-6, 200),
    "cfg2": (256, 256, 256, 1 / 256, 6, oracle.FORCE_FOURIER, 2, 1e-6, 200),
    "cfg3": (512, 512, 512, 1 / 512, 7, oracle.FORCE_UNIFORM, 3, 1e-6, 3),
    "cfg4": (1024, 256, 256, 1 / 256, 7, oracle.FORCE_CHANNEL, 4, 1e-8, 3),
}


def field_digest(x, nx, ny, nz):
    """Per-field L2 norms and sha256 of u, v, w and the mean-free pressure (compact order)."""
    nu, nv, nw = (nx - 1) * ny * nz, nx * (ny - 1) * nz, nx * ny * (nz - 1)
    parts = {"u": x[:nu], "v": x[nu:nu + nv], "w": x[nu + nv:nu + nv + nw]}
    p = x[nu + nv + nw:]
    parts["p_meanfree"] = p - p.mean()
    out = {}
    for k, v in parts.items():
        v = np.ascontiguousarray(v + 0.0)  # -0.0 -> +0.0: the sign of a zero carries no information
        out[k] = {"l2": float(np.linalg.norm(v)), "sha256": hashlib.sha256(v.tobytes()).hexdigest()}
    return out


def make(name):
    nx, ny, nz, h, lv, kind, seed, tol, maxit = CASES[name]
    t0 = time.time()
    o = oracle.Oracle(nx, ny, nz, h=h, levels=lv)
    b = oracle.forcing_box(nx, ny, nz, h, kind, seed)
    x, hist, _, st = o.sqmr(b, tol=tol, maxit=maxit)
    npres = nx * ny * nz
    p = x[-npres:] - x[-npres:].mean()
    rec = {
        "grid": [nx, ny, nz], "h": h, "levels": lv, "forcing": kind, "seed": seed, "tol": tol, "maxit": maxit,
        "eta": 1.0, "gamma": 1e-3, "nu": 1, "band_width": 1, "dgs_tiles": [list(o.dgs_tile(l)) for l in range(lv)],
        "status": st, "iterations": len(hist), "history": [float(v) for v in hist],
        "b_sha256": hashlib.sha256(np.ascontiguousarray(b).tobytes()).hexdigest(),
        "u_norm": float(np.linalg.norm(x[:-npres])), "p_norm_meanfree": float(np.linalg.norm(p)),
        "u_sum": float(x[:-npres].sum()), "fields": field_digest(x, nx, ny, nz),
        "oracle_seconds": time.time() - t0, "oracle_threads": os.cpu_count(),
    }
    with open(os.path.join(HERE, f"{name}_history.json"), "w") as f:
        json.dump(rec, f, indent=1)
    print(name, st, len(hist), hist[-1], f"{time.time() - t0:.0f} s", flush=True)


def main():
    oracle.set_threads(os.cpu_count() or 1)
    names = sys.argv[1:] or ["cfg0", "cfg1", "cfg2"]
    for name in names:
        make(name)


if __name__ == "__main__":
    main()
