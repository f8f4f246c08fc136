"""Generate the oracle golden fixtures under tests/golden/ (committed).

The reference (arXiv 2312.10615) ships no solver and pins no residual history
(SPEC:624), so these fixtures are self-pinned by the oracle after it passed the
census / structural / direct-solve tests in tests/test_oracle_*.py.  They let
the GPU tests run on a box without the oracle's 128^3 runtime, and pin the
oracle against accidental change.

    python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402

CASES = {
    # name: (n, levels, forcing kind, seed, tol)  — BASELINE.json configs 0 and 1
    "cfg0": (32, 3, oracle.FORCE_UNIFORM, 0, 1e-6),
    "cfg1": (128, 5, oracle.FORCE_UNIFORM, 1, 1e-6),
}


def main():
    oracle.set_threads(os.cpu_count() or 1)
    for name, (n, lv, kind, seed, tol) in CASES.items():
        o = oracle.Oracle(n, levels=lv)
        b = o.forcing(kind, seed)
        x, hist, _, st = o.sqmr(b, tol=tol, maxit=200)
        c = o.counts(0)
        npres = c["np"]
        p = x[-npres:] - x[-npres:].mean()
        rec = {
            "grid": [n, n, n], "levels": lv, "forcing": kind, "seed": seed, "tol": tol,
            "eta": 1.0, "gamma": 1e-3, "nu": 1, "band_width": 1,
            "status": st, "iterations": len(hist), "history": [float(v) for v in hist],
            "b_sha256": hashlib.sha256(np.ascontiguousarray(b).tobytes()).hexdigest(),
            "u_norm": float(np.linalg.norm(x[:-npres])), "p_norm_meanfree": float(np.linalg.norm(p)),
            "u_sum": float(x[:-npres].sum()),
        }
        with open(os.path.join(HERE, f"{name}_history.json"), "w") as f:
            json.dump(rec, f, indent=1)
        print(name, st, len(hist), hist[-1])


if __name__ == "__main__":
    main()
