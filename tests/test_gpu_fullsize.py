"""Full BASELINE sizes (cfg 1-4) on the GPU, where the CPU oracle cannot follow:
size-independent properties — convergence to the config tolerance, bitwise
determinism, slab-decomposition invariance, true-residual consistency, and
probe-based symmetry / linearity of L and of the V-cycle (SPEC AC 4, SPEC:108,
170, 390-391)."""
import numpy as np
import pytest

import bench
import paper_2312_10615_b200 as smg

pytestmark = pytest.mark.gpu


def solver_for(cfg, **kw):
    nx, ny, nz, h, lv, kind, seed, tol, _ = bench.CONFIGS[cfg]
    s = smg.Solver(nx, ny, nz, h=h, levels=lv, **kw)
    b = smg.forcing(nx, ny, nz, h=h, kind=kind, seed=seed)
    return s, b, tol


@pytest.mark.parametrize("cfg,max_its", [(1, 12), (2, 20), (3, 20), (4, 40)])
def test_converges_and_is_deterministic(cfg, max_its):
    s, b, tol = solver_for(cfg)
    x1, h1, _, st1 = s.sqmr(b, tol, 200)
    assert st1 == smg.SMG_CONVERGED and len(h1) <= max_its and h1[-1] < tol
    s.set_rhs(b)
    h2, st2 = s.solve_resident(tol, 200)
    assert st2 == st1 and np.array_equal(h1, h2) and np.array_equal(s.solution(), x1)
    # reported history = independently recomputed true residual
    r = b - s.apply(x1)
    assert np.isclose(np.linalg.norm(r) / np.linalg.norm(b), h1[-1], rtol=1e-9)
    # divergence control (SPEC AC 9)
    npres = s.counts()["np"]
    assert np.abs(s.apply(x1)[-npres:]).max() <= 10 * tol * np.linalg.norm(b) / np.sqrt(s.ndof())
    s.close()


def test_slab_invariance_256():
    one, b, tol = solver_for(2)
    two = smg.Solver(256, levels=6, devices=[0, 0])
    x1, h1, _, _ = one.sqmr(b, tol, 100)
    x2, h2, _, _ = two.sqmr(b, tol, 100)
    assert np.array_equal(h1, h2) and np.array_equal(x1, x2)


@pytest.mark.parametrize("cfg", [1, 2])
def test_operator_and_preconditioner_symmetry_linearity(cfg):
    s, _, _ = solver_for(cfg)
    rng = np.random.default_rng(cfg)
    n = s.ndof()
    a, c = rng.standard_normal(n), rng.standard_normal(n)
    for pen in (False, True):
        la, lc = s.apply(a, penalized=pen), s.apply(c, penalized=pen)
        assert abs(c @ la - a @ lc) <= 1e-12 * np.abs(c * la).sum()
    va, vc = s.vcycle(a), s.vcycle(c)
    assert abs(c @ va - a @ vc) <= 1e-10 * np.abs(c * va).sum()  # W^dagger symmetric
    lin = s.vcycle(2.0 * a - 0.5 * c)
    assert np.allclose(lin, 2.0 * va - 0.5 * vc, rtol=0, atol=1e-11 * np.abs(lin).max())
    assert not s.vcycle(np.zeros(n)).any()
    s.close()


def test_labelled_cylinder_fullsize_matches_oracle_golden():
    """General labelled domain at full size: the 256 x 128 x 128 cylinder channel of
    bench.py's also.labelled_cylinder line against the committed oracle golden
    (tests/golden/make_golden_labeled.py): the first MG-SQMR iterations' residual history and the
    iterate's u, v, w and mean-free p bit for bit; then the solve to 1e-6 converges, is
    deterministic, and its reported history is the true residual."""
    import hashlib
    import json
    import os

    from paper_2312_10615_b200 import scenarios

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    g = json.load(open(os.path.join(root, "tests", "golden", "labelled_cylinder_golden.json")))
    nx, ny, nz = g["grid"]
    lab = scenarios.cylinder3d(nx, ny, nz)
    assert hashlib.sha256(lab.tobytes()).hexdigest() == g["labels_sha256"]
    s = smg.Solver.from_labels(lab, h=g["h"], levels=g["levels"])
    assert s.counts() == g["counts"]
    b = smg.forcing_labels(lab, g["h"], g["forcing"], g["seed"])
    assert hashlib.sha256(b.tobytes()).hexdigest() == g["b_sha256"]
    x, h, _, st = s.sqmr(b, 1e-30, g["maxit"])
    assert h.tolist() == g["history"]
    o = 0
    for k in ("nu", "nv", "nw", "np"):
        v = np.ascontiguousarray(x[o:o + g["counts"][k]] + 0.0)
        o += g["counts"][k]
        if k == "np":
            v = np.ascontiguousarray(v - v.mean() + 0.0)
        assert abs(np.linalg.norm(v) - g["fields"][k]["l2"]) <= 1e-6 * g["fields"][k]["l2"]
        assert hashlib.sha256(v.tobytes()).hexdigest() == g["fields"][k]["sha256"], f"field {k} not bit-identical"
    x1, h1, _, st1 = s.sqmr(b, 1e-6, 200)
    assert st1 == smg.SMG_CONVERGED and len(h1) <= 25 and h1[: len(h)].tolist() == g["history"]
    s.set_rhs(b)
    h2, st2 = s.solve_resident(1e-6, 200)
    assert st2 == st1 and np.array_equal(h1, h2) and np.array_equal(s.solution(), x1)
    r = b - s.apply(x1)
    assert np.isclose(np.linalg.norm(r) / np.linalg.norm(b), h1[-1], rtol=1e-9)
    s.close()
