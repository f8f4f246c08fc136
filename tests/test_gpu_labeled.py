"""GPU parity on general labelled domains.

`smg_create_labeled` against the oracle built on the same CellGrid: Dirichlet obstacles, Exterior
(homogeneous-Neumann) cells with dropped stencil legs, coarsened labels, the mask-defined band and
the Vanka signature classes.  Every per-point op is required BIT-IDENTICAL (same arithmetic
contract as the box); the all-Interior labelling must reproduce the box kernels.
"""
import numpy as np
import pytest

import oracle
import paper_2312_10615_b200 as smg
from paper_2312_10615_b200 import scenarios

pytestmark = pytest.mark.gpu


def rnd(n, seed):
    return np.random.default_rng(seed).uniform(-1, 1, n)


def same(a, b):
    assert a.shape == b.shape
    if not np.array_equal(a, b):
        d = np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)
        pytest.fail(f"not bit-identical: max rel diff {d:.3e}")


def mixed_domain():
    """24 x 16 x 16: a Dirichlet cylinder, an Exterior outflow strip and an Exterior notch (faces
    with one and with two dropped legs, band cells against every label kind)."""
    lab = scenarios.cylinder3d(24, 16, 16, cx=8 / 24, cy=0.5, radius=3 / 16, outflow=2)
    lab[12:, 12:, :6] = scenarios.E
    return lab


DOMAINS = {
    "mixed": (mixed_domain, 1 / 16, 3),
    "porous": (lambda: scenarios.porous3d(32, 16, 16, seed=3), 1 / 16, 3),
    "brancher": (lambda: scenarios.brancher3d(32, 16, 16), 1 / 16, 3),
    "hollow": (lambda: scenarios.hollow_square3d(32, 32, 8, wall=2), 1 / 32, 2),
}


@pytest.fixture(scope="module", params=list(DOMAINS))
def pair(request):
    make, h, levels = DOMAINS[request.param]
    lab = make()
    oracle.set_threads(4)
    o = oracle.Oracle(0, levels=levels, labels=lab, h=h)
    s = smg.Solver.from_labels(lab, h=h, levels=levels)
    yield o, s, lab, h
    s.close()


def test_counts(pair):
    o, s, lab, _ = pair
    for l in range(o.levels):
        assert s.counts(l) == o.counts(l)
        assert s.ndof(l) == o.ndof(l)
    assert smg.census_labels(lab)["N"] == o.ndof(0)


@pytest.mark.parametrize("pen", [False, True])
def test_apply(pair, pen):
    o, s, _, _ = pair
    for l in range(o.levels):
        x = rnd(o.ndof(l), 10 + l)
        same(s.apply(x, l, pen), o.apply(x, l, pen))


def test_residual(pair):
    o, s, _, _ = pair
    for l in range(o.levels - 1):
        n = o.ndof(l)
        x, b = rnd(n, 1), rnd(n, 2)
        same(s.residual(x, b, l), o.residual(x, b, l))


def test_dgs_phases(pair):
    o, s, _, _ = pair
    for l in range(o.levels - 1):
        n = o.ndof(l)
        x, b = rnd(n, 3), rnd(n, 4)
        for ph in range(smg.DGS_PHASES):
            xo = o.smoother(smg.OP_DGS_PHASE, x, b, l, ph)
            same(s.smoother(smg.OP_DGS_PHASE, x, b, l, ph), xo)
            x = xo


def test_vanka_colours(pair):
    o, s, _, _ = pair
    for l in range(o.levels - 1):
        n = o.ndof(l)
        x, b = rnd(n, 5), rnd(n, 6)
        for col in range(8):
            xo = o.smoother(smg.OP_VANKA_COLOUR, x, b, l, col)
            same(s.smoother(smg.OP_VANKA_COLOUR, x, b, l, col), xo)
            x = xo


@pytest.mark.parametrize("op", [smg.OP_DGS_SYM, smg.OP_VANKA_SYM, smg.OP_SMOOTH])
def test_symmetric_smoothers(pair, op):
    o, s, _, _ = pair
    for l in range(o.levels - 1):
        n = o.ndof(l)
        x, b = rnd(n, 7), rnd(n, 8)
        same(s.smoother(op, x, b, l), o.smoother(op, x, b, l))


def test_transfers(pair):
    o, s, _, _ = pair
    for l in range(o.levels - 1):
        rf, xc = rnd(o.ndof(l), 9), rnd(o.ndof(l + 1), 10)
        same(s.restrict(rf, l), o.restrict(rf, l))
        same(s.prolong(xc, l), o.prolong(xc, l))
        # P = 8 R^T through the shared weight tables
        lhs = float(np.dot(s.prolong(xc, l), rf))
        rhs = 8.0 * float(np.dot(xc, s.restrict(rf, l)))
        assert abs(lhs - rhs) <= 1e-12 * max(abs(lhs), 1.0)


def test_coarse_solve_and_vcycle(pair):
    o, s, _, _ = pair
    b = rnd(o.ndof(o.levels - 1), 11)
    same(s.coarse_solve(b), o.coarse_solve(b))
    b = rnd(o.ndof(0), 12)
    same(s.vcycle(b), o.vcycle(b))


def test_vcycle_symmetric(pair):
    """Theorem 4 / AC 4 on a labelled domain: <u, V v> = <V u, v> on the GPU map."""
    o, s, _, _ = pair
    u, v = rnd(o.ndof(0), 13), rnd(o.ndof(0), 14)
    a, b = float(np.dot(u, s.vcycle(v))), float(np.dot(v, s.vcycle(u)))
    assert abs(a - b) <= 1e-10 * max(abs(a), abs(b))


def test_sqmr_history_and_solution(pair):
    o, s, lab, h = pair
    b = smg.forcing_labels(lab, h, smg.FORCE_UNIFORM, 21)
    same(b, o.forcing(oracle.FORCE_UNIFORM, 21))
    xo, ho, _, so = o.sqmr(b, 1e-8, 60)
    xg, hg, _, st = s.sqmr(b, 1e-8, 60)
    assert st == so == smg.SMG_CONVERGED
    same(np.asarray(hg), ho)
    same(xg, xo)
    # the solve really solved the labelled problem
    r = b - o.apply(xg)
    assert np.linalg.norm(r) / np.linalg.norm(b) < 1e-8


def test_mg_solve(pair):
    o, s, lab, h = pair
    b = smg.forcing_labels(lab, h, smg.FORCE_CHANNEL, 22)
    xo, ho, _, so = o.mg_solve(b, 1e-6, 8)
    xg, hg, _, st = s.mg_solve(b, 1e-6, 8)
    assert st == so
    same(np.asarray(hg), ho)
    same(xg, xo)


def test_all_interior_labels_equal_the_box():
    """An all-Interior labelling is the walled box: the masked kernels must reproduce the box
    kernels (and the oracle) bit for bit."""
    n, levels = 16, 3
    lab = scenarios.cavity3d(n)
    sb = smg.Solver(n, levels=levels, tile_min=-1)
    sl = smg.Solver.from_labels(lab, levels=levels)
    o = oracle.Oracle(n, levels=levels)
    try:
        b = smg.forcing(n, kind=smg.FORCE_UNIFORM, seed=5)
        same(smg.forcing_labels(lab, 1.0 / n, smg.FORCE_UNIFORM, 5), b)
        x = rnd(sb.ndof(0), 1)
        same(sl.apply(x), sb.apply(x))
        same(sl.smoother(smg.OP_SMOOTH, x, b), sb.smoother(smg.OP_SMOOTH, x, b))
        same(sl.vcycle(b), sb.vcycle(b))
        xb, hb, _, _ = sb.sqmr(b, 1e-8, 50)
        xl, hl, _, _ = sl.sqmr(b, 1e-8, 50)
        xo, ho, _, _ = o.sqmr(b, 1e-8, 50)
        same(np.asarray(hl), np.asarray(hb))
        same(np.asarray(hl), ho)
        same(xl, xb)
    finally:
        sb.close()
        sl.close()


def test_direct_on_v1_and_wcycle_labeled():
    # a small domain: direct-on-V1 inverts the dense V1 x V1 block (|V1| ~ 2000 here)
    lab = scenarios.cylinder3d(16, 8, 8, cx=0.4, cy=0.5, radius=0.2, outflow=1)
    lab[6:, 6:, :4] = scenarios.E
    for kw in ({"vanka": smg.VANKA_DIRECT}, {"cycle": 1}):
        o = oracle.Oracle(0, levels=3, labels=lab, h=1 / 8, **kw)
        s = smg.Solver.from_labels(lab, h=1 / 8, levels=3, **kw)
        try:
            b = rnd(o.ndof(0), 31)
            same(s.vcycle(b), o.vcycle(b))
        finally:
            s.close()


def test_additive_vanka_labeled():
    """Additive Vanka on a labelled domain: one application, Alg. 3 with it, the V-cycle
    and MG-SQMR bit-identical to the oracle."""
    lab = mixed_domain()
    oracle.set_threads(4)
    o = oracle.Oracle(0, levels=3, labels=lab, h=1 / 16, vanka=1, omega=0.6)
    s = smg.Solver.from_labels(lab, h=1 / 16, levels=3, vanka=smg.VANKA_ADDITIVE, omega=0.6)
    try:
        for level in range(2):
            n = o.ndof(level)
            x, b = rnd(n, 40 + level), rnd(n, 41 + level)
            same(s.smoother(smg.OP_VANKA_ADD, x, b, level), o.smoother(5, x, b, level))
            same(s.smoother(smg.OP_SMOOTH, x, b, level), o.smoother(4, x, b, level))
        b = rnd(o.ndof(0), 42)
        same(s.vcycle(b), o.vcycle(b))
        xo, ho, _, so = o.sqmr(b, 1e-6, 80)
        xg, hg, _, sg = s.sqmr(b, 1e-6, 80)
        assert so == sg
        same(np.asarray(hg), ho)
        same(xg, xo)
    finally:
        s.close()


def test_labeled_errors():
    lab = mixed_domain()
    with pytest.raises(smg.SmgError):
        smg.Solver.from_labels(lab, levels=6)  # 24 x 16 x 16 is not divisible by 32
    bad = lab.copy()
    bad[0, 0, 0] = 7
    with pytest.raises(smg.SmgError):
        smg.Solver.from_labels(bad, levels=2)
    with pytest.raises(smg.SmgError):
        smg.Solver.from_labels(np.full((8, 8, 8), scenarios.E, np.uint8), levels=2)  # no active DOF


def test_through_flow_channel_with_dirichlet_inflow():
    """Cylinder channel driven by Dirichlet data (PAPER section 6.2.2 inflow profile in, the same
    profile out; zero body force): assemble_rhs_labels -> MG-SQMR, bit-identical to the oracle, and
    the divergence control that follows from the residual bound (AC 9: the continuity rows of the
    converged residual are below tol ||b||)."""
    lab = scenarios.cylinder3d(32, 16, 16, outflow=0)
    h, eta = 0.41 / 16, 1e-3
    b = smg.assemble_rhs_labels(lab, h, *scenarios.channel_inflow(lab, 0.41, 0.45), eta=eta)
    oracle.set_threads(4)
    o = oracle.Oracle(0, levels=3, labels=lab, h=h, eta=eta)
    s = smg.Solver.from_labels(lab, h=h, levels=3, eta=eta)
    try:
        xo, ho, _, so = o.sqmr(b, 1e-8, 100)
        xg, hg, _, sg = s.sqmr(b, 1e-8, 100)
    finally:
        s.close()
    assert so == sg == smg.SMG_CONVERGED
    same(np.asarray(hg), ho)
    same(xg, xo)
    npres = o.counts(0)["np"]
    div = (o.apply(xg) - b)[-npres:]
    assert np.abs(div).max() <= 1e-8 * np.linalg.norm(b)


def test_padded_odd_extents_solve():
    """a grid with odd extents (30 x 13 x 9) padded by scenarios.pad_labels to 32 x 16 x 12
    builds a 3-level hierarchy and solves bit-identically to the oracle on the padded grid."""
    lab = scenarios.pad_labels(scenarios.cylinder3d(30, 13, 9, outflow=1), 3)
    oracle.set_threads(4)
    o = oracle.Oracle(0, levels=3, labels=lab, h=1 / 13)
    s = smg.Solver.from_labels(lab, h=1 / 13, levels=3)
    try:
        b = smg.forcing_labels(lab, 1 / 13, smg.FORCE_CHANNEL, 8)
        xo, ho, _, so = o.sqmr(b, 1e-8, 80)
        xg, hg, _, sg = s.sqmr(b, 1e-8, 80)
    finally:
        s.close()
    assert so == sg == smg.SMG_CONVERGED
    same(np.asarray(hg), ho)
    same(xg, xo)
