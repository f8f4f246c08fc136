"""General labelled domains on the CPU (no GPU): the library's host-side domain module against the
oracle, and the oracle's structural invariants on domains with obstacles and Exterior cells
(AC 3, 4, 8 analogues in 3-D).  The GPU parity tests proper are in
tests/test_gpu_labeled.py."""
import numpy as np
import pytest

import oracle
import paper_2312_10615_b200 as smg
from paper_2312_10615_b200 import scenarios

SCEN = {
    "cylinder": lambda: scenarios.cylinder3d(32, 16, 8),
    "hollow": lambda: scenarios.hollow_square3d(24, 24, 8, wall=2),
    "brancher": lambda: scenarios.brancher3d(32, 16, 8),
    "porous": lambda: scenarios.porous3d(32, 16, 16, seed=1),
}


@pytest.mark.parametrize("name", list(SCEN))
def test_host_domain_module_matches_oracle(name):
    lab = SCEN[name]()
    assert lab.dtype == np.uint8 and set(np.unique(lab)) <= {0, 1, 2}
    assert np.array_equal(SCEN[name](), lab)  # builders are deterministic
    assert smg.census_labels(lab) == oracle.census_labels(lab)
    assert smg.census_labels(lab, 2) == oracle.census_labels(lab, 2)
    c1 = smg.coarsen_labels(lab)
    assert np.array_equal(c1, oracle.coarsen_labels(lab))
    assert smg.census_labels(c1) == oracle.census_labels(c1)
    o = oracle.Oracle(0, levels=2, labels=lab, h=1 / 16)
    for kind in (smg.FORCE_UNIFORM, smg.FORCE_FOURIER, smg.FORCE_CHANNEL):
        assert np.array_equal(smg.forcing_labels(lab, 1 / 16, kind, 9), o.forcing(kind, 9))
    assert o.counts(1)["np"] == int((c1 == 1).sum())


def test_coarsening_is_monotone():
    """promoting a fine cell E -> I or I -> D never demotes the coarse label (D > I > E)."""
    rng = np.random.default_rng(0)
    rank = np.array([2, 1, 0])  # label -> order: D highest
    lab = rng.integers(0, 3, (8, 8, 8)).astype(np.uint8)
    c0 = smg.coarsen_labels(lab)
    for _ in range(50):
        z, y, x = rng.integers(0, 8, 3)
        up = lab.copy()
        if up[z, y, x] == 2:
            up[z, y, x] = 1
        elif up[z, y, x] == 1:
            up[z, y, x] = 0
        c1 = smg.coarsen_labels(up)
        assert np.all(rank[c1] >= rank[c0])


def test_census_edge_cases():
    assert smg.census_labels(np.full((4, 4, 4), 2, np.uint8))["N"] == 0          # all Exterior
    assert smg.census_labels(np.ones((3, 3, 3), np.uint8))["N"] == 81            # 27 p + 3 * 18 faces
    lab = np.ones((4, 4, 4), np.uint8)
    lab[:, :, 3] = 2
    c = smg.census_labels(lab)
    assert c["nu"] == 2 * 16 and c["np"] == 48                                    # the I|E faces are Inactive
    with pytest.raises(smg.SmgError):
        smg.coarsen_labels(np.ones((3, 4, 4), np.uint8))


def small_domain():
    lab = np.ones((8, 8, 8), np.uint8)
    lab[2:4, 3:5, 3:5] = 0   # Dirichlet block
    lab[:, :, 7] = 2         # Exterior outflow column
    lab[6:, 6:, :2] = 2      # Exterior notch
    return lab


def test_labelled_operator_is_symmetric_with_dropped_legs():
    o = oracle.Oracle(0, levels=2, labels=small_domain(), h=1 / 8)
    for pen in (False, True):
        A = o.dense(0, pen)
        assert np.abs(A - A.T).max() <= 1e-12 * np.abs(A).max()
    # a momentum row next to an Exterior cell has a reduced diagonal: 6 - dropped legs
    nv = sum(o.counts(0)[k] for k in ("nu", "nv", "nw"))
    d = np.diag(o.dense(0, False))[:nv] / 64.0
    assert set(np.round(d).astype(int)) <= {3, 4, 5, 6} and (np.round(d) < 6).any()
    # rows of A sum to (diag - active neighbours): dropped legs contribute nothing
    x = np.random.default_rng(1).standard_normal(o.ndof(0))
    assert np.allclose(o.apply(x), o.dense(0, False) @ x, rtol=1e-12, atol=1e-9)


@pytest.mark.parametrize("op", [1, 3, 4])
def test_labelled_smoothers_are_symmetric(op):
    """Theorems 1, 3, 4 on a labelled domain (AC 3 analogue): <u, S v> = <S u, v> for the maps b -> x
    of symmetric DGS, symmetric Vanka and Alg. 3 from x0 = 0."""
    o = oracle.Oracle(0, levels=2, labels=small_domain(), h=1 / 8)
    n = o.ndof(0)
    rng = np.random.default_rng(2)
    u, v = rng.standard_normal(n), rng.standard_normal(n)
    z = np.zeros(n)
    a = float(u @ o.smoother(op, z, v))
    b = float(v @ o.smoother(op, z, u))
    assert abs(a - b) <= 1e-10 * max(abs(a), abs(b))


def test_labelled_vcycle_symmetric_linear_and_transfer_adjoint():
    o = oracle.Oracle(0, levels=3, labels=scenarios.porous3d(16, 16, 16, seed=5, block=2), h=1 / 16)
    n = o.ndof(0)
    rng = np.random.default_rng(3)
    u, v = rng.standard_normal(n), rng.standard_normal(n)
    vu, vv = o.vcycle(u), o.vcycle(v)
    assert abs(u @ vv - v @ vu) <= 1e-10 * abs(u @ vv)
    assert np.allclose(o.vcycle(2.0 * u + v), 2.0 * vu + vv, rtol=1e-10, atol=1e-12)
    xc = rng.standard_normal(o.ndof(1))
    assert abs(o.prolong(xc) @ u - 8.0 * (xc @ o.restrict(u))) <= 1e-12 * abs(o.prolong(xc) @ u)


def test_robustness_split_on_obstacle_domains():
    """AC 8 analogue in 3-D (PAPER section 6.1.3): on the brancher, pure multigrid fails to reach
    1e-2 while MG-preconditioned SQMR reaches 1e-8 within 100 iterations."""
    oracle.set_threads(4)
    lab = scenarios.brancher3d(32, 16, 16)
    o = oracle.Oracle(0, levels=3, labels=lab, h=1 / 16)
    b = o.forcing(oracle.FORCE_CHANNEL, 22)
    _, hm, _, stm = o.mg_solve(b, 1e-2, 12)
    assert stm == oracle.ST_MAXIT and hm[-1] > 1e-2
    x, hs, _, sts = o.sqmr(b, 1e-8, 100)
    assert sts == oracle.ST_CONVERGED and len(hs) <= 100
    # divergence control (AC 9): ||B u||_inf <= 10 tol ||b|| / sqrt(N)
    npres = o.counts(0)["np"]
    div = o.apply(x)[-npres:]
    assert np.abs(div).max() <= 10 * 1e-8 * np.linalg.norm(b) / np.sqrt(o.ndof(0))


def test_inflow_profile():
    H = 0.41
    assert scenarios.inflow_profile(H / 2, H, 0.3) == pytest.approx(0.3)
    assert scenarios.inflow_profile(0.0, H, 0.3) == 0.0 and scenarios.inflow_profile(H, H, 0.3) == 0.0
    assert scenarios.inflow_profile(H / 2, H, 0.45, z=H / 2) == pytest.approx(0.45)
    with pytest.raises(ValueError):
        scenarios.inflow_profile(0.5, H, 0.3)


def test_assemble_rhs_with_general_dirichlet_data():
    """assemble_rhs on a labelled grid: the library's host routine against the oracle
    bit for bit, the cavity lid as a special case, and RHS compatibility."""
    lab = scenarios.cylinder3d(32, 16, 8)
    h = 0.41 / 16
    o = oracle.Oracle(0, levels=2, labels=lab, h=h, eta=1e-3)
    rng = np.random.default_rng(0)
    g = [rng.uniform(-1, 1, s) for s in smg.dirichlet_shapes(lab)]
    assert np.array_equal(smg.assemble_rhs_labels(lab, h, *g, eta=1e-3), o.dirichlet_rhs(*g))
    b0 = rng.uniform(-1, 1, o.ndof(0))
    assert np.array_equal(smg.assemble_rhs_labels(lab, h, *g, eta=1e-3, b=b0), o.dirichlet_rhs(*g, b=b0))
    n = 8
    box = scenarios.cavity3d(n)
    gu, gv, gw = [np.zeros(s) for s in smg.dirichlet_shapes(box)]
    gu[:, n + 1, :] = 1.0  # the u faces of the ring cells above the top (y = ny): the moving lid
    assert np.array_equal(smg.assemble_rhs_labels(box, 1 / n, gu, gv, gw), smg.cavity_rhs(n))
    # through-flow channel: inflow profile in, the same profile out -> continuity RHS sums to zero
    ch = scenarios.cylinder3d(32, 16, 16, outflow=0)
    b = smg.assemble_rhs_labels(ch, h, *scenarios.channel_inflow(ch, 0.41, 0.45), eta=1e-3)
    npres = int((ch == 1).sum())
    assert abs(b[-npres:].sum()) <= 1e-12 * np.abs(b[-npres:]).sum()
    with pytest.raises(ValueError):
        smg.assemble_rhs_labels(ch, h, gu, gv, gw)  # wrong shapes


def test_labelled_mgsqmr_matches_dense_direct_solve():
    """AC 6 / AC 11 analogue on a labelled domain (Dirichlet block, Exterior column and notch): the
    oracle's MG-SQMR solution against a dense direct solve of the assembled L (pressure constant
    fixed by a Lagrange multiplier) -- an independent pin of the labelled operator and solver."""
    o = oracle.Oracle(0, levels=2, labels=small_domain(), h=1 / 8)
    b = o.forcing(oracle.FORCE_UNIFORM, 3)
    x, hist, _, st = o.sqmr(b, tol=1e-11, maxit=200)
    assert st == oracle.ST_CONVERGED
    L = o.dense(0, False)
    n, npres = L.shape[0], o.counts(0)["np"]
    e = np.zeros(n)
    e[n - npres:] = 1.0
    A = np.zeros((n + 1, n + 1))
    A[:n, :n], A[:n, n], A[n, :n] = L, e, e
    xd = np.linalg.solve(A, np.append(b, 0.0))[:n]
    u, ud = x[:-npres], xd[:-npres]
    p, pd = x[-npres:] - x[-npres:].mean(), xd[-npres:] - xd[-npres:].mean()
    assert np.linalg.norm(u - ud) / np.linalg.norm(ud) < 1e-8
    assert np.linalg.norm(p - pd) / np.linalg.norm(pd) < 1e-8


def test_pad_labels_keeps_the_fine_level_problem():
    """SPEC:81 padding (Exterior cells behind an explicit Dirichlet layer): extents become divisible by
    2^(levels-1) and the fine-level DofMap and operator are those of the unpadded grid."""
    lab = scenarios.cylinder3d(30, 13, 9, outflow=1)
    pad = scenarios.pad_labels(lab, 3)
    assert all(n % 4 == 0 for n in pad.shape) and pad.shape == (12, 16, 32)
    assert np.array_equal(pad[:9, :13, :30], lab) and set(np.unique(pad[9:])) <= {0, 2}
    c0, c1 = smg.census_labels(lab), smg.census_labels(pad)
    assert c0 == c1
    o0 = oracle.Oracle(0, levels=2, labels=lab, h=1 / 13)
    o1 = oracle.Oracle(0, levels=2, labels=pad, h=1 / 13)
    x = np.random.default_rng(0).standard_normal(o0.ndof(0))
    assert np.array_equal(o0.apply(x), o1.apply(x))
    assert scenarios.pad_labels(pad, 3) is pad or np.array_equal(scenarios.pad_labels(pad, 3), pad)
