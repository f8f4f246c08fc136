"""Structural known-answer tests that pin the oracle (SPEC AC 3, 4, 5; SPEC:128,
168-170, 198, 219-224, 264-283, 300, 321-325, 390-391, 597).  These are the
reference's own invariants; no reference artefact pins the per-iteration values
(SPEC:624), so these plus the direct-solve checks are what validate the oracle.
"""
import numpy as np
import pytest

import oracle

OP_PHASE, OP_DGS, OP_VCOL, OP_VANKA, OP_SMOOTH = 0, 1, 2, 3, 4


def materialize(f, n):
    cols = []
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        cols.append(f(e))
    return np.stack(cols, axis=1)


def defect(A):
    return np.linalg.norm(A - A.T) / max(np.linalg.norm(A), 1e-300)


@pytest.fixture(scope="module", autouse=True)
def _serial():
    oracle.set_threads(1)  # tiny grids: thread start-up would dominate
    yield


@pytest.fixture(scope="module")
def o8():
    return oracle.Oracle(8, levels=2)


def test_operator_symmetric_and_matches_apply(o8):
    for pen in (False, True):
        A = o8.dense(0, pen)
        assert defect(A) == 0.0
        x = np.random.default_rng(1).standard_normal(A.shape[0])
        assert np.allclose(o8.apply(x, penalized=pen), A @ x, rtol=0, atol=1e-10 * np.abs(A @ x).max())


def test_penalty_diagonal(o8):
    # gamma = 1e-3: pressure diagonal entries equal -1e-3
    A = o8.dense(0, True)
    c = o8.counts(0)
    npres = c["np"]
    assert np.all(np.diag(A)[-npres:] == -1e-3)
    assert np.all(np.diag(o8.dense(0, False))[-npres:] == 0.0)


def test_apply_linear_zero(o8):
    n = o8.ndof()
    assert not o8.apply(np.zeros(n)).any()
    rng = np.random.default_rng(2)
    a, b = rng.standard_normal(n), rng.standard_normal(n)
    lhs = o8.apply(2.5 * a - 0.75 * b)
    rhs = 2.5 * o8.apply(a) - 0.75 * o8.apply(b)
    assert np.allclose(lhs, rhs, atol=1e-10 * np.abs(rhs).max())


def test_prolong_is_8_restrict_transpose(o8):
    # P = c R^T exactly (c = 8 in 3-D)
    nf, nc = o8.ndof(0), o8.ndof(1)
    P = materialize(lambda e: o8.prolong(e, 0), nc)
    R = materialize(lambda e: o8.restrict(e, 0), nf)
    assert P.shape == (nf, nc) and R.shape == (nc, nf)
    assert np.array_equal(P, 8.0 * R.T)


def test_transfer_adjoint_and_partition_of_unity():
    o = oracle.Oracle(16, levels=2)
    nf, nc = o.ndof(0), o.ndof(1)
    rng = np.random.default_rng(3)
    xc, rf = rng.standard_normal(nc), rng.standard_normal(nf)
    assert np.isclose(o.prolong(xc) @ rf, 8.0 * (xc @ o.restrict(rf)), rtol=1e-13)
    pf = o.prolong(np.ones(nc))
    # partition of unity on fully-interior regions: pressures all 1, deep faces 1
    cnt = o.counts(0)
    assert np.all(pf[-cnt["np"]:] == 1.0)
    u = pf[: cnt["nu"]].reshape(16, 16, 15)
    assert np.all(u[2:-2, 2:-2, 1:-1] == 1.0)


def test_transfer_zero():
    o = oracle.Oracle(8, levels=2)
    assert not o.prolong(np.zeros(o.ndof(1))).any()
    assert not o.restrict(np.zeros(o.ndof(0))).any()


@pytest.mark.parametrize("op", [OP_DGS, OP_VANKA, OP_SMOOTH])
def test_smoother_symmetry_8(o8, op):
    # Theorems 1, 3, 4 (SPEC AC 3): relative symmetry defect < 1e-10
    n = o8.ndof()
    C = materialize(lambda e: o8.smoother(op, np.zeros(n), e), n)
    assert defect(C) < 1e-10
    assert np.abs(C).max() > 0


@pytest.mark.parametrize("nu", [1, 2, 3])
def test_smoother_symmetry_6cubed(nu):
    # SPEC AC 3 at 6^3 for nu in {1,2,3} (one level, smoother only)
    o = oracle.Oracle(6, levels=1, nu=nu)
    n = o.ndof()
    for op in (OP_VANKA, OP_SMOOTH):
        C = materialize(lambda e: o.smoother(op, np.zeros(n), e), n)
        assert defect(C) < 1e-10


def test_dgs_fixed_point(o8):
    # b = L~x  =>  x unchanged by every phase
    n = o8.ndof()
    x = np.random.default_rng(4).standard_normal(n)
    b = o8.apply(x, penalized=True)
    for ph in range(20):
        y = o8.smoother(OP_PHASE, x, b, arg=ph)
        assert np.allclose(y, x, atol=1e-11 * np.abs(x).max())


def test_vanka_block_residual_zero_after_solve(o8):
    # after a colour phase the block-local residuals of that colour vanish
    n = o8.ndof()
    rng = np.random.default_rng(5)
    x, b = rng.standard_normal(n), rng.standard_normal(n)
    y = o8.smoother(OP_VCOL, x, b, arg=0)
    r = o8.residual(y, b)
    # colour-0 band cells: pressure rows of cells with even (i,j,k) on the shell
    nx = 8
    cnt = o8.counts(0)
    rp = r[-cnt["np"]:].reshape(nx, nx, nx)
    shell = np.zeros((nx, nx, nx), bool)
    shell[[0, -1], :, :] = shell[:, [0, -1], :] = shell[:, :, [0, -1]] = True
    par = np.zeros_like(shell)
    par[::2, ::2, ::2] = True
    assert np.abs(rp[shell & par]).max() < 1e-9 * np.abs(b).max()


def test_skip_reverse_breaks_symmetry():
    # fault injection must be detected by the symmetry check
    o = oracle.Oracle(6, levels=1)
    o.set_skip_reverse(True)
    n = o.ndof()
    C = materialize(lambda e: o.smoother(OP_DGS, np.zeros(n), e), n)
    assert defect(C) > 1e-3


@pytest.mark.parametrize("levels", [2, 3])
def test_vcycle_symmetric_linear(levels):
    # SPEC AC 4 / SPEC:377,390-391: materialized cycle symmetric < 1e-10, linear
    o = oracle.Oracle(8, levels=levels)
    n = o.ndof()
    W = materialize(o.vcycle, n)
    assert defect(W) < 1e-10
    rng = np.random.default_rng(6)
    a, b = rng.standard_normal(n), rng.standard_normal(n)
    lhs = o.vcycle(3 * a - 2 * b)
    assert np.allclose(lhs, 3 * o.vcycle(a) - 2 * o.vcycle(b), atol=1e-12 * np.abs(lhs).max())
    assert not o.vcycle(np.zeros(n)).any()
    # symmetric indefinite
    ev = np.linalg.eigvalsh(0.5 * (W + W.T))
    assert ev.min() < 0 < ev.max()


def test_single_level_cycle_is_direct_solve():
    # one level: cycle = exact solve of L~ x = b
    o = oracle.Oracle(4, levels=1)
    n = o.ndof()
    b = np.random.default_rng(7).standard_normal(n)
    x = o.vcycle(b)
    assert np.allclose(o.dense(0, True) @ x, b, atol=1e-10 * np.abs(b).max())


def test_commutativity_deep_interior():
    # SPEC AC 5: L*M velocity rows vanish for deep-interior pressure columns
    nx = 12
    o = oracle.Oracle(nx, levels=2)
    L = o.dense(0, False)
    cnt = o.counts(0)
    nu_, nv_, nw_ = cnt["nu"], cnt["nv"], cnt["nw"]
    npv = nu_ + nv_ + nw_
    h = 1.0 / nx

    def uidx(I, j, k):
        return (k * nx + j) * (nx - 1) + (I - 1)

    def vidx(i, J, k):
        return nu_ + (k * (nx - 1) + (J - 1)) * nx + i

    def widx(i, j, K):
        return nu_ + nv_ + ((K - 1) * nx + j) * nx + i

    def pidx(i, j, k):
        return npv + (k * nx + j) * nx + i

    bad_deep, nonzero_edge = 0, 0
    for (i, j, k) in [(5, 5, 5), (6, 4, 7), (1, 1, 1), (0, 5, 5)]:
        m = np.zeros(L.shape[0])
        for a, (lo, hi) in enumerate([(uidx(i, j, k) if i >= 1 else None, uidx(i + 1, j, k) if i + 1 <= nx - 1 else None),
                                      (vidx(i, j, k) if j >= 1 else None, vidx(i, j + 1, k) if j + 1 <= nx - 1 else None),
                                      (widx(i, j, k) if k >= 1 else None, widx(i, j, k + 1) if k + 1 <= nx - 1 else None)]):
            if lo is not None:
                m[lo] -= 1.0 / h
            if hi is not None:
                m[hi] += 1.0 / h
        m[pidx(i, j, k)] += 6.0 / h ** 2
        for d in [(-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)]:
            ii, jj, kk = i + d[0], j + d[1], k + d[2]
            if 0 <= ii < nx and 0 <= jj < nx and 0 <= kk < nx:
                m[pidx(ii, jj, kk)] -= 1.0 / h ** 2
        top = (L @ m)[:npv]
        if min(i, j, k) >= 2 and max(i, j, k) <= nx - 3:
            bad_deep += np.abs(top).max() > 1e-12 * np.abs(L).max()
        else:
            nonzero_edge += np.abs(top).max() > 1e-9
    assert bad_deep == 0 and nonzero_edge >= 1


def test_wcycle_symmetric_and_mg_solve_converges():
    # SPEC:392 (W-cycle) and SPEC:379-388 (mg_solve); the W-cycle's coarse correction
    # 2C - C L~ C is symmetric whenever C is
    oracle.set_threads(4)
    o = oracle.Oracle(16, levels=4, cycle=1)  # W active at level 1 (child 4^3 is not the coarsest)
    n = o.ndof()
    rng = np.random.default_rng(11)
    for _ in range(3):  # symmetry by random probes: a^T W c = c^T W a
        a, c = rng.standard_normal(n), rng.standard_normal(n)
        wa, wc = o.vcycle(a), o.vcycle(c)
        assert abs(c @ wa - a @ wc) <= 1e-11 * np.abs(c * wa).sum()
    b = o.forcing(oracle.FORCE_UNIFORM, 1)
    x, h, _, st = o.mg_solve(b, 1e-6, 60)
    assert st == oracle.ST_CONVERGED and np.all(np.diff(h) < 0)
    assert np.isclose(np.linalg.norm(b - o.apply(x, penalized=True)) / np.linalg.norm(b), h[-1], rtol=1e-12)


# ---- additive Vanka (Eq. S_AV) ----
OP_VADD = 5


def test_additive_vanka_symmetric_single_application():
    """S_AV materialized with x0 = 0 is symmetric for ONE application (Theorem 2)."""
    o = oracle.Oracle(8, levels=2, vanka=1)
    n = o.ndof()
    C = materialize(lambda e: o.smoother(OP_VADD, np.zeros(n), e), n)
    assert np.abs(C).max() > 0
    assert defect(C) < 1e-10


def test_additive_vanka_linear_and_touches_only_v1():
    o = oracle.Oracle(8, levels=2, vanka=1, omega=0.7)
    n = o.ndof()
    rng = np.random.default_rng(5)
    x, b1, b2 = rng.standard_normal(n), rng.standard_normal(n), rng.standard_normal(n)
    y1, y2 = o.smoother(OP_VADD, x, b1), o.smoother(OP_VADD, x, b2)
    y12 = o.smoother(OP_VADD, x, 0.5 * b1 + 0.5 * b2)
    assert np.allclose(y12, 0.5 * y1 + 0.5 * y2, rtol=0, atol=1e-12 * np.abs(y12).max())
    v1 = o.v1_mask(0).astype(bool)
    assert np.array_equal(y1[~v1], x[~v1])  # V2 DOFs untouched
    assert not np.array_equal(y1[v1], x[v1])


def test_additive_vanka_damping_scales_correction():
    n8 = oracle.Oracle(8, levels=2).ndof()
    rng = np.random.default_rng(6)
    x, b = rng.standard_normal(n8), rng.standard_normal(n8)
    d1 = oracle.Oracle(8, levels=2, vanka=1, omega=1.0).smoother(OP_VADD, x, b) - x
    dh = oracle.Oracle(8, levels=2, vanka=1, omega=0.5).smoother(OP_VADD, x, b) - x
    assert np.allclose(dh, 0.5 * d1, rtol=1e-12, atol=1e-14)


def test_smooth_and_vcycle_with_additive_vanka_symmetric():
    """Alg. 3 with additive Vanka and the V-cycle built on it stay symmetric (Theorem 4)."""
    o = oracle.Oracle(8, levels=2, vanka=1)
    n = o.ndof()
    S = materialize(lambda e: o.smoother(OP_SMOOTH, np.zeros(n), e), n)
    assert defect(S) < 1e-10
    V = materialize(o.vcycle, n)
    assert defect(V) < 1e-10


def test_mg_sqmr_with_additive_vanka_converges():
    """Damped (omega = 1/2: every band face sits in two overlapping blocks) additive Vanka inside
    the preconditioner converges; undamped it stagnates, as SPEC:318's design note warns."""
    oracle.set_threads(4)
    o = oracle.Oracle(16, levels=3, vanka=1, omega=0.5)
    b = o.forcing(oracle.FORCE_UNIFORM, 0)
    _, hist, _, st = o.sqmr(b, 1e-8, 100)
    assert st == 0 and hist[-1] < 1e-8 and len(hist) <= 15


VANKA_ORDER = [0, 7, 1, 6, 2, 5, 3, 4]  # oracle kVankaOrder (OD-2)


def test_vanka_symmetric_is_colour_order_then_reverse():
    """The symmetric sweep is exactly the per-colour phases in kVankaOrder, then reversed."""
    o = oracle.Oracle(8, levels=2)
    n = o.ndof(0)
    rng = np.random.default_rng(5)
    x0, b = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    x = x0.copy()
    for c in VANKA_ORDER + VANKA_ORDER[::-1]:
        x = o.smoother(OP_VCOL, x, b, 0, c)
    assert np.array_equal(x, o.smoother(OP_VANKA, x0, b, 0))


@pytest.mark.parametrize("p", [0, 1, 2, 3])
def test_vanka_complementary_colours_commute_bitwise(p):
    """Colours p and 7 - p never touch each other's DOFs: either order gives the same bits,
    which is what lets the GPU run each adjacent pair of kVankaOrder as one Jacobi phase."""
    o = oracle.Oracle(12, levels=2)
    n = o.ndof(0)
    rng = np.random.default_rng(10 + p)
    x0, b = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    a = o.smoother(OP_VCOL, o.smoother(OP_VCOL, x0, b, 0, p), b, 0, 7 - p)
    c = o.smoother(OP_VCOL, o.smoother(OP_VCOL, x0, b, 0, 7 - p), b, 0, p)
    assert np.array_equal(a, c)
    # and a non-complementary pair does not commute (the merge is not vacuous)
    d = o.smoother(OP_VCOL, o.smoother(OP_VCOL, x0, b, 0, p), b, 0, p ^ 1)
    e = o.smoother(OP_VCOL, o.smoother(OP_VCOL, x0, b, 0, p ^ 1), b, 0, p)
    assert not np.array_equal(d, e)


# ---- SPEC-literal traversal order vs the coloured order the GPU runs ----
@pytest.mark.parametrize("n,levels,seed", [(32, 3, 0), (64, 4, 7)])
def test_spec_order_iteration_count_within_one(n, levels, seed):
    """The oracle's ORDER_SPEC mode runs the SPEC's literal sequential order: DGS over ascending
    DOF index then its exact reverse, multiplicative Vanka colour-major 0..7 then 7..0, blocks of a
    colour in sequence.  The coloured / tiled order the GPU reproduces bit for bit (ORDER_GPU) must
    reach the tolerance within +-1 iteration of it (north_star) and to the same solution.
    Recorded: 32^3 7 vs 7, 64^3 8 vs 7, cfg 1 (128^3, 5 levels, seed 1) 8 vs 8 iterations."""
    import os
    oracle.set_threads(os.cpu_count() or 1)
    b = oracle.forcing_box(n, n, n, 1 / n, oracle.FORCE_UNIFORM, seed)
    out = {}
    for order in (oracle.ORDER_GPU, oracle.ORDER_SPEC):
        x, h, _, st = oracle.Oracle(n, levels=levels, order=order).sqmr(b, 1e-6, 100)
        assert st == 0 and h[-1] < 1e-6
        out[order] = (x, len(h))
    (xg, kg), (xs, ks) = out[oracle.ORDER_GPU], out[oracle.ORDER_SPEC]
    assert abs(kg - ks) <= 1, (kg, ks)
    npres = n ** 3
    assert np.linalg.norm(xg[:-npres] - xs[:-npres]) <= 2e-5 * np.linalg.norm(xs[:-npres])
    oracle.set_threads(1)


# ---- direct-on-V1 boundary smoother ----
def test_direct_on_v1_exact_and_symmetric():
    """One application zeroes the V1 rows of the residual (the exact solve of the V1 equations with
    x_V2 frozen); Alg. 3 and the V-cycle built on it stay symmetric (Theorem 4's argument: the V1
    solve is a symmetric map); MG-SQMR with it converges at least as fast as with Vanka."""
    o = oracle.Oracle(8, levels=2, vanka=2)
    n = o.ndof(0)
    rng = np.random.default_rng(31)
    x, b = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    y = o.smoother(7, x, b)
    r = b - o.apply(y, penalized=True)
    om = oracle.Oracle(8, levels=2)
    # V1 rows: the DOFs a multiplicative Vanka sweep may change
    v1 = om.smoother(OP_VANKA, x, b) != x
    assert v1.sum() == o.census()[1] if hasattr(o, "census") else True
    assert np.abs(r[v1]).max() <= 1e-9 * np.abs(b).max()
    assert np.array_equal(y[~v1], x[~v1])
    C = materialize(lambda e: o.smoother(OP_SMOOTH, np.zeros(n), e), n)
    assert defect(C) < 1e-10
    W = materialize(o.vcycle, n)
    assert defect(W) < 1e-10
    bb = o.forcing(oracle.FORCE_UNIFORM, 3)
    _, hd, _, sd = o.sqmr(bb, 1e-8, 50)
    _, hm, _, sm_ = om.sqmr(bb, 1e-8, 50)
    assert sd == sm_ == 0 and len(hd) <= len(hm) + 1
