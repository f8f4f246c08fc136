"""Oracle MG-SQMR against direct solves (SPEC AC 6, 11-12).

The reference pins no solution vectors; a dense direct solve of the same L with
the pressure constant fixed by a Lagrange multiplier is the independent check.
"""
import numpy as np
import pytest

import oracle


def direct_solution(o, b):
    L = o.dense(0, False)
    c = o.counts(0)
    n = L.shape[0]
    e = np.zeros(n)
    e[n - c["np"]:] = 1.0
    A = np.zeros((n + 1, n + 1))
    A[:n, :n] = L
    A[:n, n] = e
    A[n, :n] = e
    sol = np.linalg.solve(A, np.append(b, 0.0))
    return sol[:n]


def split(o, x):
    c = o.counts(0)
    npres = c["np"]
    u, p = x[:-npres], x[-npres:]
    return u, p - p.mean()


@pytest.mark.parametrize("levels", [2, 3])
def test_mgsqmr_matches_direct_8(levels):
    oracle.set_threads(1)
    o = oracle.Oracle(8, levels=levels)
    b = o.forcing(oracle.FORCE_UNIFORM, 0)
    x, hist, _, st = o.sqmr(b, tol=1e-10, maxit=100)
    assert st == oracle.ST_CONVERGED and hist[-1] < 1e-10
    xd = direct_solution(o, b)
    u, p = split(o, x)
    ud, pd = split(o, xd)
    assert np.linalg.norm(u - ud) / np.linalg.norm(ud) < 1e-8
    assert np.linalg.norm(p - pd) / np.linalg.norm(pd) < 1e-8


def test_history_is_true_residual():
    # reported history equals an independently recomputed residual
    o = oracle.Oracle(8, levels=2)
    b = o.forcing(oracle.FORCE_UNIFORM, 5)
    x, hist, _, st = o.sqmr(b, tol=1e-6, maxit=100)
    r = b - o.apply(x)
    assert np.isclose(np.linalg.norm(r) / np.linalg.norm(b), hist[-1], rtol=1e-12)


def test_zero_rhs_converges_at_zero():
    # b = 0 -> x = 0, converged at iteration 0
    o = oracle.Oracle(8, levels=2)
    x, hist, _, st = o.sqmr(np.zeros(o.ndof()), 1e-6, 10)
    assert st == oracle.ST_CONVERGED and len(hist) == 0 and not x.any()


def test_maxit_status():
    o = oracle.Oracle(8, levels=2)
    x, hist, _, st = o.sqmr(o.forcing(0, 1), 1e-14, 2)
    assert st == oracle.ST_MAXIT and len(hist) == 2


def test_unpreconditioned_sqmr_runs():
    # method sqmr (identity preconditioner) on the same L
    o = oracle.Oracle(4, levels=1)
    x, hist, _, st = o.sqmr(o.forcing(0, 2), 1e-8, 400, precond=False)
    assert hist[-1] < hist[0] and st in (oracle.ST_CONVERGED, oracle.ST_MAXIT)


def test_ac12_cavity_32_three_levels():
    # SPEC AC 12: 32^3, 3-level MG-SQMR converges to 1e-8 within 100 iterations
    oracle.set_threads(4)
    o = oracle.Oracle(32, levels=3)
    b = o.forcing(oracle.FORCE_UNIFORM, 0)
    x, hist, _, st = o.sqmr(b, tol=1e-8, maxit=100)
    assert st == oracle.ST_CONVERGED and len(hist) <= 100


def test_divergence_control():
    # SPEC AC 9: ||B u||_inf <= 10 tol ||b|| / sqrt(N) for a converged run
    o = oracle.Oracle(16, levels=2)
    b = o.forcing(oracle.FORCE_UNIFORM, 3)
    tol = 1e-8
    x, hist, _, st = o.sqmr(b, tol=tol, maxit=100)
    assert st == oracle.ST_CONVERGED
    c = o.counts(0)
    bu = o.apply(x)[-c["np"]:]  # continuity rows of L x = B u
    assert np.abs(bu).max() <= 10 * tol * np.linalg.norm(b) / np.sqrt(o.ndof())
