"""GPU parity: every hot-path op of libsmg.so (through the C-ABI) against the CPU
oracle on identical seeded inputs.

Per-point ops follow the shared arithmetic contract (no FMA on
either side), so they are required to be BIT-IDENTICAL.  Only SQMR's inner
products use a different (deterministic) summation order; solve-level parity is
held to the north_star bar: per-iteration residuals within 1e-10 relative,
iteration count within +-1, solution within 1e-6 relative L2.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle
import paper_2312_10615_b200 as smg

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pair16():
    oracle.set_threads(4)
    o = oracle.Oracle(16, levels=3)
    s = smg.Solver(16, levels=3)
    yield o, s
    s.close()


def rnd(n, seed):
    return np.random.default_rng(seed).uniform(-1, 1, n)


def same(a, b):
    assert a.shape == b.shape
    if not np.array_equal(a, b):
        d = np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)
        pytest.fail(f"not bit-identical: max rel diff {d:.3e}")


@pytest.mark.parametrize("level", [0, 1, 2])
@pytest.mark.parametrize("pen", [False, True])
def test_apply(pair16, level, pen):
    o, s = pair16
    x = rnd(o.ndof(level), 10 + level)
    same(s.apply(x, level, pen), o.apply(x, level, pen))


@pytest.mark.parametrize("level", [0, 1])
def test_residual(pair16, level):
    o, s = pair16
    n = o.ndof(level)
    x, b = rnd(n, 1), rnd(n, 2)
    same(s.residual(x, b, level), o.residual(x, b, level))


def test_counts(pair16):
    o, s = pair16
    for l in range(3):
        assert s.counts(l) == o.counts(l)
        assert s.ndof(l) == o.ndof(l)


@pytest.mark.parametrize("phase", list(range(20)))
def test_dgs_phase(pair16, phase):
    o, s = pair16
    n = o.ndof(0)
    x, b = rnd(n, 3 + phase), rnd(n, 4)
    same(s.smoother(smg.OP_DGS_PHASE, x, b, arg=phase), o.smoother(0, x, b, arg=phase))


@pytest.mark.parametrize("colour", list(range(8)))
def test_vanka_colour(pair16, colour):
    o, s = pair16
    n = o.ndof(0)
    x, b = rnd(n, 30 + colour), rnd(n, 5)
    same(s.smoother(smg.OP_VANKA_COLOUR, x, b, arg=colour), o.smoother(2, x, b, arg=colour))


@pytest.mark.parametrize("op,oop", [(smg.OP_DGS_SYM, 1), (smg.OP_VANKA_SYM, 3), (smg.OP_SMOOTH, 4)])
@pytest.mark.parametrize("level", [0, 1])
def test_symmetric_smoothers(pair16, op, oop, level):
    o, s = pair16
    n = o.ndof(level)
    x, b = rnd(n, 6), rnd(n, 7)
    same(s.smoother(op, x, b, level), o.smoother(oop, x, b, level))
    z = np.zeros(n)
    same(s.smoother(op, z, b, level), o.smoother(oop, z, b, level))


@pytest.mark.parametrize("level", [0, 1])
def test_transfers(pair16, level):
    o, s = pair16
    rf = rnd(o.ndof(level), 8)
    xc = rnd(o.ndof(level + 1), 9)
    same(s.restrict(rf, level), o.restrict(rf, level))
    same(s.prolong(xc, level), o.prolong(xc, level))


def test_coarse_solve(pair16):
    o, s = pair16
    b = rnd(o.ndof(2), 11)
    same(s.coarse_solve(b), o.coarse_solve(b))


def test_vcycle(pair16):
    o, s = pair16
    b = rnd(o.ndof(0), 12)
    same(s.vcycle(b), o.vcycle(b))


@pytest.mark.parametrize("mode", ["1", "2"])
def test_sweep_sync_modes_bitwise(pair16, mode, monkeypatch):
    """Grid-wide (1) and single-cluster (2) barrier variants of the sweeps agree bit for bit."""
    o, s = pair16
    monkeypatch.setenv("SMG_SYNC_MODE", mode)
    for level in (0, 1):
        n = o.ndof(level)
        x, b = rnd(n, 40 + level), rnd(n, 41)
        same(s.smoother(smg.OP_SMOOTH, x, b, level), o.smoother(4, x, b, level))
    b = rnd(o.ndof(0), 42)
    same(s.vcycle(b), o.vcycle(b))


def test_vcycle_symmetry_gpu_materialized():
    # SURVEY §7 f1 / SPEC AC 4 on the GPU map itself
    s = smg.Solver(8, levels=2)
    n = s.ndof()
    W = np.zeros((n, n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        W[:, j] = s.vcycle(e)
    assert np.linalg.norm(W - W.T) / np.linalg.norm(W) < 1e-10
    s.close()


def test_fault_injection_detected_on_gpu():
    s = smg.Solver(6, levels=1, flags=smg.FLAG_SKIP_REVERSE_DGS)
    n = s.ndof()
    C = np.zeros((n, n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        C[:, j] = s.smoother(smg.OP_DGS_SYM, np.zeros(n), e)
    assert np.linalg.norm(C - C.T) / np.linalg.norm(C) > 1e-3
    s.close()


def check_solve(o, s, b, tol, maxit=100):
    xo, ho, _, sto = o.sqmr(b, tol=tol, maxit=maxit)
    xg, hg, _, stg = s.sqmr(b, tol=tol, maxit=maxit)
    assert sto == stg == smg.SMG_CONVERGED
    assert abs(len(ho) - len(hg)) <= 1
    k = min(len(ho), len(hg))
    rel = np.abs(hg[:k] - ho[:k]) / ho[:k]
    assert rel.max() < 1e-10, rel  # north_star bar
    # canonical reductions (OD-12): the whole solve is bit-identical
    assert np.array_equal(hg, ho) and np.array_equal(xg, xo), rel.max()
    npres = o.counts(0)["np"]
    assert np.linalg.norm(xg[:-npres] - xo[:-npres]) / np.linalg.norm(xo[:-npres]) < 1e-6
    pg = xg[-npres:] - xg[-npres:].mean()
    po = xo[-npres:] - xo[-npres:].mean()
    assert np.linalg.norm(pg - po) / np.linalg.norm(po) < 1e-6
    return hg


@pytest.mark.parametrize("n,levels,kind,seed", [(16, 2, 0, 0), (32, 3, 0, 0), (32, 3, 1, 2), (64, 4, 0, 3)])
def test_sqmr_history_parity(n, levels, kind, seed):
    oracle.set_threads(os.cpu_count() or 1)
    o = oracle.Oracle(n, levels=levels)
    s = smg.Solver(n, levels=levels)
    b = o.forcing(kind, seed)
    check_solve(o, s, b, 1e-6)
    s.close()


def test_channel_anisotropic_parity():
    # cfg-4 shape (4:1:1 box, h = 1/ny), reduced
    oracle.set_threads(os.cpu_count() or 1)
    o = oracle.Oracle(64, 16, 16, h=1 / 16, levels=3)
    s = smg.Solver(64, 16, 16, h=1 / 16, levels=3)
    b = o.forcing(oracle.FORCE_CHANNEL, 4)
    check_solve(o, s, b, 1e-8)
    s.close()


def field_digest(x, nx, ny, nz):
    """tests/golden/make_golden.py's digest: per-field L2 and sha256 of u, v, w, mean-free p."""
    nu, nv, nw = (nx - 1) * ny * nz, nx * (ny - 1) * nz, nx * ny * (nz - 1)
    parts = {"u": x[:nu], "v": x[nu:nu + nv], "w": x[nu + nv:nu + nv + nw]}
    p = x[nu + nv + nw:]
    parts["p_meanfree"] = p - p.mean()
    return {k: {"l2": float(np.linalg.norm(v)),
                "sha256": hashlib.sha256(np.ascontiguousarray(v + 0.0).tobytes()).hexdigest()}
            for k, v in parts.items()}


GOLDEN = sorted(f[:-len("_history.json")] for f in os.listdir(os.path.join(ROOT, "tests", "golden"))
                if f.endswith("_history.json"))


@pytest.mark.parametrize("name", GOLDEN)
def test_golden_history_and_solution(name):
    """BASELINE configs against the committed oracle goldens (cfg 0-2: whole solves; cfg 3/4: the
    first iterations, generated on the GPU box's host): the residual history bit for bit, and the
    whole solution vector -- sha256 of u, v, w and the mean-free p -- bit for bit, plus the
    north_star bars (1e-10 per iteration, +-1 iteration, 1e-6 relative L2 per field)."""
    g = json.load(open(os.path.join(ROOT, "tests", "golden", f"{name}_history.json")))
    nx, ny, nz = g["grid"]
    s = smg.Solver(nx, ny, nz, h=g.get("h", 1.0 / nx), levels=g["levels"])
    b = smg.forcing(nx, ny, nz, h=g.get("h", 1.0 / nx), kind=g["forcing"], seed=g["seed"])
    assert hashlib.sha256(b.tobytes()).hexdigest() == g["b_sha256"]
    x, h, _, st = s.sqmr(b, tol=g["tol"], maxit=g.get("maxit", 200))
    s.close()
    assert st == g["status"]
    assert abs(len(h) - g["iterations"]) <= 1
    k = min(len(h), g["iterations"])
    rel = np.abs(h[:k] - np.array(g["history"][:k])) / np.array(g["history"][:k])
    assert rel.max() < 1e-10, rel
    assert h.tolist() == g["history"]  # bit-identical (canonical reductions, OD-12)
    got = field_digest(x, nx, ny, nz)
    if "fields" in g:
        for f, d in g["fields"].items():
            assert abs(got[f]["l2"] - d["l2"]) <= 1e-6 * max(d["l2"], 1e-300), f
            assert got[f]["sha256"] == d["sha256"], f"{name}: field {f} not bit-identical"
    npres = nx * ny * nz
    assert abs(np.linalg.norm(x[:-npres]) - g["u_norm"]) / g["u_norm"] < 1e-6


@pytest.mark.parametrize("kw", [{}, {"devices": [0, 0]}])
def test_sqmr_split_and_fused_updates_bitwise(kw, monkeypatch):
    """The SQMR vector updates as streaming passes before the stencil kernels (default) and evaluated
    inside them (SMG_SQMR_SPLIT=0) give the same bits -- single part and two z-slab parts (ghost planes)."""
    out = []
    for split in ("1", "0"):
        monkeypatch.setenv("SMG_SQMR_SPLIT", split)
        s = smg.Solver(32, levels=3, **kw)
        x, h, _, st = s.sqmr(smg.forcing(32, seed=9), 1e-9, 50)
        s.close()
        out.append((x, h, st))
    assert out[0][2] == out[1][2] == smg.SMG_CONVERGED
    same(out[0][1], out[1][1])
    same(out[0][0], out[1][0])


def test_edge_cases():
    s = smg.Solver(8, levels=2)
    n = s.ndof()
    x, h, _, st = s.sqmr(np.zeros(n), 1e-6, 10)
    assert st == smg.SMG_CONVERGED and len(h) == 0 and not x.any()
    x, h, _, st = s.sqmr(smg.forcing(8, seed=1), 1e-14, 2)
    assert st == smg.SMG_MAX_ITERATIONS and len(h) == 2
    with pytest.raises(ValueError):
        s.apply(np.zeros(n + 1))  # length mismatch
    with pytest.raises(smg.SmgError):
        s.smoother(smg.OP_DGS_PHASE, np.zeros(n), np.zeros(n), arg=20)
    with pytest.raises(smg.SmgError):
        s.smoother(99, np.zeros(n), np.zeros(n))
    s.close()


def test_resident_path_matches_e2e():
    s = smg.Solver(32, levels=3)
    b = smg.forcing(32, seed=0)
    x1, h1, _, st1 = s.sqmr(b, 1e-6, 100)
    s.set_rhs(b)
    h2, st2 = s.solve_resident(1e-6, 100)
    x2 = s.solution()
    assert st1 == st2 == 0 and np.array_equal(h1, h2) and np.array_equal(x1, x2)  # deterministic
    t = s.timing()
    assert t["iterations"] == len(h2) and t["solve_ms"] > 0 and t["kernel_launches"] > 100
    s.close()


@pytest.mark.parametrize("n,levels", [(32, 3), (64, 4)])
def test_mg_solve_and_wcycle_bitwise(n, levels):
    """SPEC:379-388 (mg_solve) and SPEC:395 (W-cycle) against the oracle, bit for bit."""
    oracle.set_threads(os.cpu_count() or 1)
    b = smg.forcing(n, seed=5)
    for cyc in (0, 1):
        o = oracle.Oracle(n, levels=levels, cycle=cyc)
        s = smg.Solver(n, levels=levels, cycle=cyc)
        xo, ho, _, sto = o.mg_solve(b, 1e-6, 60)
        xg, hg, _, stg = s.mg_solve(b, 1e-6, 60)
        assert sto == stg == smg.SMG_CONVERGED
        assert np.array_equal(ho, hg) and np.array_equal(xo, xg)
        xo, ho, _, _ = o.sqmr(b, 1e-6, 60)
        xg, hg, _, _ = s.sqmr(b, 1e-6, 60)
        assert np.array_equal(ho, hg) and np.array_equal(xo, xg)
        s.close()


@pytest.mark.parametrize("dims,levels,parts", [((16, 16, 16), 2, 1), ((32, 16, 16), 2, 1), ((32, 32, 32), 3, 2)])
def test_unpreconditioned_sqmr_bitwise(dims, levels, parts):
    """solve_driver method `sqmr`: Alg. 4 with the identity preconditioner
    (SMG_FLAG_NO_PRECOND) against the oracle's precond = 0 run, bit for bit -- slow to converge by
    design (PAPER Fig. 8: "the pure SQMR ... fails"), so the history is compared, not the status."""
    nx, ny, nz = dims
    o = oracle.Oracle(nx, ny, nz, h=1 / ny, levels=levels)
    kw = dict(devices=[0] * parts) if parts > 1 else {}
    s = smg.Solver(nx, ny, nz, h=1 / ny, levels=levels, flags=smg.FLAG_NO_PRECOND, **kw)
    b = o.forcing(oracle.FORCE_UNIFORM, 21)
    xo, ho, _, sto = o.sqmr(b, 1e-6, 60, precond=False)
    xg, hg, _, stg = s.sqmr(b, 1e-6, 60)
    assert sto == stg and len(ho) == len(hg) == 60
    assert np.array_equal(ho, hg) and np.array_equal(xo, xg)
    assert hg[-1] < hg[0]
    s.close()


@pytest.mark.parametrize("dims,levels", [((8, 8, 8), 2), ((16, 8, 8), 2), ((16, 16, 16), 3)])
def test_direct_on_v1_bitwise(dims, levels):
    """Direct-on-V1 boundary smoother (params.vanka = 2): the exact solve of the V1
    equations through the dense symmetric inverse of the V1 x V1 sub-block of L~ -- one application,
    Alg. 3 with it, the V-cycle and MG-SQMR bit-identical to the oracle; the V1 residual vanishes."""
    oracle.set_threads(os.cpu_count() or 1)
    nx, ny, nz = dims
    o = oracle.Oracle(nx, ny, nz, h=1 / ny, levels=levels, vanka=2)
    s = smg.Solver(nx, ny, nz, h=1 / ny, levels=levels, vanka=smg.VANKA_DIRECT)
    n = o.ndof(0)
    x, b = rnd(n, 90), rnd(n, 91)
    y = s.smoother(smg.OP_VANKA_DIRECT, x, b)
    same(y, o.smoother(7, x, b))
    y2 = s.smoother(smg.OP_VANKA_DIRECT, y, b)  # idempotent up to rounding
    assert np.abs(y2 - y).max() <= 1e-10 * np.abs(y).max()
    same(s.smoother(smg.OP_SMOOTH, x, b), o.smoother(4, x, b))
    bb = o.forcing(oracle.FORCE_UNIFORM, 13)
    same(s.vcycle(bb), o.vcycle(bb))
    xo, ho, _, sto = o.sqmr(bb, 1e-8, 40)
    xg, hg, _, stg = s.sqmr(bb, 1e-8, 40)
    assert sto == stg == smg.SMG_CONVERGED and np.array_equal(ho, hg) and np.array_equal(xo, xg)
    s.close()


def test_wcycle_symmetric_gpu():
    s = smg.Solver(16, levels=4, cycle=1)  # 16 -> 8 -> 4 -> 2: W active at level 1
    o = oracle.Oracle(16, levels=4, cycle=1)
    n = s.ndof()
    rng = np.random.default_rng(12)
    for _ in range(3):
        a, c = rng.standard_normal(n), rng.standard_normal(n)
        wa, wc = s.vcycle(a), s.vcycle(c)
        assert abs(c @ wa - a @ wc) <= 1e-11 * np.abs(c * wa).sum()
        assert np.array_equal(wa, o.vcycle(a))
    s.close()


@pytest.mark.parametrize("nu,bw,eta,gamma", [(2, 1, 1.0, 1e-3), (3, 1, 1.0, 1e-3), (1, 2, 1.0, 1e-3),
                                             (1, 1, 1e-3, 1e-3), (2, 2, 0.5, 1e-2)])
def test_parameter_sweep_bitwise(nu, bw, eta, gamma):
    """SPEC AC 3 parameter range (nu in {1,2,3}), band width, eta/gamma: whole solve bit-identical."""
    oracle.set_threads(os.cpu_count() or 1)
    o = oracle.Oracle(32, levels=3, nu=nu, band_width=bw, eta=eta, gamma=gamma)
    s = smg.Solver(32, levels=3, nu=nu, band_width=bw, eta=eta, gamma=gamma)
    b = o.forcing(oracle.FORCE_UNIFORM, 9)
    assert np.array_equal(s.vcycle(b), o.vcycle(b))
    xo, ho, _, sto = o.sqmr(b, 1e-6, 100)
    xg, hg, _, stg = s.sqmr(b, 1e-6, 100)
    assert sto == stg and np.array_equal(ho, hg) and np.array_equal(xo, xg)
    s.close()


def test_lid_driven_cavity_bitwise():
    """The paper's 3-D cavity: zero force, lid u = 1; GPU solve == oracle, flow follows the lid."""
    oracle.set_threads(os.cpu_count() or 1)
    n = 32
    b = smg.cavity_rhs(n, eta=1e-3)
    o = oracle.Oracle(n, levels=3, eta=1e-3)
    s = smg.Solver(n, levels=3, eta=1e-3)
    xo, ho, _, sto = o.sqmr(b, 1e-8, 100)
    xg, hg, _, stg = s.sqmr(b, 1e-8, 100)
    assert sto == stg == smg.SMG_CONVERGED and np.array_equal(ho, hg) and np.array_equal(xo, xg)
    u = xg[: (n - 1) * n * n].reshape(n, n, n - 1)
    assert u[:, -1, :].mean() > 0.1 and u[:, 0, :].mean() < u[:, -1, :].mean()


@pytest.mark.parametrize("mode", [{}, {"SMG_SYNC_MODE": "1"}, {"SMG_SYNC_MODE": "2"}, {"SMG_VANKA_PP": "0"},
                                  {"SMG_VANKA_PHASES": "1"},
                                  {"SMG_VANKA_KERNELS": "1"},
                                  {"SMG_VANKA_PAIRS": "0"}, {"SMG_VANKA_PAIRS": "2", "SMG_SYNC_MODE": "1"},
                                  {"SMG_VANKA_PAIRS": "2", "SMG_VANKA_KERNELS": "1"},
                                  {"SMG_VANKA_PAIRS": "0", "SMG_VANKA_PHASES": "1"}])
def test_vanka_merged_phase_bitwise(mode, monkeypatch):
    """Complementary colour pairs (p, 7 - p) share one Jacobi phase (8 phases per sweep): every
    sweep variant, merged or not, stays bit-identical to the oracle's 16-phase order."""
    for k, v in mode.items():
        monkeypatch.setenv(k, v)
    oracle.set_threads(4)
    o = oracle.Oracle(32, levels=3)
    s = smg.Solver(32, levels=3)
    for level in (0, 1):
        n = o.ndof(level)
        x, b = rnd(n, 70 + level), rnd(n, 71 + level)
        same(s.smoother(smg.OP_VANKA_SYM, x, b, level), o.smoother(3, x, b, level))
        same(s.smoother(smg.OP_SMOOTH, x, b, level), o.smoother(4, x, b, level))
    s.close()


@pytest.mark.parametrize("n,levels", [(64, 4), (128, 5)])
def test_vanka_merged_matches_unmerged(n, levels, monkeypatch):
    """Large levels (grid ping-pong sweeps): merged pairs (8-phase) == unmerged (16-phase) sweep."""
    out = []
    # 2: merge all pairs even where the default would not; REFRESH_IN=0: separate refresh launch
    for env in ({"SMG_VANKA_PAIRS": "0"}, {"SMG_VANKA_PAIRS": "2"}, {"SMG_VANKA_REFRESH_IN": "0"}):
        for k in ("SMG_VANKA_PAIRS", "SMG_VANKA_REFRESH_IN"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        s = smg.Solver(n, levels=levels)
        x = np.random.default_rng(n).uniform(-1, 1, s.ndof())
        b = np.random.default_rng(n + 1).uniform(-1, 1, s.ndof())
        out.append((s.smoother(smg.OP_VANKA_SYM, x, b), s.smoother(smg.OP_SMOOTH, x, b), s.vcycle(b)))
        s.close()
    for o in out[1:]:
        for a, c in zip(o, out[0]):
            same(a, c)


def test_vanka_per_launch_large_level_matches_persistent(monkeypatch):
    """256^3 (lists beyond the persistent ping-pong sweep): the default -- a delta and an apply launch
    per merged phase, 8 lanes per block -- == one ping-pong launch per merged phase == unmerged
    ping-pong launches == unmerged per-phase delta / apply launches."""
    out = []
    for env in ({}, {"SMG_VANKA_KERNELS": "1"}, {"SMG_VANKA_KERNELS": "1", "SMG_VANKA_PAIRS": "0"},
                {"SMG_VANKA_KERNELS": "0", "SMG_VANKA_PAIRS": "0"}):
        for k in ("SMG_VANKA_PAIRS", "SMG_VANKA_KERNELS"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        s = smg.Solver(256, levels=6)
        x = np.random.default_rng(3).uniform(-1, 1, s.ndof())
        b = np.random.default_rng(4).uniform(-1, 1, s.ndof())
        out.append(s.smoother(smg.OP_VANKA_SYM, x, b))
        s.close()
    for o in out[1:]:
        same(o, out[0])


@pytest.mark.parametrize("dims,levels,omega", [((16, 16, 16), 3, 0.5), ((32, 32, 32), 3, 0.5), ((64, 16, 16), 3, 1.0),
                                               ((48, 40, 24), 3, 0.7)])
def test_additive_vanka_bitwise(dims, levels, omega):
    """Additive Vanka: one application, Alg. 3 with it, V-cycle and MG-SQMR bit-identical."""
    oracle.set_threads(os.cpu_count() or 1)
    nx, ny, nz = dims
    o = oracle.Oracle(nx, ny, nz, h=1 / ny, levels=levels, vanka=1, omega=omega)
    s = smg.Solver(nx, ny, nz, h=1 / ny, levels=levels, vanka=smg.VANKA_ADDITIVE, omega=omega)
    for level in range(levels - 1):
        n = o.ndof(level)
        x, b = rnd(n, 80 + level), rnd(n, 81 + level)
        same(s.smoother(smg.OP_VANKA_ADD, x, b, level), o.smoother(5, x, b, level))
        same(s.smoother(smg.OP_SMOOTH, x, b, level), o.smoother(4, x, b, level))
    b = o.forcing(oracle.FORCE_UNIFORM, 12)
    same(s.vcycle(b), o.vcycle(b))
    xo, ho, _, sto = o.sqmr(b, 1e-8, 30)
    xg, hg, _, stg = s.sqmr(b, 1e-8, 30)
    assert sto == stg and np.array_equal(ho, hg) and np.array_equal(xo, xg)
    s.close()


@pytest.mark.parametrize("zseg", ["1", "2", "3", "5"])
@pytest.mark.parametrize("dims", [(16, 16, 16), (24, 16, 40)])
def test_restrict_zmarch_bitwise(dims, zseg, monkeypatch):
    """z-marching restriction (k_restrict_zm: per-plane partials reused across planes, ragged
    segments) == the oracle's R = P^T/8, bit for bit, on every level (prolongation: per cell)."""
    monkeypatch.setenv("SMG_RESTRICT_ZSEG", zseg)
    nx, ny, nz = dims
    o = oracle.Oracle(nx, ny, nz, h=1 / ny, levels=3)
    s = smg.Solver(nx, ny, nz, h=1 / ny, levels=3)
    try:
        for level in (0, 1):
            rf = rnd(o.ndof(level), 21 + level)
            same(s.restrict(rf, level), o.restrict(rf, level))
            xc = rnd(o.ndof(level + 1), 31 + level)
            same(s.prolong(xc, level), o.prolong(xc, level))
        b = rnd(o.ndof(0), 23)
        same(s.vcycle(b), o.vcycle(b))
    finally:
        s.close()


def test_restrict_zmarch_matches_per_cell_at_256():
    """At 256^3 the default restriction marches (segments of several planes): same results as
    the per-cell kernel (SMG_RESTRICT_ZM=0)."""
    out = []
    for zm in ("1", "0"):
        os.environ["SMG_RESTRICT_ZM"] = zm
        try:
            s = smg.Solver(256, levels=6)
            rf = rnd(s.ndof(0), 29)
            out.append(s.restrict(rf, 0))
            s.close()
        finally:
            os.environ.pop("SMG_RESTRICT_ZM", None)
    same(out[0], out[1])
