"""Tile-ordered DGS (OD-1 rev. 2): the TMA-staged shared-memory tile kernel
(k_dgs_tile) against the oracle's tile-ordered sweep, bit for bit, on levels forced to be
tiled (tile_min=1) at sizes the oracle finishes in seconds -- including ragged tile grids
(odd tile counts per axis), the forward half alone, single phases per tile colour, the
whole smooth / V-cycle / MG-SQMR, and the z-slab path (ghost-plane push + refresh)."""
import os

import numpy as np
import pytest

import oracle
import paper_2312_10615_b200 as smg

pytestmark = pytest.mark.gpu


def rnd(n, seed):
    return np.random.default_rng(seed).uniform(-1, 1, n)


def same(a, b):
    assert a.shape == b.shape
    if not np.array_equal(a, b):
        d = np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)
        pytest.fail(f"not bit-identical: max rel diff {d:.3e}")


SHAPES = [((32, 16, 16), 2), ((64, 32, 32), 3), ((48, 40, 24), 3), ((64, 64, 64), 4)]


@pytest.mark.parametrize("dims,levels", SHAPES)
def test_tiled_sweep_smooth_vcycle_bitwise(dims, levels):
    oracle.set_threads(os.cpu_count() or 1)
    nx, ny, nz = dims
    o = oracle.Oracle(nx, ny, nz, h=1 / ny, levels=levels, tile_min=1)
    s = smg.Solver(nx, ny, nz, h=1 / ny, levels=levels, tile_min=1)
    assert o.dgs_tile(0) == smg.dgs_tile(nx, ny, nz, 0, 1) == (8, 16, 8, 8)
    n = o.ndof(0)
    x, b = rnd(n, 1), rnd(n, 2)
    same(s.smoother(smg.OP_DGS_SYM, x, b), o.smoother(1, x, b))
    same(s.smoother(smg.OP_SMOOTH, x, b), o.smoother(4, x, b))
    bb = o.forcing(oracle.FORCE_UNIFORM, 3)
    same(s.vcycle(bb), o.vcycle(bb))
    xo, ho, _, sto = o.sqmr(bb, 1e-8, 40)
    xg, hg, _, stg = s.sqmr(bb, 1e-8, 40)
    assert sto == stg == smg.SMG_CONVERGED and np.array_equal(ho, hg) and np.array_equal(xo, xg)
    s.close()


def test_tiled_forward_half_and_phases_bitwise():
    """Forward half alone (FLAG_SKIP_REVERSE_DGS) and every single phase of every tile colour."""
    oracle.set_threads(os.cpu_count() or 1)
    dims = (48, 40, 24)
    o = oracle.Oracle(*dims, h=1 / 40, levels=3, tile_min=1)
    o.set_skip_reverse(True)
    s = smg.Solver(*dims, h=1 / 40, levels=3, tile_min=1, flags=smg.FLAG_SKIP_REVERSE_DGS)
    n = o.ndof(0)
    x, b = rnd(n, 4), rnd(n, 5)
    same(s.smoother(smg.OP_DGS_SYM, x, b), o.smoother(1, x, b))
    s.close()
    o.set_skip_reverse(False)
    s = smg.Solver(*dims, h=1 / 40, levels=3, tile_min=1)
    for T in (0, 3, 7):
        for ph in range(20):
            arg = ph + 32 * T
            same(s.smoother(smg.OP_DGS_PHASE, x, b, arg=arg), o.smoother(0, x, b, arg=arg))
    s.close()


def test_tiled_matches_untiled_rule_and_default():
    """The tiling rule is the same function on both sides; 256^3 is tiled by default, 128^3 not."""
    for dims in [(128, 128, 128), (64, 64, 64), (256, 256, 256), (1024, 256, 256), (48, 40, 24), (40, 16, 16)]:
        for lv in range(3):
            for tm in (0, 1, -1):
                got = smg.dgs_tile(*dims, lv, tm)
                nx, ny, nz = (d >> lv for d in dims)
                cells = nx * ny * nz
                thr = (1 << 24) if tm == 0 else tm
                tiled = tm >= 0 and cells >= thr and nx % 16 == 0 and ny % 8 == 0 and nz % 8 == 0 and \
                    nx >= 32 and ny >= 16 and nz >= 16
                assert got == ((8, 16, 8, 8) if tiled else (1, 0, 0, 0)), (dims, lv, tm, got)


@pytest.mark.parametrize("dims,levels,parts", [((64, 64, 64), 4, 2), ((64, 64, 64), 4, 4), ((32, 32, 64), 3, 4),
                                               ((48, 40, 48), 4, 2)])
def test_tiled_slabs_bitwise(dims, levels, parts):
    """z-slab parts with tiled levels: per tile colour one launch, the ghost-plane push of the
    boundary tiles' pressure / w-face updates, then the halo refresh -- bit-identical to one part."""
    nx, ny, nz = dims
    one = smg.Solver(nx, ny, nz, h=1 / ny, levels=levels, tile_min=1)
    many = smg.Solver(nx, ny, nz, h=1 / ny, levels=levels, tile_min=1, devices=[0] * parts)
    assert smg.dgs_tile(nx, ny, nz, 0, 1)[0] == 8
    b = smg.forcing(nx, ny, nz, h=1 / ny, kind=smg.FORCE_UNIFORM, seed=parts)
    assert np.array_equal(many.vcycle(b), one.vcycle(b))
    x1, h1, _, s1 = one.sqmr(b, 1e-8, 40)
    x2, h2, _, s2 = many.sqmr(b, 1e-8, 40)
    assert s1 == s2 == smg.SMG_CONVERGED and np.array_equal(h1, h2) and np.array_equal(x1, x2)
    one.close()
    many.close()


@pytest.mark.parametrize("dims,levels,parts", [((64, 64, 128), 4, 4), ((48, 40, 48), 4, 2)])
def test_tiled_slabs_overlap_bitwise(dims, levels, parts, monkeypatch):
    """Halo transfers overlapped with the interior tile layers (boundary tile layers first, push +
    exchange on the comm stream, interior layers on the compute stream; host.cpp dist_dgs_sym):
    parts with >= 3 tile layers take the overlapped phases; == the serial phases == one part."""
    nx, ny, nz = dims
    b = smg.forcing(nx, ny, nz, h=1 / ny, kind=smg.FORCE_UNIFORM, seed=3 + parts)
    one = smg.Solver(nx, ny, nz, h=1 / ny, levels=levels, tile_min=1)
    v1 = one.vcycle(b)
    x1, h1, _, s1 = one.sqmr(b, 1e-8, 40)
    one.close()
    for ov in ("1", "0"):  # with the overlap also the frame refresh after Vanka phases, and neither
        monkeypatch.setenv("SMG_DIST_OVERLAP", ov)
        monkeypatch.setenv("SMG_DIST_FRAMES", "2" if ov == "1" else "0")
        many = smg.Solver(nx, ny, nz, h=1 / ny, levels=levels, tile_min=1, devices=[0] * parts)
        assert np.array_equal(many.vcycle(b), v1), ov
        x2, h2, _, s2 = many.sqmr(b, 1e-8, 40)
        assert s1 == s2 == smg.SMG_CONVERGED and np.array_equal(h1, h2) and np.array_equal(x1, x2), ov
        many.close()


def test_tiled_rank_path_overlap_bitwise(monkeypatch):
    """One process per GPU with a tiled fine level (one rank, slab path forced): the captured SQMR
    iteration forks the comm stream for every tile colour (halo communicator split off the rank
    communicator, NCCL groups on the comm stream inside the graph) -- bit-identical to one part."""
    monkeypatch.setenv("SMG_FORCE_SLABS", "1")
    one = smg.Solver(64, levels=4, tile_min=1)
    r0 = smg.Solver.for_rank(0, 1, smg.nccl_unique_id(), 64, levels=4, tile_min=1, device=0)
    b = smg.forcing(64, kind=smg.FORCE_UNIFORM, seed=11)
    assert np.array_equal(r0.vcycle(b), one.vcycle(b))
    x1, h1, _, s1 = one.sqmr(b, 1e-8, 60)
    x2, h2, _, s2 = r0.sqmr(b, 1e-8, 60)
    assert s1 == s2 == smg.SMG_CONVERGED and np.array_equal(h1, h2) and np.array_equal(x1, x2)
    r0.close()
    one.close()


def test_tile_packed_b_bitwise(monkeypatch):
    """Tiled levels stage b / c_b from the tile-major packed copy k_dgs_cb<true> writes once per level
    visit (one contiguous bulk copy per tile, already parity-split) instead of TMA boxes of the level
    vector: same values in the same shared-memory slots, so V-cycle and solve are bit-identical to
    SMG_TILE_BPACK=0 (and both to the oracle: the tests above run the packed path by default)."""
    dims = (48, 40, 32)
    b = smg.forcing(*dims, h=1 / 40, kind=smg.FORCE_UNIFORM, seed=5)
    out = []
    for knob in ("1", "0"):
        monkeypatch.setenv("SMG_TILE_BPACK", knob)
        s = smg.Solver(*dims, h=1 / 40, levels=3, tile_min=1)
        v = s.vcycle(b)
        x, hh, _, st = s.sqmr(b, 1e-8, 40)
        out.append((v, x, hh, st))
        s.close()
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])
    assert np.array_equal(out[0][2], out[1][2]) and out[0][3] == out[1][3] == smg.SMG_CONVERGED


def test_tiled_cfg1_iterations_match_spec_order():
    """cfg 1 (128^3, 5 levels) with its fine level tiled: iteration count within +-1 of the
    SPEC-literal sequential order (lexicographic DGS, colour-major sequential Vanka) -- recorded 8."""
    s = smg.Solver(128, levels=5, tile_min=1 << 21)
    b = smg.forcing(128, kind=smg.FORCE_UNIFORM, seed=1)
    _, h, _, st = s.sqmr(b, 1e-6, 100)
    assert st == smg.SMG_CONVERGED and abs(len(h) - 8) <= 1
    s.close()
