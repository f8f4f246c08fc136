"""z-slab decomposition — the multi-GPU data path
emulated with several parts on one GPU: every result must be bit-identical to
the single-part solve (per-point arithmetic unchanged, halos exchanged after
every phase, canonical reductions combined from per-plane partials)."""
import numpy as np
import pytest

import paper_2312_10615_b200 as smg

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,levels,parts", [(16, 3, 2), (32, 3, 2), (32, 3, 4), (64, 4, 4)])
def test_vcycle_and_apply_bitwise(n, levels, parts):
    one = smg.Solver(n, levels=levels)
    many = smg.Solver(n, levels=levels, devices=[0] * parts)
    b = np.random.default_rng(n + parts).uniform(-1, 1, one.ndof())
    assert np.array_equal(many.apply(b), one.apply(b))
    assert np.array_equal(many.apply(b, penalized=True), one.apply(b, penalized=True))
    assert np.array_equal(many.vcycle(b), one.vcycle(b))
    one.close()
    many.close()


@pytest.mark.parametrize("n,levels,parts,kind", [(32, 3, 2, 0), (64, 4, 2, 1), (64, 4, 8, 0)])
def test_sqmr_bitwise(n, levels, parts, kind):
    one = smg.Solver(n, levels=levels)
    many = smg.Solver(n, levels=levels, devices=[0] * parts)
    b = smg.forcing(n, kind=kind, seed=7)
    x1, h1, _, s1 = one.sqmr(b, 1e-6, 100)
    x2, h2, _, s2 = many.sqmr(b, 1e-6, 100)
    assert s1 == s2 == smg.SMG_CONVERGED
    assert np.array_equal(h1, h2) and np.array_equal(x1, x2)
    one.close()
    many.close()


@pytest.mark.parametrize("n,levels,parts,bw", [(64, 4, 2, 1), (64, 4, 4, 2), (64, 4, 8, 2), (32, 3, 4, 3)])
def test_vanka_halo_frames_bitwise(n, levels, parts, bw, monkeypatch):
    """After a Vanka phase a slab level refreshes only the frames of its boundary planes (the band
    DOFs along the x and y walls; host.cpp exchange_frame) unless the slab is too thin (whole
    planes): both == one part, for band widths 1-3 (thin-slab fallback at 32^3 / 4 parts, bw 3)."""
    one = smg.Solver(n, levels=levels, band_width=bw)
    b = smg.forcing(n, kind=smg.FORCE_UNIFORM, seed=20 + parts)
    v1 = one.vcycle(b)
    x1, h1, _, s1 = one.sqmr(b, 1e-8, 60)
    one.close()
    for fr in ("2", "0"):  # 2: frames wherever the geometry allows (default: large planes only)
        monkeypatch.setenv("SMG_DIST_FRAMES", fr)
        many = smg.Solver(n, levels=levels, band_width=bw, devices=[0] * parts)
        assert np.array_equal(many.vcycle(b), v1), fr
        x2, h2, _, s2 = many.sqmr(b, 1e-8, 60)
        assert s1 == s2 and np.array_equal(h1, h2) and np.array_equal(x1, x2), fr
        many.close()


def test_default_gather_below_64_cubed_bitwise(monkeypatch):
    """Production slab plan (levels below 64^3 cells gathered: here only the fine level is split and the
    32^3 sub-cycle runs replicated on every part after the all-gather) == one part."""
    monkeypatch.delenv("SMG_SLAB_MIN_CELLS", raising=False)
    assert smg.slab_plan(64, 64, 64, 4, 4, 0)[0] == 1
    one = smg.Solver(64, levels=4)
    many = smg.Solver(64, levels=4, devices=[0] * 4)
    b = smg.forcing(64, kind=smg.FORCE_UNIFORM, seed=8)
    assert np.array_equal(many.vcycle(b), one.vcycle(b))
    x1, h1, _, s1 = one.sqmr(b, 1e-8, 60)
    x2, h2, _, s2 = many.sqmr(b, 1e-8, 60)
    assert s1 == s2 == smg.SMG_CONVERGED and np.array_equal(h1, h2) and np.array_equal(x1, x2)
    one.close()
    many.close()


@pytest.mark.parametrize("maxit", [0, 1, 2, 5])
def test_slab_two_reduction_order_statuses(maxit):
    """Slab contexts run SQMR with two reductions per iteration (the q step of iteration j + 1 before the
    convergence test of iteration j; host.cpp sqmr_iteration), one part with three finals: status,
    iteration count, history and the returned iterate agree bit for bit when maxit cuts the solve short,
    and on a zero right-hand side."""
    one = smg.Solver(32, levels=3)
    many = smg.Solver(32, levels=3, devices=[0, 0])
    b = smg.forcing(32, kind=smg.FORCE_UNIFORM, seed=44)
    x1, h1, _, s1 = one.sqmr(b, 1e-10, maxit)
    x2, h2, _, s2 = many.sqmr(b, 1e-10, maxit)
    assert s1 == s2 and len(h1) == len(h2) == maxit and np.array_equal(h1, h2) and np.array_equal(x1, x2)
    z = np.zeros_like(b)
    xz1, hz1, _, sz1 = one.sqmr(z, 1e-10, 5)
    xz2, hz2, _, sz2 = many.sqmr(z, 1e-10, 5)
    assert sz1 == sz2 == smg.SMG_CONVERGED and len(hz1) == len(hz2) == 0 and not xz1.any() and not xz2.any()
    one.close()
    many.close()


@pytest.mark.parametrize("n,levels,parts", [(48, 5, 2), (48, 4, 4)])
def test_odd_slab_levels_bitwise(n, levels, parts):
    """Levels whose slab would be odd stay replicated: 48^3 with 5 levels on 2 parts
    distributes 3 levels and still matches one part bit for bit."""
    one = smg.Solver(n, levels=levels)
    many = smg.Solver(n, levels=levels, devices=[0] * parts)
    b = smg.forcing(n, kind=smg.FORCE_UNIFORM, seed=17)
    assert np.array_equal(many.vcycle(b), one.vcycle(b))
    x1, h1, _, s1 = one.sqmr(b, 1e-6, 60)
    x2, h2, _, s2 = many.sqmr(b, 1e-6, 60)
    assert s1 == s2 and np.array_equal(h1, h2) and np.array_equal(x1, x2)
    one.close()
    many.close()


@pytest.mark.parametrize("n,levels,parts", [(64, 5, 2), (64, 4, 4)])
def test_wcycle_slabs_bitwise(n, levels, parts):
    """W-cycle on slab parts (second recursive call on distributed and replicated children) ==
    the single-part W-cycle, bit for bit (dist_vcycle used to ignore cycle = 1)."""
    one = smg.Solver(n, levels=levels, cycle=1)
    many = smg.Solver(n, levels=levels, cycle=1, devices=[0] * parts)
    b = smg.forcing(n, kind=smg.FORCE_UNIFORM, seed=19)
    assert np.array_equal(many.vcycle(b), one.vcycle(b))
    x1, h1, _, s1 = one.sqmr(b, 1e-6, 60)
    x2, h2, _, s2 = many.sqmr(b, 1e-6, 60)
    assert s1 == s2 and np.array_equal(h1, h2) and np.array_equal(x1, x2)
    one.close()
    many.close()


def test_channel_slabs_bitwise():
    one = smg.Solver(64, 16, 16, h=1 / 16, levels=3)
    many = smg.Solver(64, 16, 16, h=1 / 16, levels=3, devices=[0, 0])
    b = smg.forcing(64, 16, 16, h=1 / 16, kind=smg.FORCE_CHANNEL, seed=4)
    x1, h1, _, _ = one.sqmr(b, 1e-8, 100)
    x2, h2, _, _ = many.sqmr(b, 1e-8, 100)
    assert np.array_equal(h1, h2) and np.array_equal(x1, x2)


def test_resident_path_slabs():
    many = smg.Solver(32, levels=3, devices=[0, 0])
    b = smg.forcing(32, seed=0)
    x1, h1, _, _ = many.sqmr(b, 1e-6, 100)
    many.set_rhs(b)
    h2, st = many.solve_resident(1e-6, 100)
    assert st == 0 and np.array_equal(h1, h2) and np.array_equal(many.solution(), x1)


def test_nccl_rank_path_bitwise(monkeypatch):
    """smg_create_rank (one process per GPU, NCCL transport) with one rank and the slab path
    forced: NCCL all-reduce of the plane partials, in-place all-gather of the first replicated
    level, per-rank broadcast of the solution and (empty) halo groups; bit-identical to 1 part."""
    monkeypatch.setenv("SMG_FORCE_SLABS", "1")
    one = smg.Solver(32, levels=3)
    r0 = smg.Solver.for_rank(0, 1, smg.nccl_unique_id(), 32, levels=3, device=0)
    b = smg.forcing(32, kind=smg.FORCE_UNIFORM, seed=9)
    assert np.array_equal(r0.apply(b), one.apply(b))
    assert np.array_equal(r0.vcycle(b), one.vcycle(b))
    x1, h1, _, s1 = one.sqmr(b, 1e-6, 100)
    x2, h2, _, s2 = r0.sqmr(b, 1e-6, 100)
    assert s1 == s2 == smg.SMG_CONVERGED
    assert np.array_equal(h1, h2) and np.array_equal(x1, x2)
    r0.close()
    one.close()


@pytest.mark.parametrize("zseg", ["2", "3"])
def test_restrict_zmarch_slabs_bitwise(zseg, monkeypatch):
    """z-marching restriction on slab parts (local plane ranges, ghost planes) == one part."""
    monkeypatch.setenv("SMG_RESTRICT_ZSEG", zseg)
    one = smg.Solver(32, levels=3)
    many = smg.Solver(32, levels=3, devices=[0, 0])
    b = np.random.default_rng(7).uniform(-1, 1, one.ndof())
    assert np.array_equal(many.vcycle(b), one.vcycle(b))
    one.close()
    many.close()


def _ndev():
    import ctypes
    try:
        rt = ctypes.CDLL("libcudart.so")
    except OSError:
        try:
            import torch
            return torch.cuda.device_count()
        except Exception:
            return 1
    n = ctypes.c_int(0)
    return n.value if rt.cudaGetDeviceCount(ctypes.byref(n)) == 0 else 1


@pytest.mark.skipif(_ndev() < 2, reason="needs >= 2 visible GPUs (peer copies over NVLink between real devices)")
@pytest.mark.parametrize("n,levels", [(64, 4), (128, 5)])
def test_two_device_parts_bitwise(n, levels):
    """In-process z-slab parts on DIFFERENT devices (one stream each, event barriers, peer halo
    copies): bit-identical to one device.  Runs whenever the box exposes at least two GPUs."""
    ndev = min(_ndev(), 8)
    while n % ndev or (n // ndev) % 2:
        ndev -= 1
    one = smg.Solver(n, levels=levels)
    many = smg.Solver(n, levels=levels, devices=list(range(ndev)))
    b = smg.forcing(n, kind=smg.FORCE_UNIFORM, seed=23)
    assert np.array_equal(many.vcycle(b), one.vcycle(b))
    x1, h1, _, s1 = one.sqmr(b, 1e-6, 60)
    x2, h2, _, s2 = many.sqmr(b, 1e-6, 60)
    assert s1 == s2 == smg.SMG_CONVERGED and np.array_equal(h1, h2) and np.array_equal(x1, x2)
    one.close()
    many.close()
