"""Out-of-bounds detection without compute-sanitizer (closed on this GPU pool, see
profiles/r2d_sanitize_memcheck.log): with SMG_GUARD=1 every device buffer of a context sits between
two 4 KiB guard bands of 0xA5.  A kernel that stores outside its buffer dirties a band
(smg_check_guards > 0); a kernel that READS outside its buffer picks up 0xA5 garbage instead of a
neighbouring allocation's zeros and breaks the bit-identity with the unguarded run.  Covers every
kernel family: cluster / grid cooperative Vanka, per-step and tile-ordered (TMA) DGS, transfers,
coarse GEMV, the fused SQMR graph, z-slab parts and the labelled-domain kernels."""
import numpy as np
import pytest

import paper_2312_10615_b200 as smg
from paper_2312_10615_b200 import scenarios

pytestmark = pytest.mark.gpu

CASES = {
    "box64_4lv": lambda: (smg.Solver(64, levels=4), smg.forcing(64, seed=1)),
    "box48x32x16_w": lambda: (smg.Solver(48, 32, 16, h=1 / 16, levels=3, cycle=1), smg.forcing(48, 32, 16, h=1 / 16, seed=2)),
    "tiled32x16x16": lambda: (smg.Solver(32, 16, 16, h=1 / 16, levels=2, tile_min=1),
                              smg.forcing(32, 16, 16, h=1 / 16, seed=3)),
    "slabs2": lambda: (smg.Solver(64, levels=4, devices=[0, 0]), smg.forcing(64, seed=4)),
    "direct_v1": lambda: (smg.Solver(16, levels=2, vanka=smg.VANKA_DIRECT), smg.forcing(16, seed=5)),
    "additive": lambda: (smg.Solver(32, levels=3, vanka=smg.VANKA_ADDITIVE, omega=0.7), smg.forcing(32, seed=6)),
    "labelled_porous": lambda: (smg.Solver.from_labels(scenarios.porous3d(32, 16, 16, seed=3), h=1 / 16, levels=3),
                                smg.forcing_labels(scenarios.porous3d(32, 16, 16, seed=3), 1 / 16, 0, 7)),
}


@pytest.mark.parametrize("name", list(CASES))
def test_no_out_of_bounds_access(name, monkeypatch):
    monkeypatch.delenv("SMG_GUARD", raising=False)
    s, b = CASES[name]()
    try:
        x0, h0, _, st0 = s.sqmr(b, 1e-8, 40)
        v0 = s.vcycle(b)
        assert s.check_guards() == 0  # guards off: always 0
    finally:
        s.close()
    monkeypatch.setenv("SMG_GUARD", "1")
    s, b = CASES[name]()
    try:
        x1, h1, _, st1 = s.sqmr(b, 1e-8, 40)
        v1 = s.vcycle(b)
        assert s.check_guards() == 0, "a kernel stored outside its buffer"
    finally:
        s.close()
    assert st0 == st1
    assert np.array_equal(h0, h1) and np.array_equal(x0, x1) and np.array_equal(v0, v1), \
        "a kernel read outside its buffer (guard bytes changed the result)"
