"""Deterministic label builders for the paper's 3-D benchmark domains (SPEC module `scenarios`,
SPEC:460-505; PAPER section 6).

Each builder returns a uint8 array shaped (nz, ny, nx) of CellLabels -- 0 Dirichlet, 1 Interior,
2 Exterior -- for `Solver.from_labels` / `smg_create_labeled`.  Obstacles are
rasterised by cell-centre membership; channel walls are the implicit Dirichlet ring;
an outflow is a column of Exterior cells (homogeneous Neumann).  Extents are
chosen by the caller as multiples of 2^(levels-1).  The exact coordinates of the hollow-square,
brancher and porous obstacles are unpublished: the geometries follow the SPEC's
reconstruction and expose their parameters.  Host-side numpy only; nothing here is on the hot path.
"""
from __future__ import annotations

import numpy as np

D, I, E = 0, 1, 2


def _grid(nx, ny, nz):
    zz, yy, xx = np.meshgrid(np.arange(nz) + 0.5, np.arange(ny) + 0.5, np.arange(nx) + 0.5, indexing="ij")
    return np.full((nz, ny, nx), I, np.uint8), xx, yy, zz


def _outflow(lab, cells=1):
    lab[:, :, lab.shape[2] - cells:] = E  # the last x column(s): Exterior => homogeneous Neumann outflow
    return lab


def cavity3d(n):
    """Unit cube of n^3 Interior cells inside the implicit ring (PAPER section 6.2.1)."""
    return np.full((n, n, n), I, np.uint8)


def cylinder3d(nx, ny, nz, cx=0.2 / 2.2, cy=0.2 / 0.41, radius=0.05 / 0.41, outflow=1):
    """Channel with a cylinder along z (PAPER section 6.2.2): centre (cx * nx, cy * ny) and radius
    radius * ny in cells (defaults: the paper's 2.2 x 0.41 channel, cylinder at (0.2, 0.2), r = 0.05),
    Dirichlet obstacle, Exterior outflow column."""
    lab, xx, yy, _ = _grid(nx, ny, nz)
    lab[(xx - cx * nx) ** 2 + (yy - cy * ny) ** 2 < (radius * ny) ** 2] = D
    return _outflow(lab, outflow)


def hollow_square3d(nx, ny, nz, side=0.5, wall=1, gap=0.25, outflow=1):
    """Centred square annulus (extruded along z) with one inlet gap facing the inflow:
    outer side `side` * min(nx, ny) cells, walls `wall` cells thick, a gap of `gap` * side on its
    low-x wall."""
    lab, xx, yy, _ = _grid(nx, ny, nz)
    half = 0.5 * side * min(nx, ny)
    mx, my = 0.5 * nx, 0.5 * ny
    outer = (np.abs(xx - mx) < half) & (np.abs(yy - my) < half)
    inner = (np.abs(xx - mx) < half - wall) & (np.abs(yy - my) < half - wall)
    ring = outer & ~inner
    inlet = (xx < mx - half + wall) & (np.abs(yy - my) < 0.5 * gap * 2 * half)
    lab[ring & ~inlet] = D
    return _outflow(lab, outflow)


def brancher3d(nx, ny, nz, baffles=3, thickness=1, slots=2, outflow=1):
    """Evenly spaced rectangular baffles across the channel, each leaving `slots` evenly spaced
    openings, alternating the slot offset from baffle to baffle."""
    lab, xx, yy, _ = _grid(nx, ny, nz)
    for k in range(baffles):
        x0 = (k + 1) * nx // (baffles + 1)
        wall = (xx > x0) & (xx < x0 + thickness)
        period = ny / slots
        phase = 0.25 * period if k % 2 else 0.75 * period
        open_ = np.abs(((yy - phase) % period) - 0.5 * period) > 0.5 * period - max(1.0, 0.15 * period)
        lab[wall & ~open_] = D
    return _outflow(lab, outflow)


def porous3d(nx, ny, nz, porosity=0.5, seed=0, x0=0.25, x1=0.75, block=2, outflow=1):
    """A slab x0..x1 of randomly placed solid blocks (block^3 cells) at the given porosity, seeded
    (SPEC:496); blocks keep the coarser levels' labelling faithful to the fine one."""
    lab, xx, _, _ = _grid(nx, ny, nz)
    rng = np.random.default_rng(seed)
    bz, by, bx = (nz + block - 1) // block, (ny + block - 1) // block, (nx + block - 1) // block
    solid = rng.random((bz, by, bx)) >= porosity
    solid = np.repeat(np.repeat(np.repeat(solid, block, 0), block, 1), block, 2)[:nz, :ny, :nx]
    lab[solid & (xx > x0 * nx) & (xx < x1 * nx)] = D
    return _outflow(lab, outflow)


def inflow_profile(y, H, ubar, z=None):
    """PAPER section 6.1.2 / 6.2.2 inflow: 2-D parabola 4 ubar y (H - y) / H^2 (mean ubar... the
    paper's `ubar` normalisation: the value at the centreline), 3-D 16 ubar y z (H - y)(H - z) / H^4."""
    y = np.asarray(y, float)
    if np.any(y < 0) or np.any(y > H):
        raise ValueError("coordinate outside [0, H]")
    if z is None:
        return 4.0 * ubar * y * (H - y) / H ** 2
    z = np.asarray(z, float)
    if np.any(z < 0) or np.any(z > H):
        raise ValueError("coordinate outside [0, H]")
    return 16.0 * ubar * y * z * (H - y) * (H - z) / H ** 4


def pad_labels(labels, levels, wall=True):
    """Pad a labelled grid to extents divisible by 2^(levels-1) ("pad with Exterior cells";
    smg_create_labeled wants divisible extents).  wall=True first adds one explicit Dirichlet layer on
    every padded side, so the faces that touched the implicit Dirichlet ring stay Dirichlet-valued
     -- the fine-level DofMap and operator are then exactly those of the unpadded grid;
    without it the padded side becomes a homogeneous-Neumann boundary."""
    lab = np.ascontiguousarray(labels, np.uint8)
    m = 1 << (levels - 1)
    out = lab
    for axis in range(3):
        n = out.shape[axis]
        extra = (-n) % m
        if extra == 0:
            continue
        if wall and extra < 1:
            extra += m
        shape = list(out.shape)
        shape[axis] = extra
        pad = np.full(shape, E, np.uint8)
        if wall:
            idx = [slice(None)] * 3
            idx[axis] = slice(0, 1)
            pad[tuple(idx)] = D
        out = np.concatenate([out, pad], axis=axis)
    return out


def channel_inflow(labels, H, ubar, through=True):
    """Dirichlet data of the 3-D channel inflow (PAPER section 6.2.2): u = 16 ubar y z (H - y)(H - z) / H^4
    on the u faces of the inflow plane x = 0 (y, z at the face centres, channel height and depth H
    over ny and nz cells), 0 on every other Dirichlet face.  through: the same profile is prescribed
    on the plane x = nx (use a grid without an Exterior outflow column).  Under the SPEC's Neumann
    rule an Interior|Exterior face is Inactive and carries no normal flux, so an
    inflow-only data set violates RHS compatibility; prescribing the outflow keeps the
    net boundary flux zero.  Returns (g_u, g_v, g_w) for `assemble_rhs_labels` /
    `smg_assemble_rhs_labeled`."""
    nz, ny, nx = np.asarray(labels).shape
    gu = np.zeros((nz + 2, ny + 2, nx + 1))
    y = (np.arange(ny) + 0.5) * H / ny
    z = (np.arange(nz) + 0.5) * H / nz
    gu[1:-1, 1:-1, 0] = inflow_profile(y[None, :], H, ubar, z=z[:, None])
    if through:
        gu[:, :, -1] = gu[:, :, 0]
    return gu, np.zeros((nz + 2, ny + 1, nx + 2)), np.zeros((nz + 1, ny + 2, nx + 2))


def write_domain_file(path, labels, h):
    """Domain file of SPEC:88: header `3 nx ny nz h`, then one character per cell (D / I / E),
    row-major with x fastest, one x row per line.  `solver run|census` reads it ("domain" key)."""
    lab = np.ascontiguousarray(labels, np.uint8)
    nz, ny, nx = lab.shape
    chars = np.array([b"D", b"I", b"E"])[lab]
    with open(path, "wb") as f:
        f.write(f"3 {nx} {ny} {nz} {h!r}\n".encode())
        for z in range(nz):
            for y in range(ny):
                f.write(b"".join(chars[z, y]) + b"\n")


def read_domain_file(path):
    """Inverse of write_domain_file: (labels shaped (nz, ny, nx), h)."""
    with open(path) as f:
        dim, nx, ny, nz, h = f.readline().split()
        if int(dim) != 3:
            raise ValueError("3-D domain files only")
        body = "".join(f.read().split())
    lut = {"D": D, "I": I, "E": E}
    lab = np.array([lut[c] for c in body], np.uint8).reshape(int(nz), int(ny), int(nx))
    return lab, float(h)
