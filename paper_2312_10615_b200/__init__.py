"""B200-native MG-preconditioned SQMR Stokes solver (arXiv 2312.10615 hot path).

Thin ctypes mirror of the C-ABI in ``include/smg.h`` (the host C++ API in
``include/stokesmg/solver.hpp`` binds the same symbols).  Everything numeric
runs in ``libsmg.so`` (sm_100a kernels); there is no Python or CPU fallback —
importing this package on a machine without the built library, or calling a
solver entry point without a CUDA device, raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SMG_LIB") or os.path.join(_HERE, "libsmg.so")  # SMG_LIB: tools-only builds

SMG_CONVERGED, SMG_MAX_ITERATIONS, SMG_BREAKDOWN = 0, 1, 2
FLAG_SKIP_REVERSE_DGS = 1
FLAG_NO_PRECOND = 2  # method `sqmr`: identity preconditioner
FORCE_UNIFORM, FORCE_FOURIER, FORCE_CHANNEL = 0, 1, 2

# smoother op codes of smg_smoother (include/smg.h)
OP_DGS_PHASE, OP_DGS_SYM, OP_VANKA_COLOUR, OP_VANKA_SYM, OP_SMOOTH, OP_VANKA_ADD = 0, 1, 2, 3, 4, 5
VANKA_MULTIPLICATIVE, VANKA_ADDITIVE, VANKA_DIRECT = 0, 1, 2
OP_VANKA_DIRECT = 7  # one direct-on-V1 solve
DGS_PHASES = 20


class SmgError(RuntimeError):
    pass


class GridDesc(C.Structure):
    _fields_ = [("dim", C.c_int), ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("h", C.c_double)]


class Params(C.Structure):
    _fields_ = [("eta", C.c_double), ("gamma", C.c_double), ("levels", C.c_int), ("nu", C.c_int),
                ("band_width", C.c_int), ("flags", C.c_int), ("cycle", C.c_int), ("vanka", C.c_int),
                ("omega", C.c_double), ("dgs_tile_min", C.c_int64)]


class History(C.Structure):
    _fields_ = [("capacity", C.c_int), ("count", C.c_int), ("rel_residual", C.POINTER(C.c_double)),
                ("seconds", C.POINTER(C.c_double))]


class Timing(C.Structure):
    _fields_ = [("solve_ms", C.c_double), ("h2d_ms", C.c_double), ("d2h_ms", C.c_double),
                ("iterations", C.c_int), ("kernel_launches", C.c_int64)]


EXPORTED = [
    "smg_create", "smg_destroy", "smg_last_error", "smg_version", "smg_num_levels", "smg_level_ndof",
    "smg_apply", "smg_residual", "smg_smoother", "smg_restrict", "smg_prolong", "smg_coarse_solve",
    "smg_vcycle", "smg_sqmr_solve", "smg_set_rhs", "smg_solve_resident", "smg_get_solution",
    "smg_last_timing", "smg_time_kernel", "smg_host_alloc", "smg_host_free", "smg_forcing",
    "smg_profiler_range", "smg_slab_plan", "smg_mg_solve", "smg_census", "smg_assemble_rhs",
    "smg_nccl_unique_id", "smg_create_rank", "smg_dgs_tile",
    "smg_create_labeled", "smg_coarsen_labels", "smg_census_labeled", "smg_forcing_labeled",
    "smg_check_guards", "smg_assemble_rhs_labeled",
]
LAB_DIRICHLET, LAB_INTERIOR, LAB_EXTERIOR = 0, 1, 2  # CellLabel

_lib = None
_D = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_U8 = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


def lib():
    """Load libsmg.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise SmgError(f"{LIB_PATH} is missing: run `make` (or __graft_entry__.build())")
    L = C.CDLL(LIB_PATH)
    P = C.c_void_p
    L.smg_create.argtypes = [C.POINTER(GridDesc), C.POINTER(Params), C.c_int, C.POINTER(C.c_int),
                             C.POINTER(P)]
    L.smg_destroy.argtypes = [P]
    L.smg_nccl_unique_id.argtypes = [C.c_char_p]
    L.smg_create_rank.argtypes = [C.POINTER(GridDesc), C.POINTER(Params), C.c_int, C.c_int, C.c_int, C.c_char_p,
                                  C.POINTER(P)]
    L.smg_last_error.restype = C.c_char_p
    L.smg_last_error.argtypes = [P]
    L.smg_version.restype = C.c_char_p
    L.smg_num_levels.argtypes = [P]
    L.smg_level_ndof.restype = C.c_int64
    L.smg_level_ndof.argtypes = [P, C.c_int, np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")]
    L.smg_apply.argtypes = [P, C.c_int, C.c_int, _D, _D]
    L.smg_residual.argtypes = [P, C.c_int, _D, _D, _D]
    L.smg_smoother.argtypes = [P, C.c_int, C.c_int, C.c_int, _D, _D]
    L.smg_restrict.argtypes = [P, C.c_int, _D, _D]
    L.smg_prolong.argtypes = [P, C.c_int, _D, _D]
    L.smg_coarse_solve.argtypes = [P, _D, _D]
    L.smg_vcycle.argtypes = [P, _D, _D]
    L.smg_sqmr_solve.argtypes = [P, C.c_void_p, C.c_void_p, C.c_double, C.c_int, C.POINTER(History),
                                 C.POINTER(C.c_int)]
    L.smg_set_rhs.argtypes = [P, C.c_void_p]
    L.smg_mg_solve.argtypes = [P, C.c_void_p, C.c_void_p, C.c_double, C.c_int, C.POINTER(History), C.POINTER(C.c_int)]
    L.smg_solve_resident.argtypes = [P, C.c_double, C.c_int, C.POINTER(History), C.POINTER(C.c_int)]
    L.smg_get_solution.argtypes = [P, C.c_void_p]
    L.smg_last_timing.argtypes = [P, C.POINTER(Timing)]
    L.smg_time_kernel.argtypes = [P, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
    L.smg_profiler_range.argtypes = [C.c_int]
    L.smg_assemble_rhs.argtypes = [C.POINTER(GridDesc), C.c_double, C.c_int, C.c_double, C.c_void_p]
    L.smg_census.restype = C.c_int64
    L.smg_census.argtypes = [C.POINTER(GridDesc), C.c_int, C.c_void_p]
    L.smg_slab_plan.argtypes = [C.POINTER(GridDesc), C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int),
                                C.POINTER(C.c_int)]
    L.smg_dgs_tile.argtypes = [C.POINTER(GridDesc), C.c_int, C.c_int64, C.POINTER(C.c_int)]
    L.smg_host_alloc.restype = C.c_void_p
    L.smg_host_alloc.argtypes = [C.c_int64]
    L.smg_host_free.argtypes = [C.c_void_p]
    L.smg_forcing.argtypes = [C.POINTER(GridDesc), C.c_int, C.c_uint64, C.c_void_p, C.c_int]
    L.smg_create_labeled.argtypes = [C.POINTER(GridDesc), _U8, C.POINTER(Params), C.c_int, C.POINTER(P)]
    L.smg_coarsen_labels.argtypes = [C.POINTER(GridDesc), _U8, _U8]
    L.smg_census_labeled.restype = C.c_int64
    L.smg_census_labeled.argtypes = [C.POINTER(GridDesc), _U8, C.c_int,
                                     np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")]
    L.smg_forcing_labeled.argtypes = [C.POINTER(GridDesc), _U8, C.c_int, C.c_uint64, _D]
    L.smg_assemble_rhs_labeled.argtypes = [C.POINTER(GridDesc), _U8, C.c_double, _D, _D, _D, _D]
    L.smg_check_guards.restype = C.c_int64
    L.smg_check_guards.argtypes = [P]
    _lib = L
    return L


def ndof_box(nx, ny, nz):
    return (nx - 1) * ny * nz + nx * (ny - 1) * nz + nx * ny * (nz - 1) + nx * ny * nz


def forcing(nx, ny=None, nz=None, h=None, kind=FORCE_UNIFORM, seed=0, threads=None, out=None):
    """Synthetic BASELINE forcing (compact order), generated by the host library."""
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    h = 1.0 / nx if h is None else h
    n = ndof_box(nx, ny, nz)
    b = np.empty(n) if out is None else out
    assert b.dtype == np.float64 and b.size == n and b.flags.c_contiguous
    g = GridDesc(3, nx, ny, nz, h)
    rc = lib().smg_forcing(C.byref(g), kind, seed, b.ctypes.data, threads or os.cpu_count() or 1)
    if rc != 0:
        raise SmgError(f"smg_forcing failed ({rc})")
    return b


def _labels3(labels):
    lab = np.ascontiguousarray(labels, dtype=np.uint8)
    if lab.ndim != 3:
        raise ValueError("labels must be shaped (nz, ny, nx)")
    return lab


def census_labels(labels, band_width=1):
    """classify_dofs + partition_band census of a labelled grid (host only):
    labels shaped (nz, ny, nx), 0 Dirichlet / 1 Interior / 2 Exterior."""
    lab = _labels3(labels)
    nz, ny, nx = lab.shape
    out = np.zeros(6, np.int64)
    n = lib().smg_census_labeled(C.byref(GridDesc(3, nx, ny, nz, 1.0)), lab.ravel(), band_width, out)
    if n < 0:
        raise SmgError(f"smg_census_labeled failed ({n})")
    return {"N": int(out[0]), "V1": int(out[1]), "nu": int(out[2]), "nv": int(out[3]), "nw": int(out[4]),
            "np": int(out[5])}


def coarsen_labels(labels):
    """coarsen_grid of a labelled grid with even extents (host only)."""
    lab = _labels3(labels)
    nz, ny, nx = lab.shape
    out = np.zeros((nz // 2, ny // 2, nx // 2), np.uint8)
    rc = lib().smg_coarsen_labels(C.byref(GridDesc(3, nx, ny, nz, 1.0)), lab.ravel(), out.reshape(-1))
    if rc != 0:
        raise SmgError(f"smg_coarsen_labels failed ({rc}): extents must be even and >= 2")
    return out


def forcing_labels(labels, h, kind=FORCE_UNIFORM, seed=0):
    """Synthetic forcing on the active faces of a labelled grid (compact order of its DofMap)."""
    lab = _labels3(labels)
    nz, ny, nx = lab.shape
    b = np.zeros(census_labels(lab)["N"])
    rc = lib().smg_forcing_labeled(C.byref(GridDesc(3, nx, ny, nz, h)), lab.ravel(), kind, seed, b)
    if rc != 0:
        raise SmgError(f"smg_forcing_labeled failed ({rc})")
    return b


def dirichlet_shapes(labels):
    """Shapes (z, y, x) of the Dirichlet face-value arrays g_u, g_v, g_w of smg_assemble_rhs_labeled:
    n + 1 faces along the component's axis, n + 2 along the others (ring faces included)."""
    nz, ny, nx = np.asarray(labels).shape
    return (nz + 2, ny + 2, nx + 1), (nz + 2, ny + 1, nx + 2), (nz + 1, ny + 2, nx + 2)


def assemble_rhs_labels(labels, h, gu, gv, gw, eta=1.0, b=None):
    """assemble_rhs with general Dirichlet data on a labelled grid (host only):
    returns b (default 0) plus the stencil legs into Dirichlet-valued faces."""
    lab = _labels3(labels)
    nz, ny, nx = lab.shape
    gs = [np.ascontiguousarray(g, np.float64) for g in (gu, gv, gw)]
    for g, shp in zip(gs, dirichlet_shapes(lab)):
        if g.shape != shp:
            raise ValueError(f"Dirichlet data shaped {g.shape}, expected {shp}")
    out = np.zeros(census_labels(lab)["N"]) if b is None else np.array(b, np.float64, copy=True)
    rc = lib().smg_assemble_rhs_labeled(C.byref(GridDesc(3, nx, ny, nz, h)), lab.ravel(), eta,
                                        gs[0].ravel(), gs[1].ravel(), gs[2].ravel(), out)
    if rc != 0:
        raise SmgError(f"smg_assemble_rhs_labeled failed ({rc})")
    return out


def slab_plan(nx, ny, nz, levels, nparts, rank, h=None):
    """Host-only z-slab plan of the library: (ndist, [(z0, nzl) per level])."""
    g = GridDesc(3, nx, ny, nz, 1.0 / nx if h is None else h)
    z0 = (C.c_int * levels)()
    nzl = (C.c_int * levels)()
    nd = lib().smg_slab_plan(C.byref(g), levels, nparts, rank, z0, nzl)
    return nd, [(z0[l], nzl[l]) for l in range(levels)]


def dgs_tile(nx, ny, nz, level=0, tile_min=0):
    """DGS tiling of a level (host only): (tile colours, tile_x, tile_y, tile_z); (1, 0, 0, 0) untiled."""
    g = GridDesc(3, nx, ny, nz, 1.0 / nx)
    out = (C.c_int * 4)()
    rc = lib().smg_dgs_tile(C.byref(g), level, int(tile_min), out)
    if rc != 0:
        raise SmgError(f"smg_dgs_tile failed ({rc})")
    return tuple(out)


def cavity_rhs(nx, ny=None, nz=None, h=None, eta=1.0, lid=1.0):
    """Right-hand side of the lid-driven cavity (zero body force, u = lid on the top y face)."""
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    h = 1.0 / nx if h is None else h
    b = np.zeros(ndof_box(nx, ny, nz))
    rc = lib().smg_assemble_rhs(C.byref(GridDesc(3, nx, ny, nz, h)), eta, 0, lid, b.ctypes.data)
    if rc != 0:
        raise SmgError(f"smg_assemble_rhs failed ({rc})")
    return b


class PinnedArray:
    """float64 array in page-locked host memory (smg_host_alloc)."""

    def __init__(self, n):
        self.n = int(n)
        self.ptr = lib().smg_host_alloc(self.n * 8)
        if not self.ptr:
            raise SmgError("smg_host_alloc failed")
        self.array = np.ctypeslib.as_array(C.cast(self.ptr, C.POINTER(C.c_double)), shape=(self.n,))

    def __del__(self):
        if getattr(self, "ptr", None):
            lib().smg_host_free(self.ptr)
            self.ptr = None


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (smg_nccl_unique_id) for Solver.for_rank; call on rank 0 only."""
    buf = C.create_string_buffer(128)
    rc = lib().smg_nccl_unique_id(buf)
    if rc != 0:
        raise SmgError(f"smg_nccl_unique_id failed ({rc}); see stderr")
    return buf.raw


class Solver:
    """One device context (hierarchy + buffers) for a walled box of nx*ny*nz cells."""

    def __init__(self, nx, ny=None, nz=None, h=None, eta=1.0, gamma=1e-3, levels=2, nu=1, band_width=1,
                 flags=0, device=0, devices=None, cycle=0, vanka=0, omega=1.0, tile_min=0):
        """devices: list of CUDA device ids, one z-slab part each (repeat an id to emulate several
        parts on one GPU).  Default: a single part on `device`.  tile_min: cell count from which a
        level's DGS sweep runs in tile order (0: 256^3, the default; -1: never)."""
        ny = nx if ny is None else ny
        nz = nx if nz is None else nz
        h = 1.0 / nx if h is None else h
        L = lib()
        self.grid = GridDesc(3, nx, ny, nz, h)
        self.params = Params(eta, gamma, levels, nu, band_width, flags, cycle, vanka, omega, int(tile_min))
        ctx = C.c_void_p()
        devs = list(devices) if devices else [device]
        arr = (C.c_int * len(devs))(*devs)
        rc = L.smg_create(C.byref(self.grid), C.byref(self.params), len(devs), arr, C.byref(ctx))
        if rc != 0:
            raise SmgError(f"smg_create failed ({rc}); see stderr")
        self._ctx = ctx
        self.levels = L.smg_num_levels(ctx)
        self.dims = (nx, ny, nz)

    @classmethod
    def from_labels(cls, labels, h=None, eta=1.0, gamma=1e-3, levels=2, nu=1, band_width=1, flags=0, device=0,
                    cycle=0, vanka=0, omega=1.0):
        """General labelled domain (smg_create_labeled): labels shaped (nz, ny, nx) with
        0 Dirichlet, 1 Interior, 2 Exterior cells inside the implicit Dirichlet ring."""
        lab = _labels3(labels)
        nz, ny, nx = lab.shape
        h = 1.0 / nx if h is None else h
        self = cls.__new__(cls)
        self.grid = GridDesc(3, nx, ny, nz, h)
        self.params = Params(eta, gamma, levels, nu, band_width, flags, cycle, vanka, omega, -1)
        ctx = C.c_void_p()
        rc = lib().smg_create_labeled(C.byref(self.grid), lab.ravel(), C.byref(self.params), device, C.byref(ctx))
        if rc != 0:
            raise SmgError(f"smg_create_labeled failed ({rc}); see stderr")
        self._ctx = ctx
        self.levels = lib().smg_num_levels(ctx)
        self.dims = (nx, ny, nz)
        return self

    @classmethod
    def for_rank(cls, rank, nranks, nccl_id, nx, ny=None, nz=None, h=None, eta=1.0, gamma=1e-3, levels=2, nu=1,
                 band_width=1, flags=0, device=0, cycle=0, vanka=0, omega=1.0, tile_min=0):
        """Rank `rank` of a one-process-per-GPU z-slab solver (smg_create_rank): every rank
        calls this with the same 128-byte NCCL id (nccl_unique_id() on rank 0, broadcast by
        the launcher) and its own device; later calls are collective."""
        ny = nx if ny is None else ny
        nz = nx if nz is None else nz
        h = 1.0 / nx if h is None else h
        self = cls.__new__(cls)
        self.grid = GridDesc(3, nx, ny, nz, h)
        self.params = Params(eta, gamma, levels, nu, band_width, flags, cycle, vanka, omega, int(tile_min))
        if len(nccl_id) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        ctx = C.c_void_p()
        rc = lib().smg_create_rank(C.byref(self.grid), C.byref(self.params), rank, nranks, device,
                                   bytes(nccl_id), C.byref(ctx))
        if rc != 0:
            raise SmgError(f"smg_create_rank failed ({rc}); see stderr")
        self._ctx = ctx
        self.levels = lib().smg_num_levels(ctx)
        self.dims = (nx, ny, nz)
        return self

    def close(self):
        if getattr(self, "_ctx", None):
            lib().smg_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        self.close()

    def _check(self, rc):
        if rc != 0:
            raise SmgError(f"smg error {rc}: {lib().smg_last_error(self._ctx).decode()}")

    def check_guards(self):
        """Guard-band bytes overwritten by any kernel (needs SMG_GUARD=1 at creation; 0 = clean)."""
        n = lib().smg_check_guards(self._ctx)
        if n < 0:
            self._check(int(n))
        return int(n)

    def ndof(self, level=0):
        c = np.zeros(5, np.int64)
        return int(lib().smg_level_ndof(self._ctx, level, c))

    def dgs_tiled(self, level=0):
        """True if the level's DGS sweep runs in tile order (k_dgs_tile) under this solver's tile_min."""
        nx, ny, nz = self.dims
        return dgs_tile(nx, ny, nz, level, self.params.dgs_tile_min)[0] == 8

    def counts(self, level=0):
        c = np.zeros(5, np.int64)
        lib().smg_level_ndof(self._ctx, level, c)
        return {"nu": int(c[0]), "nv": int(c[1]), "nw": int(c[2]), "np": int(c[3]), "V1": int(c[4])}

    def _vec(self, x, level):
        x = np.ascontiguousarray(x, np.float64)
        if x.size != self.ndof(level):
            raise ValueError("length mismatch (SPEC:125)")
        return x

    def apply(self, x, level=0, penalized=False):
        x = self._vec(x, level)
        y = np.empty_like(x)
        self._check(lib().smg_apply(self._ctx, level, int(penalized), x, y))
        return y

    def residual(self, x, b, level=0):
        x, b = self._vec(x, level), self._vec(b, level)
        r = np.empty_like(x)
        self._check(lib().smg_residual(self._ctx, level, x, b, r))
        return r

    def smoother(self, op, x, b, level=0, arg=0):
        xx = np.array(self._vec(x, level), copy=True)
        self._check(lib().smg_smoother(self._ctx, level, op, arg, xx, self._vec(b, level)))
        return xx

    def restrict(self, rf, level=0):
        rc = np.empty(self.ndof(level + 1))
        self._check(lib().smg_restrict(self._ctx, level, self._vec(rf, level), rc))
        return rc

    def prolong(self, xc, level=0):
        xf = np.empty(self.ndof(level))
        self._check(lib().smg_prolong(self._ctx, level, self._vec(xc, level + 1), xf))
        return xf

    def coarse_solve(self, b):
        lc = self.levels - 1
        x = np.empty(self.ndof(lc))
        self._check(lib().smg_coarse_solve(self._ctx, self._vec(b, lc), x))
        return x

    def vcycle(self, b):
        x = np.empty(self.ndof(0))
        self._check(lib().smg_vcycle(self._ctx, self._vec(b, 0), x))
        return x

    def sqmr(self, b, tol=1e-6, maxit=200, out=None):
        """End-to-end MG-SQMR: host b in, host x out.  Returns (x, history, seconds, status)."""
        b = self._vec(b, 0)
        x = np.empty(self.ndof(0)) if out is None else out
        hist = np.zeros(maxit)
        secs = np.zeros(maxit)
        h = History(maxit, 0, hist.ctypes.data_as(C.POINTER(C.c_double)),
                    secs.ctypes.data_as(C.POINTER(C.c_double)))
        st = C.c_int(-1)
        self._check(lib().smg_sqmr_solve(self._ctx, b.ctypes.data, x.ctypes.data, tol, maxit, C.byref(h),
                                         C.byref(st)))
        return x, hist[: h.count].copy(), secs[: h.count].copy(), st.value

    def mg_solve(self, b, tol=1e-6, maxit=100):
        """Pure multigrid on L~. Returns (x, history, seconds, status)."""
        b = self._vec(b, 0)
        x = np.empty(self.ndof(0))
        hist = np.zeros(maxit)
        secs = np.zeros(maxit)
        h = History(maxit, 0, hist.ctypes.data_as(C.POINTER(C.c_double)),
                    secs.ctypes.data_as(C.POINTER(C.c_double)))
        st = C.c_int(-1)
        self._check(lib().smg_mg_solve(self._ctx, b.ctypes.data, x.ctypes.data, tol, maxit, C.byref(h),
                                       C.byref(st)))
        return x, hist[: h.count].copy(), secs[: h.count].copy(), st.value

    def set_rhs(self, b):
        b = self._vec(b, 0)
        self._check(lib().smg_set_rhs(self._ctx, b.ctypes.data))

    def solve_resident(self, tol=1e-6, maxit=200):
        hist = np.zeros(maxit)
        secs = np.zeros(maxit)
        h = History(maxit, 0, hist.ctypes.data_as(C.POINTER(C.c_double)),
                    secs.ctypes.data_as(C.POINTER(C.c_double)))
        st = C.c_int(-1)
        self._check(lib().smg_solve_resident(self._ctx, tol, maxit, C.byref(h), C.byref(st)))
        return hist[: h.count].copy(), st.value

    def solution(self):
        x = np.empty(self.ndof(0))
        self._check(lib().smg_get_solution(self._ctx, x.ctypes.data))
        return x

    def timing(self):
        t = Timing()
        self._check(lib().smg_last_timing(self._ctx, C.byref(t)))
        return {"solve_ms": t.solve_ms, "h2d_ms": t.h2d_ms, "d2h_ms": t.d2h_ms, "iterations": t.iterations,
                "kernel_launches": int(t.kernel_launches)}

    def time_kernel(self, which, reps=10, level=0):
        ms = C.c_double(0)
        self._check(lib().smg_time_kernel(self._ctx, which, level, reps, C.byref(ms)))
        return ms.value
