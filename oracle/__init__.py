"""ctypes wrapper of the CPU oracle (``oracle/liboracle.so``) — TEST INFRASTRUCTURE ONLY.

The oracle restates the reference's MG-SQMR Stokes path (SPEC.md / PAPER.md of
arXiv 2312.10615; see the header of ``stokes_oracle.cpp``).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference arm may
import this module, and only as the checker or the CPU baseline — never as the
thing measured or shipped.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

ST_CONVERGED, ST_MAXIT, ST_BREAKDOWN = 0, 1, 2
FORCE_UNIFORM, FORCE_FOURIER, FORCE_CHANNEL = 0, 1, 2
ORDER_GPU, ORDER_SPEC = 0, 1

_D = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_I64 = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_U8 = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


def build() -> None:
    subprocess.check_call(["make", "-s", "-C", _HERE])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.orc_last_error.restype = C.c_char_p
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_create.restype = C.c_void_p
        L.orc_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                 C.c_int, C.c_int, C.c_int, C.c_int64]
        L.orc_create_labeled.restype = C.c_void_p
        L.orc_create_labeled.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, _U8, C.c_double, C.c_double,
                                         C.c_int, C.c_int, C.c_int]
        L.orc_set_order.argtypes = [C.c_void_p, C.c_int]
        L.orc_dgs_tile.argtypes = [C.c_void_p, C.c_int, np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")]
        L.orc_destroy.argtypes = [C.c_void_p]
        L.orc_nlevels.argtypes = [C.c_void_p]
        L.orc_ndof.restype = C.c_int64
        L.orc_ndof.argtypes = [C.c_void_p, C.c_int]
        L.orc_counts.argtypes = [C.c_void_p, C.c_int, _I64]
        L.orc_v1_mask.argtypes = [C.c_void_p, C.c_int, _U8]
        L.orc_set_skip_reverse.argtypes = [C.c_void_p, C.c_int]
        L.orc_apply.argtypes = [C.c_void_p, C.c_int, C.c_int, _D, _D]
        L.orc_residual.argtypes = [C.c_void_p, C.c_int, _D, _D, _D]
        L.orc_smoother.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, _D, _D]
        L.orc_restrict.argtypes = [C.c_void_p, C.c_int, _D, _D]
        L.orc_prolong.argtypes = [C.c_void_p, C.c_int, _D, _D]
        L.orc_coarse_solve.argtypes = [C.c_void_p, _D, _D]
        L.orc_vcycle.argtypes = [C.c_void_p, _D, _D]
        L.orc_assemble_dense.argtypes = [C.c_void_p, C.c_int, C.c_int, _D]
        L.orc_coarse_inverse.argtypes = [C.c_void_p, _D]
        L.orc_sqmr.argtypes = [C.c_void_p, _D, _D, C.c_double, C.c_int, C.c_int, _D, _D,
                               C.POINTER(C.c_int)]
        L.orc_forcing.argtypes = [C.c_void_p, C.c_int, C.c_uint64, _D]
        L.orc_set_cycle.argtypes = [C.c_void_p, C.c_int]
        L.orc_set_vanka.argtypes = [C.c_void_p, C.c_int, C.c_double]
        L.orc_mg_solve.argtypes = [C.c_void_p, _D, _D, C.c_double, C.c_int, _D, _D, C.POINTER(C.c_int)]
        L.orc_census_box.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _I64]
        L.orc_coarsen_labels.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _U8, _U8]
        L.orc_census_labels.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _U8, C.c_int, _I64]
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


FORCE_CAVITY = 3  # lid-driven cavity: Dirichlet data only (u = 1 on the top y face)


def forcing_box(nx, ny, nz, h, kind=FORCE_UNIFORM, seed=0, eta=1.0):
    L = lib()
    L.orc_set_forcing_eta.argtypes = [C.c_double]
    L.orc_set_forcing_eta(eta)
    L.orc_forcing_box.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_uint64, _D]
    n = (nx - 1) * ny * nz + nx * (ny - 1) * nz + nx * ny * (nz - 1) + nx * ny * nz
    b = np.empty(n)
    L.orc_forcing_box(nx, ny, nz, h, kind, seed, b)
    return b


def census_box(dim: int, nx: int, ny: int, nz: int = 1, width: int = 1):
    out = np.zeros(2, np.int64)
    lib().orc_census_box(dim, nx, ny, nz, width, out)
    return int(out[0]), int(out[1])


def census_labels(labels: np.ndarray, width: int = 1):
    """labels: uint8 array shaped (nz, ny, nx) or (ny, nx); 0=D, 1=I, 2=E."""
    lab = np.ascontiguousarray(labels, dtype=np.uint8)
    dim = lab.ndim
    nz, ny, nx = (lab.shape if dim == 3 else (1,) + lab.shape)
    out = np.zeros(6, np.int64)
    lib().orc_census_labels(dim, nx, ny, nz, lab.ravel(), width, out)
    return {"N": int(out[0]), "V1": int(out[1]), "nu": int(out[2]), "nv": int(out[3]),
            "nw": int(out[4]), "np": int(out[5])}


def coarsen_labels(labels: np.ndarray) -> np.ndarray:
    lab = np.ascontiguousarray(labels, dtype=np.uint8)
    dim = lab.ndim
    shp = lab.shape if dim == 3 else (1,) + lab.shape
    nz, ny, nx = shp
    cshape = ((nz + 1) // 2 if dim == 3 else 1, (ny + 1) // 2, (nx + 1) // 2)
    out = np.zeros(int(np.prod(cshape)), np.uint8)
    lib().orc_coarsen_labels(dim, nx, ny, nz, lab.ravel(), out)
    return out.reshape(cshape if dim == 3 else cshape[1:])


class Oracle:
    """Walled box of nx*ny*nz interior cells (implicit Dirichlet ring), spacing h."""

    def __init__(self, nx, ny=None, nz=None, h=None, eta=1.0, gamma=1e-3, levels=2, nu=1,
                 band_width=1, cycle=0, vanka=0, omega=1.0, tile_min=0, order=ORDER_GPU, labels=None):
        """labels (optional): uint8 array shaped (nz, ny, nx), 0 = Dirichlet, 1 = Interior,
        2 = Exterior -- a general labelled domain inside the implicit Dirichlet ring;
        nx, ny, nz are then taken from its shape.
        tile_min: cell count from which a level's DGS sweep is tile-ordered (0: 256^3, the
        GPU default; -1: never).  order: ORDER_GPU (the coloured order the GPU reproduces bit
        for bit) or ORDER_SPEC (SPEC-literal sequential lexicographic DGS / colour-major Vanka)."""
        L = lib()
        if labels is not None:
            lab = np.ascontiguousarray(labels, dtype=np.uint8)
            nz, ny, nx = lab.shape
            h = 1.0 / nx if h is None else h
            self._h = L.orc_create_labeled(nx, ny, nz, h, lab.ravel(), eta, gamma, levels, nu, band_width)
        else:
            ny = nx if ny is None else ny
            nz = nx if nz is None else nz
            h = 1.0 / nx if h is None else h
            self._h = L.orc_create(nx, ny, nz, h, eta, gamma, levels, nu, band_width, int(tile_min))
        if not self._h:
            raise RuntimeError("oracle: " + L.orc_last_error().decode())
        self.dims = (nx, ny, nz)
        self.levels = L.orc_nlevels(self._h)
        self.nu = nu
        L.orc_set_cycle(self._h, int(cycle))
        L.orc_set_vanka(self._h, int(vanka), float(omega))  # 0 multiplicative, 1 additive
        L.orc_set_order(self._h, int(order))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_destroy(self._h)
            self._h = None

    def ndof(self, level=0) -> int:
        return int(lib().orc_ndof(self._h, level))

    def counts(self, level=0):
        c = np.zeros(5, np.int64)
        lib().orc_counts(self._h, level, c)
        return {"nu": int(c[0]), "nv": int(c[1]), "nw": int(c[2]), "np": int(c[3]), "V1": int(c[4])}

    def dgs_tile(self, level=0):
        """(tile colours, tile_x, tile_y, tile_z) of a level's DGS ordering (1, 0, 0, 0: untiled)."""
        out = np.zeros(4, np.int32)
        lib().orc_dgs_tile(self._h, level, out)
        return tuple(int(v) for v in out)

    def v1_mask(self, level=0):
        m = np.zeros(self.ndof(level), np.uint8)
        lib().orc_v1_mask(self._h, level, m)
        return m.astype(bool)

    def set_skip_reverse(self, flag: bool):
        lib().orc_set_skip_reverse(self._h, int(bool(flag)))

    def apply(self, x, level=0, penalized=False):
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty_like(x)
        lib().orc_apply(self._h, level, int(penalized), x, y)
        return y

    def residual(self, x, b, level=0):
        r = np.empty(self.ndof(level))
        lib().orc_residual(self._h, level, np.ascontiguousarray(x, np.float64),
                           np.ascontiguousarray(b, np.float64), r)
        return r

    def smoother(self, op, x, b, level=0, arg=0):
        xx = np.array(x, np.float64, copy=True)
        rc = lib().orc_smoother(self._h, level, op, arg, xx, np.ascontiguousarray(b, np.float64))
        if rc != 0:
            raise RuntimeError(lib().orc_last_error().decode())
        return xx

    def restrict(self, rf, level=0):
        rc = np.empty(self.ndof(level + 1))
        lib().orc_restrict(self._h, level, np.ascontiguousarray(rf, np.float64), rc)
        return rc

    def prolong(self, xc, level=0):
        xf = np.empty(self.ndof(level))
        lib().orc_prolong(self._h, level, np.ascontiguousarray(xc, np.float64), xf)
        return xf

    def coarse_solve(self, b):
        x = np.empty(self.ndof(self.levels - 1))
        lib().orc_coarse_solve(self._h, np.ascontiguousarray(b, np.float64), x)
        return x

    def coarse_inverse(self):
        n = self.ndof(self.levels - 1)
        k = np.empty(n * n)
        lib().orc_coarse_inverse(self._h, k)
        return k.reshape(n, n)

    def vcycle(self, b):
        x = np.empty(self.ndof(0))
        lib().orc_vcycle(self._h, np.ascontiguousarray(b, np.float64), x)
        return x

    def dense(self, level=0, penalized=False):
        n = self.ndof(level)
        a = np.zeros(n * n)
        lib().orc_assemble_dense(self._h, level, int(penalized), a)
        return a.reshape(n, n)

    def sqmr(self, b, tol=1e-6, maxit=200, precond=True):
        b = np.ascontiguousarray(b, np.float64)
        x = np.empty(self.ndof(0))
        hist = np.zeros(maxit)
        secs = np.zeros(maxit)
        it = C.c_int(0)
        st = lib().orc_sqmr(self._h, b, x, tol, maxit, int(precond), hist, secs, C.byref(it))
        return x, hist[: it.value].copy(), secs[: it.value].copy(), int(st)

    def mg_solve(self, b, tol=1e-6, maxit=100):
        """Pure multigrid on L~: returns (x, history, seconds, status)."""
        b = np.ascontiguousarray(b, np.float64)
        x = np.empty(self.ndof(0))
        hist = np.zeros(maxit)
        secs = np.zeros(maxit)
        it = C.c_int(0)
        st = lib().orc_mg_solve(self._h, b, x, tol, maxit, hist, secs, C.byref(it))
        return x, hist[: it.value].copy(), secs[: it.value].copy(), int(st)

    def dirichlet_rhs(self, gu, gv, gw, b=None):
        """assemble_rhs with general Dirichlet face data: returns b + the stencil legs
        into Dirichlet faces; g_c shaped with n_a + 1 along its own axis, n_a + 2 along the others
        (ring faces included), as (z, y, x) arrays."""
        L = lib()
        L.orc_dirichlet_rhs.argtypes = [C.c_void_p, _D, _D, _D, _D]
        bb = np.zeros(self.ndof(0)) if b is None else np.array(b, np.float64, copy=True)
        L.orc_dirichlet_rhs(self._h, *(np.ascontiguousarray(g, np.float64).ravel() for g in (gu, gv, gw)), bb)
        return bb

    def forcing(self, kind=FORCE_UNIFORM, seed=0):
        b = np.empty(self.ndof(0))
        lib().orc_forcing(self._h, kind, seed, b)
        return b


def set_debug(flags: int) -> None:
    """Experiment knobs (tests/diagnostics only): 1 sequential Vanka, 2 DGS M-columns on V2 only,
    4 reflecting tangential Dirichlet ghosts."""
    L = lib()
    L.orc_set_debug.argtypes = [C.c_int]
    L.orc_set_debug(int(flags))
