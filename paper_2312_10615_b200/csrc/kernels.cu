// kernels.cu — sm_100a CUDA kernels of the MG-SQMR Stokes hot path.
//
// Every per-point formula follows the arithmetic contract of DESIGN.md §4
// (same operand order as oracle/stokes_oracle.cpp; compiled with -fmad=false so
// no contraction), which makes each kernel bit-identical to the CPU oracle.
// Only the BLAS-1 reductions use a different (fixed, deterministic) order.
//
// Reference: SPEC.md modules discretization (apply),
// smoothers (DGS SPEC:258-283, Vanka SPEC:284-301), transfer,
// multigrid coarse solve, krylov.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include <cooperative_groups.h>
#include <cuda.h>

#include "smg_internal.h"

namespace smg {

static std::atomic<int64_t> g_launches{0};
static std::atomic<int> g_launch_err{0};
int64_t launch_count() { return g_launches.load(); }
// First launch-configuration error since the last call (0 if none); the host
// turns it into SMG_ECUDA so a rejected launch can never pass silently.
int take_launch_error() { return g_launch_err.exchange(0); }
static inline void note(cudaError_t e) {
    if (e != cudaSuccess) {
        int z = 0;
        g_launch_err.compare_exchange_strong(z, static_cast<int>(e));
    }
}
static inline void count() { g_launches.fetch_add(1, std::memory_order_relaxed); }

namespace {

constexpr int BX = 32, BY = 8;

// Programmatic dependent launch: kernels launched by launch_k may start while the
// previous kernel drains; they wait here (before touching memory) until it has
// completed and its writes are visible.  A no-op for ordinary launches.
// The trigger right after lets the next kernel's blocks be scheduled as soon as every
// block of this one has started (they then wait for this grid's completion).
__device__ __forceinline__ void pdl_wait() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

inline dim3 cell_grid(const Geom& g) { return dim3((g.nx + BX - 1) / BX, (g.ny + BY - 1) / BY, g.nz); }

struct Cell {
    int x, y, z;
    int64_t i;
};

__device__ __forceinline__ bool thread_cell(const Geom& g, Cell& c) {
    c.x = blockIdx.x * BX + threadIdx.x;
    c.y = blockIdx.y * BY + threadIdx.y;
    c.z = blockIdx.z;
    if (c.x >= g.nx || c.y >= g.ny) return false;
    c.i = g.slot(c.x, c.y, c.z);
    return true;
}

// band membership (V1) of the cell at LOCAL plane z, decided on global coordinates
__device__ __forceinline__ bool band_cell(const LevelK& L, int x, int y, int z) {
    const Geom& g = L.g;
    const int zz = g.gz(z);
    return x < L.bw || y < L.bw || zz < L.bw || x >= g.nx - L.bw || y >= g.ny - L.bw || zz >= g.gnz - L.bw;
}

// Momentum row of L~ at the face stored at slot i of field F (stride of the
// normal axis sn): eta/h^2 (6 u - sum of 6 neighbours, order x-,x+,y-,y+,z-,z+)
// + (p_right - p_left)/h.
template <class AF, class AP>
__device__ __forceinline__ double mom(const LevelK& L, AF F, AP P, int64_t i, int64_t sn) {
    const int64_t sy = L.g.sy, sz = L.g.sz;
    double s = F[i - 1] + F[i + 1];
    s = s + F[i - sy];
    s = s + F[i + sy];
    s = s + F[i - sz];
    s = s + F[i + sz];
    const double lap = 6.0 * F[i] - s;
    return L.eta_h2 * lap + (P[i] - P[i - sn]) * L.inv_h;
}

// Continuity row of L~ at cell slot i: -(div u)/h - gamma p.
template <class AU, class AV, class AW, class AP>
__device__ __forceinline__ double cont(const LevelK& L, AU U, AV V, AW W, AP P, int64_t i, double gamma) {
    const double div = (U[i + 1] - U[i]) + (V[i + L.g.sy] - V[i]) + (W[i + L.g.sz] - W[i]);
    return -div * L.inv_h - gamma * P[i];
}

// Labelled levels: momentum diagonal 6 - (dropped Neumann legs) of the low face `comp` of a cell
// (SPEC:124, 176), and the momentum row with that diagonal (the oracle's vdiag[f] * x[f] - s).
__device__ __forceinline__ double cls_diag(uint32_t c, int comp) {
    return static_cast<double>((c >> (CLS_DIAG_SHIFT + 3 * comp)) & 7u);
}
template <class AF, class AP>
__device__ __forceinline__ double mom_d(const LevelK& L, AF F, AP P, int64_t i, int64_t sn, double diag) {
    const int64_t sy = L.g.sy, sz = L.g.sz;
    double s = F[i - 1] + F[i + 1];
    s = s + F[i - sy];
    s = s + F[i + sy];
    s = s + F[i - sz];
    s = s + F[i + sz];
    const double lap = diag * F[i] - s;
    return L.eta_h2 * lap + (P[i] - P[i - sn]) * L.inv_h;
}

// ------------------------------------------------------------- apply ------
__global__ void k_apply(LevelK L, const double* __restrict__ X, const double* __restrict__ B,
                        double* __restrict__ Y, double gamma) {
    pdl_wait();
    Cell c;
    if (!thread_cell(L.g, c)) return;
    const Geom& g = L.g;
    const int64_t fs = g.fs;
    const double *U = X, *V = X + fs, *W = X + 2 * fs, *P = X + 3 * fs;
    const int64_t i = c.i;
    if (c.x >= 1) {
        const double y = mom(L, U, P, i, 1);
        Y[i] = B ? B[i] - y : y;
    }
    if (c.y >= 1) {
        const double y = mom(L, V, P, i, g.sy);
        Y[fs + i] = B ? B[fs + i] - y : y;
    }
    if (g.gz(c.z) >= 1) {
        const double y = mom(L, W, P, i, g.sz);
        Y[2 * fs + i] = B ? B[2 * fs + i] - y : y;
    }
    const double y = cont(L, U, V, W, P, i, gamma);
    Y[3 * fs + i] = B ? B[3 * fs + i] - y : y;
}

// ---------------------------------------------------------------- DGS ------
// Velocity phase (Alg. 2 with M_.j = e_j): GS on V2 faces of one red-black
// colour, x_f += (b_f - (L~x)_f) / d_v.  Same-colour faces do not couple.
__global__ void k_dgs_vel(LevelK L, double* __restrict__ X, const double* __restrict__ B, int colour) {
    Cell c;
    if (!thread_cell(L.g, c)) return;
    const Geom& g = L.g;
    if (((c.x + c.y + g.gz(c.z)) & 1) != colour) return;
    const int64_t fs = g.fs, i = c.i;
    double *U = X, *V = X + fs, *W = X + 2 * fs;
    const double* P = X + 3 * fs;
    const bool here = band_cell(L, c.x, c.y, c.z);
    if (c.x >= 1 && !here && !band_cell(L, c.x - 1, c.y, c.z)) {
        const double r = B[i] - mom(L, U, P, i, 1);
        U[i] = U[i] + r / L.dv;
    }
    if (c.y >= 1 && !here && !band_cell(L, c.x, c.y - 1, c.z)) {
        const double r = B[fs + i] - mom(L, V, P, i, g.sy);
        V[i] = V[i] + r / L.dv;
    }
    if (g.gz(c.z) >= 1 && !here && !band_cell(L, c.x, c.y, c.z - 1)) {
        const double r = B[2 * fs + i] - mom(L, W, P, i, g.sz);
        W[i] = W[i] + r / L.dv;
    }
}

__device__ __forceinline__ int pcolour(const Geom& g, const Cell& c) {
    return (c.x & 1) + 2 * (c.y & 1) + 4 * (g.gz(c.z) & 1);
}

// Forward pressure phase, part 1: delta_C = (b_C - (L~x)_C) / d_p on V2 cells of
// the parity colour (8 colours, OD-1), 0 elsewhere (written for every cell).
__global__ void k_dgs_pdelta(LevelK L, const double* __restrict__ X, const double* __restrict__ B,
                             double* __restrict__ D, int colour) {
    Cell c;
    if (!thread_cell(L.g, c)) return;
    const int64_t fs = L.g.fs, i = c.i;
    double d = 0.0;
    if (pcolour(L.g, c) == colour && !band_cell(L, c.x, c.y, c.z)) {
        const double r = B[3 * fs + i] - cont(L, X, X + fs, X + 2 * fs, X + 3 * fs, i, L.gamma);
        d = r / L.dp;
    }
    D[i] = d;
}

// Forward pressure phase, part 2: x += sum_C delta_C M_.C in gather form
// (faces: (delta_left - delta_right)/h; pressures: eta/h^2 (6 delta - sum nbr)).
__global__ void k_dgs_papply(LevelK L, double* __restrict__ X, const double* __restrict__ D) {
    Cell c;
    if (!thread_cell(L.g, c)) return;
    const Geom& g = L.g;
    const int64_t fs = g.fs, i = c.i, sy = g.sy, sz = g.sz;
    const double dc = D[i];
    if (c.x >= 1) X[i] = X[i] + (D[i - 1] - dc) * L.inv_h;
    if (c.y >= 1) X[fs + i] = X[fs + i] + (D[i - sy] - dc) * L.inv_h;
    if (g.gz(c.z) >= 1) X[2 * fs + i] = X[2 * fs + i] + (D[i - sz] - dc) * L.inv_h;
    double s = D[i - 1] + D[i + 1];
    s = s + D[i - sy];
    s = s + D[i + sy];
    s = s + D[i - sz];
    s = s + D[i + sz];
    X[3 * fs + i] = X[3 * fs + i] + L.eta_h2 * (6.0 * dc - s);
}

// Reverse (left-preconditioned) pressure phase: x_C += m_C^T (b - L~x) / d_p on
// V2 cells of the parity colour (radius-2 gather; same-colour cells are never
// face neighbours and never read each other's pressure: one pass is race-free).
template <class AX>
__device__ __forceinline__ double prev_value(const LevelK& L, AX X, int64_t i);
__global__ void k_dgs_prev(LevelK L, double* __restrict__ X, const double* __restrict__ B, int colour) {
    (void)B;
    Cell c;
    if (!thread_cell(L.g, c)) return;
    if (pcolour(L.g, c) != colour || band_cell(L, c.x, c.y, c.z)) return;
    X[3 * L.g.fs + c.i] = prev_value(L, X, c.i);
}

// c_b = m_C^T b: the b part of the reverse pressure update, same operation order as
// the L~x part in prev_value (faces right - left in x, y, z; 6 r_C - neighbours x-, x+, ...).
// PACK (tiled levels): also L.bp, the level's b and c_b in tile-major order -- per 16 x 8 x 8 tile
// (x fastest) 5 blocks of 1024 doubles: b_u, b_v, b_w, b_p in the tile kernel's x-parity-split row
// order (tile_bi) and c_b in natural order (tile_ti), 40 KB contiguous.  b is fixed during a level
// visit while k_dgs_tile stages a tile's b 32 times (2 smooths x 16 launches): from the padded level
// vector every 128-byte tile row straddles two DRAM lines (2x over-fetch); from L.bp it is one
// contiguous bulk copy, already split.
template <bool PACK>
__global__ void k_dgs_cb(LevelK L, const double* __restrict__ B, double* __restrict__ CB) {
    pdl_wait();
    Cell c;
    if (!thread_cell(L.g, c)) return;
    const Geom& g = L.g;
    const int64_t fs = g.fs, sy = g.sy, sz = g.sz, i = c.i;
    const double *BU = B, *BV = B + fs, *BW = B + 2 * fs, *BP = B + 3 * fs;
    const double fl = ((BU[i + 1] - BU[i]) + (BV[i + sy] - BV[i])) + (BW[i + sz] - BW[i]);
    double s = BP[i - 1] + BP[i + 1];
    s = s + BP[i - sy];
    s = s + BP[i + sy];
    s = s + BP[i - sz];
    s = s + BP[i + sz];
    const double cb = fl * L.inv_h + L.eta_h2 * (6.0 * BP[i] - s);
    CB[i] = cb;
    if (PACK) {
        const int tx = c.x >> 4, ty = c.y >> 3, tz = c.z >> 3, lx = c.x & 15, ly = c.y & 7, lz = c.z & 7;
        double* t = L.bp + (static_cast<int64_t>(tz * (g.ny >> 3) + ty) * (g.nx >> 4) + tx) * 5120;
        const int bi = ((lz * 8 + ly) << 4) + (lx & 1) * 8 + (lx >> 1);
        t[bi] = BU[i];
        t[1024 + bi] = BV[i];
        t[2048 + bi] = BW[i];
        t[3072 + bi] = BP[i];
        t[4096 + (lz * 8 + ly) * 16 + lx] = cb;
    }
}

__global__ void k_vanka_apply(LevelK L, double* __restrict__ X, const int32_t* __restrict__ cells,
                              const uint8_t* __restrict__ masks, int n, const double* __restrict__ delta,
                              const uint8_t* __restrict__ amask) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const Geom& g = L.g;
    const int64_t fs = g.fs, i = cells[t];
    // amask (z-slabs): which of the 7 slots this part owns (bit 6 = pressure)
    const int am = amask ? amask[t] : 127;
    const int m = masks[t] & am;
    const double* d = delta + static_cast<int64_t>(t) * 8;
    if (m & 1) X[i] = X[i] + d[0];
    if (m & 2) X[i + 1] = X[i + 1] + d[1];
    if (m & 4) X[fs + i] = X[fs + i] + d[2];
    if (m & 8) X[fs + i + g.sy] = X[fs + i + g.sy] + d[3];
    if (m & 16) X[2 * fs + i] = X[2 * fs + i] + d[4];
    if (m & 32) X[2 * fs + i + g.sz] = X[2 * fs + i + g.sz] + d[5];
    if (am & 64) X[3 * fs + i] = X[3 * fs + i] + d[6];
}

// ------------------------------------------------------------ transfer ------
// Restriction R = (1/8) P^T, gathered per coarse DOF.  Weight
// tables: normal {1/2, 1, 1/2} over fine faces 2I-1..2I+1, tangential
// {1/4, 3/4, 3/4, 1/4} over fine cells 2J-1..2J+2; summation order: normal
// innermost, then the tangential axes in x,y,z order.
__device__ __forceinline__ double restrict_face(const double* __restrict__ R, int64_t base, int64_t sn,
                                                int64_t sa, int64_t sb) {
    // base = fine slot of (normal 2I, tangential 2J, 2K); legs offset from it
    const double wI[3] = {0.5, 1.0, 0.5};
    const double wT[4] = {0.25, 0.75, 0.75, 0.25};
    double acc_b = 0.0;
#pragma unroll
    for (int ib = 0; ib < 4; ++ib) {
        double acc_a = 0.0;
#pragma unroll
        for (int ia = 0; ia < 4; ++ia) {
            const int64_t o = base + (ib - 1) * sb + (ia - 1) * sa;
            double sn_ = 0.0;
#pragma unroll
            for (int in = 0; in < 3; ++in) sn_ = sn_ + wI[in] * R[o + (in - 1) * sn];
            acc_a = acc_a + wT[ia] * sn_;
        }
        acc_b = acc_b + wT[ib] * acc_a;
    }
    return 0.125 * acc_b;
}

__global__ void k_restrict(LevelK F, LevelK C, const double* __restrict__ R, double* __restrict__ BC, int zc_lo) {
    pdl_wait();
    const Geom &fg = F.g, &cg = C.g;
    Cell c;
    c.x = blockIdx.x * BX + threadIdx.x;
    c.y = blockIdx.y * BY + threadIdx.y;
    c.z = zc_lo + blockIdx.z;
    if (c.x >= cg.nx || c.y >= cg.ny) return;
    c.i = cg.slot(c.x, c.y, c.z);
    const int64_t ffs = fg.fs, cfs = cg.fs;
    const int fz = 2 * cg.gz(c.z) - fg.z0;  // fine local plane of the coarse cell's lower child
    const int64_t fb = fg.slot(2 * c.x, 2 * c.y, fz);
    const int64_t sx = 1, sy = fg.sy, sz = fg.sz;
    if (c.x >= 1) BC[c.i] = restrict_face(R, fb, sx, sy, sz);                   // u: a = y, b = z
    if (c.y >= 1) BC[cfs + c.i] = restrict_face(R + ffs, fb, sy, sx, sz);       // v: a = x, b = z
    if (cg.gz(c.z) >= 1) BC[2 * cfs + c.i] = restrict_face(R + 2 * ffs, fb, sz, sx, sy);  // w: a = x, b = y
    const double* RP = R + 3 * ffs;
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int ii = 0; ii < 2; ++ii) s = s + RP[fb + k * sz + j * sy + ii];
    BC[3 * cfs + c.i] = 0.125 * s;
}

// z-marching restriction: a thread owns one coarse column (x, y) and walks a segment of
// coarse planes.  For the u and v faces the tangential-b axis is z, so restrict_face's inner
// partial acc_a depends on the fine plane only: computed once per fine plane (same
// operations), it serves coarse planes K and K+1 (fine planes 2K+1, 2K+2 are 2K'-1, 2K' of
// K' = K+1).  For w the normal axis is z: the 16 values of fine plane 2K+1 are kept in
// registers for the next coarse plane.  Loads per coarse cell 152 -> 88; every sum is
// restrict_face's in the same order, so the result is bit-identical to k_restrict.
// u: normal x, a = y, b = z.  v: normal y, a = x, b = z.
// build-time A/B: CTAs per SM the register allocation of k_restrict_zm targets.  4 (64 registers, no
// spill) measured slower than the free allocation (80 registers, 3 CTAs/SM): cfg 3 fine restrict
// 1.27 -> 1.65 ms (profiles/r1s5_rzm4_ab.txt)
#ifndef SMG_RZM_MINB
#define SMG_RZM_MINB 1
#endif
__device__ __forceinline__ double restrict_partial_a(const double* __restrict__ R, int64_t o, int64_t sn,
                                                     int64_t sa) {
    // o = fine slot (normal 2I, a 2J, plane zf); acc_a of restrict_face for that plane
    const double wI[3] = {0.5, 1.0, 0.5};
    const double wT[4] = {0.25, 0.75, 0.75, 0.25};
    double acc_a = 0.0;
#pragma unroll
    for (int ia = 0; ia < 4; ++ia) {
        double sn_ = 0.0;
#pragma unroll
        for (int in = 0; in < 3; ++in) sn_ = sn_ + wI[in] * R[o + (ia - 1) * sa + (in - 1) * sn];
        acc_a = acc_a + wT[ia] * sn_;
    }
    return acc_a;
}

__global__ void __launch_bounds__(256, SMG_RZM_MINB) k_restrict_zm(LevelK F, LevelK C, const double* __restrict__ R,
                                                     double* __restrict__ BC, int zc_lo, int zc_hi, int zseg) {
    pdl_wait();
    const Geom &fg = F.g, &cg = C.g;
    const int cx = blockIdx.x * BX + threadIdx.x, cy = blockIdx.y * BY + threadIdx.y;
    if (cx >= cg.nx || cy >= cg.ny) return;
    const int K0 = zc_lo + blockIdx.z * zseg, K1 = min(K0 + zseg, zc_hi);
    if (K0 >= K1) return;
    const int64_t ffs = fg.fs, cfs = cg.fs;
    const int64_t sx = 1, sy = fg.sy, sz = fg.sz;
    const double *RU = R, *RV = R + ffs, *RW = R + 2 * ffs, *RP = R + 3 * ffs;
    const double wI[3] = {0.5, 1.0, 0.5};
    const double wT[4] = {0.25, 0.75, 0.75, 0.25};
    // fine slot of (2cx, 2cy, local fine plane 2K) for coarse local plane K
    auto fbase = [&](int K) { return fg.slot(2 * cx, 2 * cy, 2 * cg.gz(K) - fg.z0); };
    int64_t fb = fbase(K0);
    // fine planes 2K-1 and 2K of the first coarse plane
    double au0 = restrict_partial_a(RU, fb - sz, sx, sy), au1 = restrict_partial_a(RU, fb, sx, sy);
    double av0 = restrict_partial_a(RV, fb - sz, sy, sx), av1 = restrict_partial_a(RV, fb, sy, sx);
    double wm[4][4];  // w at fine plane 2K-1: [ib (y)][ia (x)]
#pragma unroll
    for (int ib = 0; ib < 4; ++ib)
#pragma unroll
        for (int ia = 0; ia < 4; ++ia) wm[ib][ia] = RW[fb - sz + (ib - 1) * sy + (ia - 1) * sx];
    for (int K = K0; K < K1; ++K) {
        if (K > K0) fb = fbase(K);
        const int64_t ci = cg.slot(cx, cy, K);
        const double au2 = restrict_partial_a(RU, fb + sz, sx, sy), au3 = restrict_partial_a(RU, fb + 2 * sz, sx, sy);
        const double av2 = restrict_partial_a(RV, fb + sz, sy, sx), av3 = restrict_partial_a(RV, fb + 2 * sz, sy, sx);
        if (cx >= 1) {
            double acc_b = 0.0;
            acc_b = acc_b + wT[0] * au0;
            acc_b = acc_b + wT[1] * au1;
            acc_b = acc_b + wT[2] * au2;
            acc_b = acc_b + wT[3] * au3;
            BC[ci] = 0.125 * acc_b;
        }
        if (cy >= 1) {
            double acc_b = 0.0;
            acc_b = acc_b + wT[0] * av0;
            acc_b = acc_b + wT[1] * av1;
            acc_b = acc_b + wT[2] * av2;
            acc_b = acc_b + wT[3] * av3;
            BC[cfs + ci] = 0.125 * acc_b;
        }
        au0 = au2;
        au1 = au3;
        av0 = av2;
        av1 = av3;
        // w: normal z innermost over fine planes 2K-1 (carried), 2K, 2K+1 (carried on)
        double acc_b = 0.0;
#pragma unroll
        for (int ib = 0; ib < 4; ++ib) {
            double acc_a = 0.0;
#pragma unroll
            for (int ia = 0; ia < 4; ++ia) {
                const int64_t o = fb + (ib - 1) * sy + (ia - 1) * sx;
                const double w1 = RW[o], w2 = RW[o + sz];
                double sn_ = 0.0;
                sn_ = sn_ + wI[0] * wm[ib][ia];
                sn_ = sn_ + wI[1] * w1;
                sn_ = sn_ + wI[2] * w2;
                acc_a = acc_a + wT[ia] * sn_;
                wm[ib][ia] = w2;
            }
            acc_b = acc_b + wT[ib] * acc_a;
        }
        if (cg.gz(K) >= 1) BC[2 * cfs + ci] = 0.125 * acc_b;
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int ii = 0; ii < 2; ++ii) s = s + RP[fb + k * sz + j * sy + ii];
        BC[3 * cfs + ci] = 0.125 * s;
    }
}


// Prolongation x_f += P e_c.  Tangential legs of fine index J:
// (J>>1, 3/4) then (J odd ? (J>>1)+1 : (J>>1)-1, 1/4); normal: I even ->
// (I/2, 1), I odd -> ((I-1)/2, 1/2), ((I+1)/2, 1/2).  Legs to wall/ghost slots
// read 0 (dropped, no renormalisation).
// (fx, fy, fz) are GLOBAL fine indices; coarse slots are addressed through
// cg.slot with local coarse planes (cg.z0 subtracted).
// Unrolled per component: the coarse legs are base, base + da (second tangential
// a leg), base + db, base + db + da, and + dn for the second normal leg; the same
// operations in the same order as the loop form (normal innermost, then a, then b).
template <int COMP>
__device__ __forceinline__ double prolong_face(const double* __restrict__ E, const Geom& cg, int fx, int fy, int fz) {
    constexpr int TA = COMP == 0 ? 1 : 0, TB = COMP == 2 ? 1 : 2;
    const int f[3] = {fx, fy, fz};
    const int I = f[COMP];
    int c[3];
    c[COMP] = I >> 1;  // even I: I/2 (weight 1); odd I: (I-1)/2 and (I+1)/2 (1/2 each)
    c[TA] = f[TA] >> 1;
    c[TB] = f[TB] >> 1;
    const int64_t st[3] = {1, cg.sy, cg.sz};
    const int64_t base = cg.slot(c[0], c[1], c[2] - cg.z0);
    const int64_t da = (f[TA] & 1) ? st[TA] : -st[TA];
    const int64_t db = (f[TB] & 1) ? st[TB] : -st[TB];
    const int64_t dn = st[COMP];
    const bool odd = I & 1;
    auto sn = [&](int64_t o) {
        double s = 0.0;
        if (!odd) {
            s = s + 1.0 * E[o];
        } else {
            s = s + 0.5 * E[o];
            s = s + 0.5 * E[o + dn];
        }
        return s;
    };
    const double s00 = sn(base), s01 = sn(base + da), s10 = sn(base + db), s11 = sn(base + db + da);
    double sb = 0.0;
    double sa = 0.0;
    sa = sa + 0.75 * s00;
    sa = sa + 0.25 * s01;
    sb = sb + 0.75 * sa;
    sa = 0.0;
    sa = sa + 0.75 * s10;
    sa = sa + 0.25 * s11;
    sb = sb + 0.25 * sa;
    return sb;
}

__global__ void k_prolong_add(LevelK F, LevelK C, const double* __restrict__ E, double* __restrict__ X) {
    pdl_wait();
    Cell c;
    if (!thread_cell(F.g, c)) return;
    const Geom &fg = F.g, &cg = C.g;
    const int64_t ffs = fg.fs, cfs = cg.fs;
    const int z = fg.gz(c.z);
    if (c.x >= 1) X[c.i] = X[c.i] + prolong_face<0>(E, cg, c.x, c.y, z);
    if (c.y >= 1) X[ffs + c.i] = X[ffs + c.i] + prolong_face<1>(E + cfs, cg, c.x, c.y, z);
    if (z >= 1) X[2 * ffs + c.i] = X[2 * ffs + c.i] + prolong_face<2>(E + 2 * cfs, cg, c.x, c.y, z);
    X[3 * ffs + c.i] = X[3 * ffs + c.i] + E[3 * cfs + cg.slot(c.x >> 1, c.y >> 1, (z >> 1) - cg.z0)];
}


// ------------------------------------------------------------- coarse ------
// x = K b with the symmetric dense inverse K (OD-4).  Fixed order: partial sums
// over 64-column chunks, chunks accumulated in ascending order (same as the
// oracle).  K symmetric => column j of K is row j, read coalesced across rows.
constexpr int CG_ROWS = 32, CG_LANES = 32;
__global__ void k_coarse_gemv(const double* __restrict__ K, const int32_t* __restrict__ slots, int n,
                              const double* __restrict__ B, double* __restrict__ X, int accumulate) {
    pdl_wait();
    extern __shared__ double part[];  // [nchunks][CG_ROWS]
    const int row = blockIdx.x * CG_ROWS + threadIdx.x;
    const int nchunks = (n + 63) / 64;
    for (int ch = threadIdx.y; ch < nchunks; ch += CG_LANES) {
        double p = 0.0;
        if (row < n) {
            const int j1 = min(n, ch * 64 + 64);
            for (int j = ch * 64; j < j1; ++j) p = p + K[static_cast<int64_t>(j) * n + row] * __ldg(&B[slots[j]]);
        }
        part[ch * CG_ROWS + threadIdx.x] = p;
    }
    __syncthreads();
    if (threadIdx.y == 0 && row < n) {
        double s = 0.0;
        for (int ch = 0; ch < nchunks; ++ch) s = s + part[ch * CG_ROWS + threadIdx.x];
        X[slots[row]] = accumulate ? X[slots[row]] + s : s;
    }
}

// --------------------------------------------------------- pack/unpack ------
// Compact FieldVector order: u (x in 1..nx-1), v, w, p, each lexicographic with
// x fastest.
__global__ void k_pack(LevelK L, const double* __restrict__ X, double* __restrict__ out, int unpack) {
    pdl_wait();
    Cell c;
    if (!thread_cell(L.g, c)) return;
    const Geom& g = L.g;
    const int64_t nx = g.nx, ny = g.ny, nz = g.gnz, fs = g.fs;
    const int64_t nu = (nx - 1) * ny * nz, nv = nx * (ny - 1) * nz, nw = nx * ny * (nz - 1);
    const int64_t x = c.x, y = c.y, z = g.gz(c.z);
    if (x >= 1) {
        const int64_t k = (z * ny + y) * (nx - 1) + (x - 1);
        if (unpack) const_cast<double*>(X)[c.i] = out[k]; else out[k] = X[c.i];
    }
    if (y >= 1) {
        const int64_t k = nu + (z * (ny - 1) + (y - 1)) * nx + x;
        if (unpack) const_cast<double*>(X)[fs + c.i] = out[k]; else out[k] = X[fs + c.i];
    }
    if (z >= 1) {
        const int64_t k = nu + nv + ((z - 1) * ny + y) * nx + x;
        if (unpack) const_cast<double*>(X)[2 * fs + c.i] = out[k]; else out[k] = X[2 * fs + c.i];
    }
    const int64_t k = nu + nv + nw + (z * ny + y) * nx + x;
    if (unpack) const_cast<double*>(X)[3 * fs + c.i] = out[k]; else out[k] = X[3 * fs + c.i];
}

// ------------------------------------------------------------- BLAS-1 ------
constexpr int RED_T = 256;

// Canonical inner product (OD-12 rev. 2) -- the order the fused SQMR kernels
// produce natively, restated by the oracle (cdot in oracle/stokes_oracle.cpp):
//   * a block is 32 x-lanes by 8 y-rows of one z-block of kDotZB planes (the k_apply grid);
//   * a thread adds, over its cell's planes in ascending z, ((p_u + p_v) + p_w) + p_p, the
//     products of the four fields at the cell's slot (inactive slots hold 0: product +0);
//   * the 32 lanes of a row combine by the shuffle-down tree (o = 16..1), the 8 row sums are
//     added in ascending row order into the block partial, stored at the global block index
//     ((zb * GY + by) * GX + bx) -- so z-slab parts fill disjoint entries;
//   * k_final: thread t of 256 adds partials t, t + 256, ... in ascending order, then the
//     shuffle-down tree per warp, then the 8 warp sums in ascending order.
constexpr int kDotZB = kDotZBlock;
__device__ __forceinline__ double cell4(double pu, double pv, double pw, double pp) { return ((pu + pv) + pw) + pp; }

// block partials of up to two products, written to part[blk] and part[nblk + blk]
__device__ __forceinline__ void block_partial2(double v0, double v1, double* __restrict__ part, int64_t nblk,
                                               int64_t blk) {
    __shared__ double ws0[8], ws1[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v0 = v0 + __shfl_down_sync(0xffffffffu, v0, o);
        v1 = v1 + __shfl_down_sync(0xffffffffu, v1, o);
    }
    if (threadIdx.x == 0) {
        ws0[threadIdx.y] = v0;
        ws1[threadIdx.y] = v1;
    }
    __syncthreads();
    if (threadIdx.x == 0 && threadIdx.y == 0) {
        double s0 = ws0[0], s1 = ws1[0];
#pragma unroll
        for (int w = 1; w < 8; ++w) {
            s0 = s0 + ws0[w];
            s1 = s1 + ws1[w];
        }
        part[blk] = s0;
        part[nblk + blk] = s1;
    }
}
// the same block reduction of one value, stored as the block's partial of the SECOND inner product
// (the first one's slot, written by an earlier kernel of the same pair, stays)
__device__ __forceinline__ void block_partial_second(double v0, double* __restrict__ part, int64_t nblk, int64_t blk) {
    __shared__ double ws0[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v0 = v0 + __shfl_down_sync(0xffffffffu, v0, o);
    if (threadIdx.x == 0) ws0[threadIdx.y] = v0;
    __syncthreads();
    if (threadIdx.x == 0 && threadIdx.y == 0) {
        double s0 = ws0[0];
#pragma unroll
        for (int w = 1; w < 8; ++w) s0 = s0 + ws0[w];
        part[nblk + blk] = s0;
    }
}
// global block index of this CTA; grid (GX, GY, local z-blocks), slab parts start on a z-block
__device__ __forceinline__ int64_t dot_blk(const Geom& g) {
    const int64_t GX = gridDim.x, GY = gridDim.y;
    const int64_t zb = blockIdx.z + g.z0 / kDotZB;
    return (zb * GY + blockIdx.y) * GX + blockIdx.x;
}
__host__ __device__ inline int64_t dot_nblk(const Geom& g) {
    return static_cast<int64_t>((g.nx + 31) / 32) * ((g.ny + 7) / 8) * ((g.gnz + kDotZB - 1) / kDotZB);
}

__global__ void __launch_bounds__(RED_T) k_cdot(Geom g, const double* __restrict__ a, const double* __restrict__ b,
                                                const double* __restrict__ c, const double* __restrict__ d,
                                                double* __restrict__ partials) {
    pdl_wait();
    const int x = blockIdx.x * 32 + threadIdx.x, y = blockIdx.y * 8 + threadIdx.y;
    const int zl = blockIdx.z * kDotZB, zh = min(g.nz, zl + kDotZB);
    const int64_t fs = g.fs;
    double v0 = 0.0, v1 = 0.0;
    if (x < g.nx && y < g.ny)
        for (int z = zl; z < zh; ++z) {
            const int64_t i = g.slot(x, y, z);
            v0 = v0 + cell4(a[i] * b[i], a[fs + i] * b[fs + i], a[2 * fs + i] * b[2 * fs + i],
                            a[3 * fs + i] * b[3 * fs + i]);
            if (c)
                v1 = v1 + cell4(c[i] * d[i], c[fs + i] * d[fs + i], c[2 * fs + i] * d[2 * fs + i],
                                c[3 * fs + i] * d[3 * fs + i]);
        }
    block_partial2(v0, v1, partials, dot_nblk(g), dot_blk(g));
}

// the final combination of nblk partials (two products); result to out[0], out[1]
__device__ __forceinline__ void final2(const double* __restrict__ part, int64_t nblk, double* out) {
    __shared__ double ws0[8], ws1[8];
    const int t = threadIdx.x;
    double s0 = 0.0, s1 = 0.0;
    for (int64_t k = t; k < nblk; k += 256) {
        s0 = s0 + part[k];
        s1 = s1 + part[nblk + k];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s0 = s0 + __shfl_down_sync(0xffffffffu, s0, o);
        s1 = s1 + __shfl_down_sync(0xffffffffu, s1, o);
    }
    if ((t & 31) == 0) {
        ws0[t >> 5] = s0;
        ws1[t >> 5] = s1;
    }
    __syncthreads();
    if (t == 0) {
        double a = ws0[0], b = ws1[0];
#pragma unroll
        for (int w = 1; w < 8; ++w) {
            a = a + ws0[w];
            b = b + ws1[w];
        }
        out[0] = a;
        out[1] = b;
    }
}
__global__ void __launch_bounds__(256) k_cdot_final(const double* __restrict__ partials, int64_t nblk,
                                                    double* __restrict__ out) {
    pdl_wait();
    final2(partials, nblk, out);
}

// ---- fused SQMR steps (Alg. 4; north_star: AXPYs fused with the inner products) ----
// The vector updates are evaluated on the fly at every slot a stencil reads, with the oracle's
// per-element expressions: q_new = t + beta q (line 9), x_new = x + (cd d + cq q) (line 7); each
// thread stores the new values of its own cell only.
// The momentum row (mom) and continuity row (cont) of the contract on a vector given by an
// index functor v(j) (absolute indices, field f at f * fs): the same operand order.
template <class VF>
__device__ __forceinline__ double mom_f(const LevelK& L, const VF& v, int64_t i, int64_t sn, int64_t po,
                                        double diag = 6.0) {
    double s = v(i - 1) + v(i + 1);
    s = s + v(i - L.g.sy);
    s = s + v(i + L.g.sy);
    s = s + v(i - L.g.sz);
    s = s + v(i + L.g.sz);
    const double lap = diag * v(i) - s;
    return L.eta_h2 * lap + (v(po) - v(po - sn)) * L.inv_h;
}
template <class VF>
__device__ __forceinline__ double cont_f(const LevelK& L, const VF& v, int64_t i, double gamma) {
    const int64_t fs = L.g.fs;
    const double div = (v(i + 1) - v(i)) + (v(fs + i + L.g.sy) - v(fs + i)) + (v(2 * fs + i + L.g.sz) - v(2 * fs + i));
    return -div * L.inv_h - gamma * v(3 * fs + i);
}

// Lines 9 + 5 of iteration j: q = t + beta q (written to Q1), t = L q (to Tn), sigma = q.t as
// block partials.  Grid = the dot grid; on slab parts with a neighbour below / above, the
// first / last z-block also writes q on the ghost plane -1 / nz (its inputs are valid there),
// so the next iteration needs no exchange of q.
// M: general labelled level (activity and momentum diagonals from L.cls instead of coordinates).
// UPD: the vector update is evaluated on the fly (one pass over the vectors); !UPD: the update has
// been written by k_q_upd / k_xd_upd (a streaming pass at copy bandwidth) and the stencil reads the
// stored vector -- one load per stencil point instead of two or three (same values, same bits).
template <bool M, bool UPD>
__global__ void __launch_bounds__(256) k_apply_q(LevelK L, const double* __restrict__ T,
                                                 const double* __restrict__ Q0, double* __restrict__ Q1,
                                                 double* __restrict__ Tn, const double* __restrict__ sc,
                                                 double* __restrict__ partials, int halo_lo, int halo_hi, int second) {
    pdl_wait();
    if (sc[S_STATUS] != 0.0) return;
    const Geom& g = L.g;
    const int64_t fs = g.fs;
    const double beta = sc[S_BETA];
    auto q = [&](int64_t j) { return UPD ? T[j] + beta * Q0[j] : Q1[j]; };  // the oracle's q[i] = t[i] + beta q[i]
    const int x = blockIdx.x * 32 + threadIdx.x, y = blockIdx.y * 8 + threadIdx.y;
    const int zl = blockIdx.z * kDotZB, zh = min(g.nz, zl + kDotZB);
    double v = 0.0;
    if (x < g.nx && y < g.ny) {
        auto put_q = [&](int64_t i) {
#pragma unroll
            for (int f = 0; f < 4; ++f) Q1[f * fs + i] = q(f * fs + i);
        };
        if (UPD && halo_lo && blockIdx.z == 0) put_q(g.slot(x, y, -1));
        if (UPD && halo_hi && zh == g.nz) put_q(g.slot(x, y, g.nz));
#pragma unroll 1
        for (int z = zl; z < zh; ++z) {
            const int64_t i = g.slot(x, y, z);
            const uint32_t cm = M ? L.cls[i] : 0u;
            double c4;
            {
                const double qu = q(i);
                double tu = 0.0;
                if (M ? (cm & CLS_U) != 0 : x >= 1) Tn[i] = tu = mom_f(L, q, i, 1, 3 * fs + i, M ? cls_diag(cm, 0) : 6.0);
                if (UPD) Q1[i] = qu;
                c4 = qu * tu;
            }
            {
                const double qv = q(fs + i);
                double tv = 0.0;
                if (M ? (cm & CLS_V) != 0 : y >= 1)
                    Tn[fs + i] = tv = mom_f(L, q, fs + i, g.sy, 3 * fs + i, M ? cls_diag(cm, 1) : 6.0);
                if (UPD) Q1[fs + i] = qv;
                c4 = c4 + qv * tv;
            }
            {
                const double qw = q(2 * fs + i);
                double tw = 0.0;
                if (M ? (cm & CLS_W) != 0 : g.gz(z) >= 1)
                    Tn[2 * fs + i] = tw = mom_f(L, q, 2 * fs + i, g.sz, 3 * fs + i, M ? cls_diag(cm, 2) : 6.0);
                if (UPD) Q1[2 * fs + i] = qw;
                c4 = c4 + qw * tw;
            }
            const double qp = q(3 * fs + i);
            double tp = 0.0;
            if (!M || (cm & CLS_P)) Tn[3 * fs + i] = tp = cont_f(L, q, i, 0.0);
            if (UPD) Q1[3 * fs + i] = qp;
            v = v + (c4 + qp * tp);  // ((p_u + p_v) + p_w) + p_p
        }
    }
    // second: sigma of the NEXT iteration rides in the second slot next to this iteration's ||r||^2
    if (second) block_partial_second(v, partials, dot_nblk(g), dot_blk(g));
    else block_partial2(v, 0.0, partials, dot_nblk(g), dot_blk(g));
}

// Lines 7 + 8 of iteration j: d = cd d + cq q, x = x + d (written to D1, X1), then the true
// residual r = b - L x as block partials of ||r||^2 (r itself is never stored).  Ghost planes
// as in k_apply_q.
template <bool M, bool UPD>
__global__ void __launch_bounds__(256, M ? 3 : 4) k_apply_x(LevelK L, const double* __restrict__ X0,
                                                 const double* __restrict__ D0, const double* __restrict__ Q,
                                                 const double* __restrict__ B, double* __restrict__ X1,
                                                 double* __restrict__ D1, const double* __restrict__ sc,
                                                 double* __restrict__ partials, int halo_lo, int halo_hi) {
    pdl_wait();
    if (sc[S_STATUS] != 0.0) return;
    const Geom& g = L.g;
    const int64_t fs = g.fs;
    const double cd = sc[S_CD], cq = sc[S_CQ];
    auto dn = [&](int64_t j) { return cd * D0[j] + cq * Q[j]; };  // the oracle's d[i] = cd d[i] + cq q[i]
    auto xn = [&](int64_t j) { return UPD ? X0[j] + dn(j) : X1[j]; };  // x[i] = x[i] + d[i]
    const int x = blockIdx.x * 32 + threadIdx.x, y = blockIdx.y * 8 + threadIdx.y;
    const int zl = blockIdx.z * kDotZB, zh = min(g.nz, zl + kDotZB);
    double v = 0.0;
    if (x < g.nx && y < g.ny) {
        auto put_xd = [&](int64_t i) {
#pragma unroll
            for (int f = 0; f < 4; ++f) {
                const double d = dn(f * fs + i);
                D1[f * fs + i] = d;
                X1[f * fs + i] = X0[f * fs + i] + d;
            }
        };
        if (UPD && halo_lo && blockIdx.z == 0) put_xd(g.slot(x, y, -1));
        if (UPD && halo_hi && zh == g.nz) put_xd(g.slot(x, y, g.nz));
#pragma unroll 1
        for (int z = zl; z < zh; ++z) {
            const int64_t i = g.slot(x, y, z);
            const uint32_t cm = M ? L.cls[i] : 0u;
            double ru = 0.0, rv = 0.0, rw = 0.0, rp = 0.0;
            if (M ? (cm & CLS_U) != 0 : x >= 1) ru = B[i] - mom_f(L, xn, i, 1, 3 * fs + i, M ? cls_diag(cm, 0) : 6.0);
            if (M ? (cm & CLS_V) != 0 : y >= 1)
                rv = B[fs + i] - mom_f(L, xn, fs + i, g.sy, 3 * fs + i, M ? cls_diag(cm, 1) : 6.0);
            if (M ? (cm & CLS_W) != 0 : g.gz(z) >= 1)
                rw = B[2 * fs + i] - mom_f(L, xn, 2 * fs + i, g.sz, 3 * fs + i, M ? cls_diag(cm, 2) : 6.0);
            if (!M || (cm & CLS_P)) rp = B[3 * fs + i] - cont_f(L, xn, i, 0.0);
            if (UPD) put_xd(i);
            v = v + cell4(ru * ru, rv * rv, rw * rw, rp * rp);
        }
    }
    block_partial2(v, 0.0, partials, dot_nblk(g), dot_blk(g));
}

// The SQMR vector updates as streaming passes (for the !UPD stencil kernels): per cell of the level
// (and of the ghost planes a slab part fills for its neighbours), all four fields.
__global__ void __launch_bounds__(256) k_q_upd(Geom g, const double* __restrict__ T, const double* __restrict__ Q0,
                                               double* __restrict__ Q1, const double* __restrict__ sc, int halo_lo,
                                               int halo_hi) {
    pdl_wait();
    if (sc[S_STATUS] != 0.0) return;
    const int x = blockIdx.x * BX + threadIdx.x, y = blockIdx.y * BY + threadIdx.y;
    const int z = static_cast<int>(blockIdx.z) - halo_lo;
    if (x >= g.nx || y >= g.ny || z >= g.nz + halo_hi) return;
    const double beta = sc[S_BETA];
    const int64_t i = g.slot(x, y, z), fs = g.fs;
#pragma unroll
    for (int f = 0; f < 4; ++f) Q1[f * fs + i] = T[f * fs + i] + beta * Q0[f * fs + i];
}
__global__ void __launch_bounds__(256) k_xd_upd(Geom g, const double* __restrict__ X0, const double* __restrict__ D0,
                                                const double* __restrict__ Q, double* __restrict__ X1,
                                                double* __restrict__ D1, const double* __restrict__ sc, int halo_lo,
                                                int halo_hi) {
    pdl_wait();
    if (sc[S_STATUS] != 0.0) return;
    const int x = blockIdx.x * BX + threadIdx.x, y = blockIdx.y * BY + threadIdx.y;
    const int z = static_cast<int>(blockIdx.z) - halo_lo;
    if (x >= g.nx || y >= g.ny || z >= g.nz + halo_hi) return;
    const double cd = sc[S_CD], cq = sc[S_CQ];
    const int64_t i = g.slot(x, y, z), fs = g.fs;
#pragma unroll
    for (int f = 0; f < 4; ++f) {
        const double d = cd * D0[f * fs + i] + cq * Q[f * fs + i];
        D1[f * fs + i] = d;
        X1[f * fs + i] = X0[f * fs + i] + d;
    }
}

__global__ void k_axpy(double* __restrict__ y, const double* __restrict__ x, double alpha, int64_t n) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        y[k] = y[k] + alpha * x[k];
}
__global__ void k_xpby(double* __restrict__ y, const double* __restrict__ x, double beta, int64_t n) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        y[k] = x[k] + beta * y[k];
}
__global__ void k_dx_update(double* __restrict__ d, double* __restrict__ x, const double* __restrict__ q,
                            double cd, double cq, int64_t n) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const double dn = cd * d[k] + cq * q[k];
        d[k] = dn;
        x[k] = x[k] + dn;
    }
}

// ------------------------------------------- cooperative smoother sweeps ------
// One launch per symmetric sweep: the phases of the sweep run back to back in a
// persistent grid separated by grid-wide barriers (all blocks co-resident).
// Per-point arithmetic is the same as the single-phase kernels above.
namespace cg = cooperative_groups;

#ifdef SMG_TRACE  // tools-only build (make trace): per-warp phase timestamps of the Vanka sweep
__device__ unsigned long long* g_trace = nullptr;
__device__ __forceinline__ void trace_stamp(int ph, int stamp) {
    if (g_trace && (threadIdx.x & 31) == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        const int64_t w = (static_cast<int64_t>(ph) * gridDim.x + blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
        g_trace[w * 4 + stamp] = t;
    }
}
#define SMG_TRACE_STAMP(ph, k) trace_stamp(ph, k)
#else
#define SMG_TRACE_STAMP(ph, k)
#endif

// Barrier between phases: MODE 0 = whole cooperative grid, MODE 1 = one thread
// block cluster (<= 16 CTAs; barrier.cluster with release/acquire semantics).
template <int MODE>
__device__ __forceinline__ void phase_sync() {
    if constexpr (MODE == 0) cg::this_grid().sync();
    else if constexpr (MODE == 1) cg::this_cluster().sync();
    else __syncthreads();  // MODE 2: single CTA (shared-memory-resident level)
}

struct VankaLists {
    const int32_t* cells[8];
    const uint8_t* masks[8];
    int n[8];
    // Lists are indexed by parity colour (i&1)+2(j&1)+4(k&1).  The sweep visits the parities
    // in the order kVankaOrder = 0,7,1,6,2,5,3,4 and back (oracle vanka_symmetric): every
    // adjacent pair (m, 7-m) differs in all three parities, no block of one reads or writes
    // a DOF of the other (each residual stencil reaches along one axis), so the pair runs as
    // ONE Jacobi phase with bit-identical results.  Bit m of `pairs` set: list m holds the
    // parity-m blocks (first first[m] entries) followed by the parity-(7-m) blocks and list
    // 7-m has no phase of its own.  All four pairs merged: 8 phases per symmetric sweep.
    int pairs;
    int first[4];
};
// phase k (0..15) of a symmetric sweep -> colour list, -1 if the phase is folded away
__device__ __forceinline__ int vanka_phase_list(const VankaLists& vl, int k) {
    const int j = k < 8 ? k : 15 - k;
    const int p = vanka_order(j);
    return ((j & 1) && ((vl.pairs >> (7 - p)) & 1)) ? -1 : p;
}
// parity colour of entry t of list c
__device__ __forceinline__ int vanka_entry_colour(const VankaLists& vl, int c, int t) {
    return (c < 4 && ((vl.pairs >> c) & 1) && t >= vl.first[c]) ? 7 - c : c;
}
// parity colours a phase on list c updates (bit mask)
__device__ __forceinline__ int vanka_list_cmask(const VankaLists& vl, int c) {
    return (c < 4 && ((vl.pairs >> c) & 1)) ? ((1 << c) | (1 << (7 - c))) : (1 << c);
}

// nu symmetric multiplicative Vanka sweeps (kVankaOrder, then reversed), Jacobi
// within a colour.  Each thread owns up to CPT blocks of the colour: it loads
// their residual stencils, keeps the block's own 7 values and its correction
// in registers, waits at the barrier (all reads of the phase done), then
// stores own + delta (bit-identical to re-loading, since only this thread
// writes those DOFs in the phase) and waits again.  The 64 local inverses sit
// in shared memory.
template <int MODE, int CPT>
__device__ __forceinline__ void vanka_sweeps(const LevelK& L, double* __restrict__ X, const double* __restrict__ B,
                                             const VankaLists& vl, const double* __restrict__ Ks, int nu, int tid,
                                             int nth) {
    const Geom& g = L.g;
    const int64_t fs = g.fs, sy = g.sy, sz = g.sz;
    const int64_t off[7] = {0, 1, fs, fs + sy, 2 * fs, 2 * fs + sz, 3 * fs};
    for (int sweep = 0; sweep < nu; ++sweep)
        for (int k = 0; k < 16; ++k) {
            const int col = vanka_phase_list(vl, k);
            if (col < 0) continue;
            const int n = vl.n[col];
            int64_t slot[CPT];
            int msk[CPT];
            double own[CPT][7], dl[CPT][7];
#pragma unroll
            for (int j = 0; j < CPT; ++j) {
                const int t = tid + j * nth;
                msk[j] = -1;
                if (t >= n) continue;
                const int64_t i = vl.cells[col][t];
                const int m = vl.masks[col][t];
                slot[j] = i;
                msk[j] = m;
                const double *U = X, *V = X + fs, *W = X + 2 * fs, *P = X + 3 * fs;
                double r[7];
                r[0] = (m & 1) ? B[i] - mom(L, U, P, i, 1) : 0.0;
                r[1] = (m & 2) ? B[i + 1] - mom(L, U, P, i + 1, 1) : 0.0;
                r[2] = (m & 4) ? B[fs + i] - mom(L, V, P, i, sy) : 0.0;
                r[3] = (m & 8) ? B[fs + i + sy] - mom(L, V, P, i + sy, sy) : 0.0;
                r[4] = (m & 16) ? B[2 * fs + i] - mom(L, W, P, i, sz) : 0.0;
                r[5] = (m & 32) ? B[2 * fs + i + sz] - mom(L, W, P, i + sz, sz) : 0.0;
                r[6] = B[3 * fs + i] - cont(L, U, V, W, P, i, L.gamma);
#pragma unroll
                for (int q = 0; q < 7; ++q) own[j][q] = X[i + off[q]];
                const double* K = Ks + m * 49;
#pragma unroll
                for (int s2 = 0; s2 < 7; ++s2) {
                    double acc = 0.0;
#pragma unroll
                    for (int q = 0; q < 7; ++q) acc = acc + K[s2 * 7 + q] * r[q];
                    dl[j][s2] = acc;
                }
            }
            phase_sync<MODE>();
#pragma unroll
            for (int j = 0; j < CPT; ++j) {
                const int m = msk[j];
                if (m < 0) continue;
                const int64_t i = slot[j];
#pragma unroll
                for (int q = 0; q < 6; ++q)
                    if (m & (1 << q)) X[i + off[q]] = own[j][q] + dl[j][q];
                X[i + off[6]] = own[j][6] + dl[j][6];
            }
            phase_sync<MODE>();
        }
}

template <int MODE, int CPT>
__global__ void __launch_bounds__(512) k_vanka_sym_coop(LevelK L, double* __restrict__ X,
                                                        const double* __restrict__ B, VankaLists vl,
                                                        const double* __restrict__ ktab, int nu) {
    __shared__ double Ks[64 * 49];
    for (int k = threadIdx.x; k < 64 * 49; k += blockDim.x) Ks[k] = ktab[k];
    __syncthreads();
    vanka_sweeps<MODE, CPT>(L, X, B, vl, Ks, nu, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

// Row residual of one Vanka block slot, gathered without divergence: lane s8 of
// the block's 8-lane group (0..5 the faces uL,uR,vL,vR,wL,wR; 6 the pressure)
// issues the same nine loads at lane-dependent offsets, then evaluates mom()
// (faces) or cont() (pressure) on them in exactly their operation order.  A
// per-lane switch would serialise seven dependent L2 round trips per phase.
// own = the slot's current value (the centre load).  Call only for s8 < 7 on
// a real block (every offset then stays inside the padded vector).
template <class AX>
__device__ __forceinline__ double vanka_slot_residual(const LevelK& L, AX X, const double* __restrict__ B,
                                                      int64_t i, int m, int s8, double& own) {
    const Geom& g = L.g;
    const int64_t fs = g.fs, sy = g.sy, sz = g.sz;
    const bool mom_row = s8 < 6;
    const int d = s8 >> 1;
    const int64_t st = d == 0 ? 1 : (d == 1 ? sy : sz);
    const int64_t jj = i + ((s8 & 1) ? st : 0);  // face slot (cell slot for the pressure row)
    const int64_t j = d * fs + jj;
    const int64_t p3 = 3 * fs;
    const int64_t o0 = mom_row ? j - 1 : i + 1, o1 = mom_row ? j + 1 : i;
    const int64_t o2 = mom_row ? j - sy : fs + i + sy, o3 = mom_row ? j + sy : fs + i;
    const int64_t o4 = mom_row ? j - sz : 2 * fs + i + sz, o5 = mom_row ? j + sz : 2 * fs + i;
    const int64_t o6 = mom_row ? j : p3 + i;
    const int64_t o7 = p3 + (mom_row ? jj : i), o8 = p3 + (mom_row ? jj - st : i);
    const double a0 = X[o0], a1 = X[o1], a2 = X[o2], a3 = X[o3], a4 = X[o4], a5 = X[o5], a6 = X[o6];
    const double a7 = X[o7], a8 = X[o8], bb = B[o6];
    own = a6;
    // mom(): eta/h^2 (6 F[j] - sum of the 6 neighbours x-,x+,y-,y+,z-,z+) + (P[j] - P[j - st]) / h
    double sm = a0 + a1;
    sm = sm + a2;
    sm = sm + a3;
    sm = sm + a4;
    sm = sm + a5;
    const double lap = 6.0 * a6 - sm;
    const double vm = L.eta_h2 * lap + (a7 - a8) * L.inv_h;
    // cont(): -((U[i+1]-U[i]) + (V[i+sy]-V[i]) + (W[i+sz]-W[i])) / h - gamma p
    const double div = (a0 - a1) + (a2 - a3) + (a4 - a5);
    const double vc = -div * L.inv_h - L.gamma * a6;
    const bool on = mom_row ? ((m >> s8) & 1) != 0 : true;
    return on ? bb - (mom_row ? vm : vc) : 0.0;
}

// Lane-parallel Vanka: 8 lanes per block; lane s < 7 computes residual slot s
// and owns DOF s; delta_s = sum_q K[s][q] r_q gathers r_q by warp shuffles in
// ascending q (same order as the oracle).  Each thread holds at most CPT
// (own, delta) pairs across the barrier.
template <int MODE, int CPT, class AX = double*>
__device__ __forceinline__ void vanka_sweeps8(const LevelK& L, AX X, const double* __restrict__ B,
                                              const VankaLists& vl, const double* __restrict__ Ks, int nu, int tid,
                                              int nth) {
    const Geom& g = L.g;
    const int64_t fs = g.fs, sy = g.sy, sz = g.sz;
    const int lane = threadIdx.x & 31, s8 = lane & 7;
    const int groups = nth >> 3, grp = tid >> 3;
    const int64_t offs = s8 == 0 ? 0 : s8 == 1 ? 1 : s8 == 2 ? fs : s8 == 3 ? fs + sy : s8 == 4 ? 2 * fs
                         : s8 == 5 ? 2 * fs + sz : 3 * fs;
    // this group's block of every colour, loaded once (slot << 7 | mask; -1 = none): removes a
    // dependent global load from every phase step
    constexpr bool kPre = CPT == 1;
    int64_t pre[8];
    if (kPre)
#pragma unroll
        for (int c = 0; c < 8; ++c)
            pre[c] = grp < vl.n[c] ? ((static_cast<int64_t>(vl.cells[c][grp]) << 7) | vl.masks[c][grp]) : -1;
    for (int sweep = 0; sweep < nu; ++sweep)
        for (int k = 0; k < 16; ++k) {
            const int col = vanka_phase_list(vl, k);
            if (col < 0) continue;
            const int n = vl.n[col];
            double own[CPT], dl[CPT];
            int64_t dst[CPT];
#pragma unroll
            for (int j = 0; j < CPT; ++j) {
                const int t = grp + j * groups;
                dst[j] = -1;
                // whole warps iterate together (shuffles); inactive groups use t = -1
                const bool act = t < n;
                int64_t i = 0;
                int m = 0;
                if (act) {
                    if (kPre) {
                        int64_t e = 0;
#pragma unroll
                        for (int c = 0; c < 8; ++c)
                            if (c == col) e = pre[c];
                        i = e >> 7;
                        m = static_cast<int>(e & 127);
                    } else {
                        i = vl.cells[col][t];
                        m = vl.masks[col][t];
                    }
                }
                double r = 0.0;
                if (act && s8 < 7) r = vanka_slot_residual(L, X, B, i, m, s8, own[j]);
                const double* K = Ks + m * 49 + (s8 < 7 ? s8 : 0) * 7;
                double acc = 0.0;
#pragma unroll
                for (int q = 0; q < 7; ++q) {
                    const double rq = __shfl_sync(0xffffffffu, r, (lane & ~7) + q);
                    acc = acc + K[q] * rq;
                }
                dl[j] = acc;
                if (act && s8 < 7 && (s8 == 6 || (m & (1 << s8)))) dst[j] = i + offs;
            }
            phase_sync<MODE>();
#pragma unroll
            for (int j = 0; j < CPT; ++j)
                if (dst[j] >= 0) X[dst[j]] = own[j] + dl[j];
            phase_sync<MODE>();
        }
}

// Ping-pong variant: one barrier per colour phase.  Phase k (k = 0..16 nu - 1)
// reads buffer X_k (XA for even k) and writes X_{k+1}: the new values of its
// colour's blocks and a copy of the blocks updated by phase k-1, so X_{k+1}
// holds the full state after phase k (it held the state after phase k-2, and
// only those two colours changed).  Reads and writes never share a buffer
// within a phase.  Before the sweep XB must equal XA on every DOF a Vanka
// residual reads (refresh list).  An even phase count: the result ends in XA.
// One ping-pong colour phase (list col; pcol = list of the previous phase, -1 if none):
// reads Xc, writes the phase's blocks and the carried previous-phase blocks into Xn.
// pre (CPT == 1, optional): this lane group's entry of every list, preloaded.
template <int CPT, bool PRE>
__device__ __forceinline__ void vanka_pp_phase(const LevelK& L, const double* __restrict__ Xc,
                                               double* __restrict__ Xn, const double* __restrict__ B,
                                               const VankaLists& vl, const double* __restrict__ Ks, int col, int pcol,
                                               const int64_t* pre, int tid, int nth) {
    const Geom& g = L.g;
    const int64_t fs = g.fs, sy = g.sy, sz = g.sz;
    const int lane = threadIdx.x & 31, s8 = lane & 7;
    const int groups = nth >> 3, grp = tid >> 3;
    const int64_t offs = s8 == 0 ? 0 : s8 == 1 ? 1 : s8 == 2 ? fs : s8 == 3 ? fs + sy : s8 == 4 ? 2 * fs
                         : s8 == 5 ? 2 * fs + sz : 3 * fs;
    // pre (PRE): CPT 1 -> pre[list]; CPT 2 (all four pairs merged, lists 0..3) -> pre[2 list + j]
    auto block_of = [&](int c, int j, int t, int64_t& i, int& m) {
        if constexpr (PRE) {
            int64_t e = 0;
#pragma unroll
            for (int q = 0; q < 8 / CPT; ++q)
                if (q == c) e = pre[q * CPT + j];
            i = e >> 7;
            m = static_cast<int>(e & 127);
        } else {
            i = vl.cells[c][t];
            m = vl.masks[c][t];
        }
    };
    const int cmask = vanka_list_cmask(vl, col);  // parity colours of this phase
    const int n = vl.n[col];
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
        const int t = grp + j * groups;
        const bool act = t < n;
        int64_t i = 0;
        int m = 0;
        if (act) block_of(col, j, t, i, m);
        double r = 0.0, own = 0.0;
        // the previous phase's block this lane carries into Xn (decided and loaded before the
        // gather, so its L2 round trip overlaps the residual loads): all its DOFs except those
        // this phase rewrites -- the same colour twice in a row (turning points), or a face
        // shared with a band cell of a colour of this phase (colours one parity bit apart)
        bool carry = false;
        int64_t cdst = 0;
        double cval = 0.0;
        if (pcol >= 0 && pcol != col && t < vl.n[pcol] && s8 < 7) {
            int64_t ip;
            int mp;
            block_of(pcol, j, t, ip, mp);
            carry = s8 == 6 || (mp & (1 << s8));
            if (carry && s8 < 6 && ((cmask >> (vanka_entry_colour(vl, pcol, t) ^ (1 << (s8 >> 1)))) & 1)) {
                const int zl = static_cast<int>(ip / sz) - g.zg;
                const int64_t rem = ip - static_cast<int64_t>(zl + g.zg) * sz;
                const int y = static_cast<int>(rem / sy) - 1;
                const int x = static_cast<int>(rem - static_cast<int64_t>(y + 1) * sy) - g.xo;
                const int d = (s8 & 1) ? 1 : -1;
                const int ax = s8 >> 1;
                if (band_cell(L, x + (ax == 0 ? d : 0), y + (ax == 1 ? d : 0), zl + (ax == 2 ? d : 0)))
                    carry = false;
            }
            if (carry) {
                cdst = ip + offs;
                cval = Xc[cdst];
            }
        }
        if (act && s8 < 7) r = vanka_slot_residual(L, Xc, B, i, m, s8, own);
#ifdef SMG_TRACE
        if (__any_sync(0xffffffffu, r == 1.2345e300)) g_trace[0] = 0;  // wait for the gather
#endif
        const double* K = Ks + m * 49 + (s8 < 7 ? s8 : 0) * 7;
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < 7; ++q) {
            const double rq = __shfl_sync(0xffffffffu, r, (lane & ~7) + q);
            acc = acc + K[q] * rq;
        }
        if (act && s8 < 7 && (s8 == 6 || (m & (1 << s8)))) Xn[i + offs] = own + acc;
        if (carry) Xn[cdst] = cval;
    }
}

// Ping-pong variant: one barrier per colour phase.  Phase k (k = 0..16 nu - 1)
// reads buffer X_k (XA for even k) and writes X_{k+1}: the new values of its
// colour's blocks and a copy of the blocks updated by phase k-1, so X_{k+1}
// holds the full state after phase k (it held the state after phase k-2, and
// only those two colours changed).  Reads and writes never share a buffer
// within a phase.  Before the sweep XB must equal XA on every DOF a Vanka
// residual reads (refresh list).  An even phase count: the result ends in XA.
template <int MODE, int CPT>
__device__ __forceinline__ void vanka_sweeps_pp(const LevelK& L, double* __restrict__ XA, double* __restrict__ XB,
                                                const double* __restrict__ B, const VankaLists& vl,
                                                const double* __restrict__ Ks, int nu, int tid, int nth) {
    const int grp = tid >> 3, groups = nth >> 3;
    // this lane group's block of every list, loaded once (slot << 7 | mask; -1 = none): CPT 1 for
    // all 8 lists, CPT 2 when the four merged pair lists are the only ones
    constexpr bool kPre = CPT == 1 || CPT == 2;
    const bool pre_ok = CPT == 1 || vl.pairs == 0xf;
    int64_t pre[8];
    if (kPre && pre_ok)
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int c = q / CPT, t = grp + (q % CPT) * groups;
            pre[q] = t < vl.n[c] ? ((static_cast<int64_t>(vl.cells[c][t]) << 7) | vl.masks[c][t]) : -1;
        }
    // executed phases alternate the buffers; an even count per sweep, so the result ends in XA
    int ph = 0, pcol = -1;
    for (int kk = 0; kk < 16 * nu; ++kk) {
        const int col = vanka_phase_list(vl, kk & 15);
        if (col < 0) continue;
        const double* __restrict__ Xc = (ph & 1) ? XB : XA;
        double* __restrict__ Xn = (ph & 1) ? XA : XB;
        SMG_TRACE_STAMP(ph, 0);
        if (kPre && pre_ok) vanka_pp_phase<CPT, kPre>(L, Xc, Xn, B, vl, Ks, col, pcol, pre, tid, nth);
        else vanka_pp_phase<CPT, false>(L, Xc, Xn, B, vl, Ks, col, pcol, pre, tid, nth);
        SMG_TRACE_STAMP(ph, 2);
        phase_sync<MODE>();
        SMG_TRACE_STAMP(ph, 3);
        pcol = col;
        ++ph;
    }
}

// ---- additive Vanka (Eq. S_AV) ----
// k_vadd_delta: every band block solves against the same x (8 lanes per block, the
// multiplicative sweep's slot residuals and shuffle-gathered local solve) and
// stores its correction by destination: D7 = [lo faces u, v, w at the block's own
// slot | hi faces u, v, w at the neighbour slot | p].  k_vadd_apply: each V1 DOF
// is written by one thread, x += omega * ((0.0 + corr of the lower block) + corr
// of the upper block), i.e. the oracle's ascending-cell summation order.
// M: labelled level (face diagonals from L.cls, signature class from kidx, "the neighbour has a block"
// from its DofMap bits instead of its distance to the wall).
template <bool M>
__device__ __forceinline__ double vanka_slot_residual_m(const LevelK& L, const double* __restrict__ X,
                                                        const double* __restrict__ B, int64_t i, int m, int s8);
template <bool M>
__global__ void __launch_bounds__(256) k_vadd_delta(LevelK L, const double* __restrict__ X,
                                                    const double* __restrict__ B, const int32_t* __restrict__ cells,
                                                    const uint8_t* __restrict__ masks,
                                                    const uint16_t* __restrict__ kidx, int n,
                                                    const double* __restrict__ ktab, double* __restrict__ D7) {
    pdl_wait();
    const Geom& g = L.g;
    const int64_t fs = g.fs;
    const int lane = threadIdx.x & 31, s8 = lane & 7;
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 3;
    const bool act = t < n;
    int64_t i = 0;
    int m = 0, ki = 0;
    if (act) {
        i = cells[t];
        m = masks[t];
        ki = M ? kidx[t] : m;
    }
    double r = 0.0, own = 0.0;
    if (act && s8 < 7) r = M ? vanka_slot_residual_m<true>(L, X, B, i, m, s8) : vanka_slot_residual(L, X, B, i, m, s8, own);
    const double* K = ktab + static_cast<int64_t>(ki) * 49 + (s8 < 7 ? s8 : 0) * 7;
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < 7; ++q) {
        const double rq = __shfl_sync(0xffffffffu, r, (lane & ~7) + q);
        acc = acc + __ldg(K + q) * rq;
    }
    if (!act || s8 >= 7 || !(s8 == 6 || (m & (1 << s8)))) return;
    if (s8 == 6) {
        D7[6 * fs + i] = acc;
    } else {
        const int ax = s8 >> 1;
        const int64_t st = ax == 0 ? 1 : (ax == 1 ? g.sy : g.sz);
        if (s8 & 1) D7[(3 + ax) * fs + i + st] = acc;
        else D7[ax * fs + i] = acc;
    }
}

template <bool M>
__global__ void __launch_bounds__(256) k_vadd_apply(LevelK L, double* __restrict__ X,
                                                    const int32_t* __restrict__ cells,
                                                    const uint8_t* __restrict__ masks, int n,
                                                    const double* __restrict__ D7, double omega) {
    pdl_wait();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const Geom& g = L.g;
    const int64_t fs = g.fs, i = cells[t];
    const int m = masks[t];
    const int zl = static_cast<int>(i / g.sz) - g.zg;
    const int64_t rem = i - static_cast<int64_t>(zl + g.zg) * g.sz;
    const int y = static_cast<int>(rem / g.sy) - 1;
    const int x = static_cast<int>(rem - static_cast<int64_t>(y + 1) * g.sy) - g.xo;
    X[3 * fs + i] = X[3 * fs + i] + omega * (0.0 + D7[6 * fs + i]);
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        const int64_t st = ax == 0 ? 1 : (ax == 1 ? g.sy : g.sz);
        const int dx = ax == 0, dy = ax == 1, dz = ax == 2;
        if (m & (1 << (2 * ax))) {  // low face: the lower cell's block (if band) first, then this one
            double acc = 0.0;
            const bool lower_block = M ? (L.cls[i - st] & (CLS_P | CLS_BAND)) == (CLS_P | CLS_BAND)
                                       : band_cell(L, x - dx, y - dy, zl - dz);
            if (lower_block) acc = acc + D7[(3 + ax) * fs + i];
            acc = acc + D7[ax * fs + i];
            X[ax * fs + i] = X[ax * fs + i] + omega * acc;
        }
        const bool upper_block = M ? (L.cls[i + st] & (CLS_P | CLS_BAND)) == (CLS_P | CLS_BAND)
                                   : band_cell(L, x + dx, y + dy, zl + dz);
        if ((m & (1 << (2 * ax + 1))) && !upper_block) {  // high face, this block only
            X[ax * fs + i + st] = X[ax * fs + i + st] + omega * (0.0 + D7[(3 + ax) * fs + i + st]);
        }
    }
}

// One ping-pong phase per launch (graph nodes instead of grid barriers); the
// local inverses are read through L1 (26 masks occur in a box).
template <int CPT>
__global__ void __launch_bounds__(256) k_vanka_ppk(LevelK L, const double* __restrict__ Xc, double* __restrict__ Xn,
                                                   const double* __restrict__ B, VankaLists vl,
                                                   const double* __restrict__ ktab, int col, int pcol) {
    pdl_wait();
    vanka_pp_phase<CPT, false>(L, Xc, Xn, B, vl, ktab, col, pcol, nullptr, blockIdx.x * blockDim.x + threadIdx.x,
                               gridDim.x * blockDim.x);
}

// SMG_VKPP_THREADS / SMG_VKPP_MINB (build-time A/B): launch bounds of the persistent ping-pong
// sweep.  Its occupancy matters (build A/Bs on one box, cfg 1 solve): 74 -> 94 registers
// (3 -> 2 CTAs/SM) cost 19.43 vs 18.63 ms; (256, 4) = 64 registers, 4 CTAs/SM: 19.12 -> 18.87 ms.
// (A 512-thread cooperative CTA, SMG_COOP_THREADS=512, then finds no occupancy and takes the
// next sweep variant.)
#ifndef SMG_VKPP_THREADS
#define SMG_VKPP_THREADS 256
#endif
#ifndef SMG_VKPP_MINB
#define SMG_VKPP_MINB 4
#endif
template <int MODE, int CPT>
__global__ void __launch_bounds__(SMG_VKPP_THREADS, SMG_VKPP_MINB) k_vanka_pp(LevelK L, double* __restrict__ XA, double* __restrict__ XB,
                                                  const double* __restrict__ B, VankaLists vl,
                                                  const double* __restrict__ ktab, int nu,
                                                  const int32_t* __restrict__ refresh, int64_t nrefresh) {
    __shared__ double Ks[64 * 49];
    for (int k = threadIdx.x; k < 64 * 49; k += blockDim.x) Ks[k] = ktab[k];
    // XB = XA on the read set minus the first phase's DOFs, concurrently with the first phase
    // (which reads only XA and writes only its own DOFs of XB); the first barrier orders both.
    // Replaces a k_refresh launch per sweep (SMG_VANKA_REFRESH_IN=0 restores it): cfg 1 solve
    // 18.75 -> 18.69 ms and 18.76 -> 18.69 ms on two boxes (fine sweep 0.075 -> 0.073 ms).
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < nrefresh;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t k = refresh[t];
        XB[k] = XA[k];
    }
    __syncthreads();
    vanka_sweeps_pp<MODE, CPT>(L, XA, XB, B, vl, Ks, nu, blockIdx.x * blockDim.x + threadIdx.x,
                               gridDim.x * blockDim.x);
}

__global__ void k_refresh(const int32_t* __restrict__ lst, int64_t n, const double* __restrict__ src,
                          double* __restrict__ dst) {
    pdl_wait();
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = lst[t];
        dst[k] = src[k];
    }
}

template <int MODE, int CPT>
__global__ void __launch_bounds__(512) k_vanka8(LevelK L, double* __restrict__ X, const double* __restrict__ B,
                                                VankaLists vl, const double* __restrict__ ktab, int nu) {
    __shared__ double Ks[64 * 49];
    for (int k = threadIdx.x; k < 64 * 49; k += blockDim.x) Ks[k] = ktab[k];
    __syncthreads();
    vanka_sweeps8<MODE, CPT>(L, X, B, vl, Ks, nu, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

// Cell updates below load everything a cell needs before their first store:
// X, D and the faces of one cell are reached through one pointer, so a store
// would otherwise order every later load behind it (one L2 round trip each).
// Same additions in the same order as the plain forms, hence bit-identical.
// A velocity-phase cell update split into its loads and its stores, so a thread
// holding several cells issues all their loads first (cells of one phase never
// read each other's writes).
struct VelUpd {
    int64_t i;
    double u0, v0, w0, ru, rv, rw;
    bool du, dv, dw;
};
template <class AX>
__device__ __forceinline__ VelUpd vel_load(const LevelK& L, AX X, const double* __restrict__ B, int x, int y, int z,
                                           bool valid) {
    const Geom& g = L.g;
    const int64_t fs = g.fs;
    VelUpd u;
    u.i = valid ? g.slot(x, y, z) : 0;
    const int64_t i = u.i;
    const auto U = X, V = X + fs, W = X + 2 * fs, P = X + 3 * fs;
    const bool here = !valid || band_cell(L, x, y, z);
    u.du = x >= 1 && !here && !band_cell(L, x - 1, y, z);
    u.dv = y >= 1 && !here && !band_cell(L, x, y - 1, z);
    u.dw = g.gz(z) >= 1 && !here && !band_cell(L, x, y, z - 1);
    u.ru = u.rv = u.rw = u.u0 = u.v0 = u.w0 = 0.0;
    if (u.du) { u.u0 = U[i]; u.ru = B[i] - mom(L, U, P, i, 1); }
    if (u.dv) { u.v0 = V[i]; u.rv = B[fs + i] - mom(L, V, P, i, g.sy); }
    if (u.dw) { u.w0 = W[i]; u.rw = B[2 * fs + i] - mom(L, W, P, i, g.sz); }
    return u;
}
template <class AX>
__device__ __forceinline__ void vel_store(const LevelK& L, AX X, const VelUpd& u) {
    const int64_t fs = L.g.fs;
    if (u.du) X[u.i] = u.u0 + u.ru / L.dv;
    if (u.dv) X[fs + u.i] = u.v0 + u.rv / L.dv;
    if (u.dw) X[2 * fs + u.i] = u.w0 + u.rw / L.dv;
}
template <class AX>
__device__ __forceinline__ void dgs_vel_cell(const LevelK& L, AX X, const double* __restrict__ B, int x, int y, int z) {
    vel_store(L, X, vel_load(L, X, B, x, y, z, true));
}

// Reverse (left-preconditioned) pressure update of the cell at slot i: the new p_i =
// p_i + (c_b - m_i^T L~x) / d_p, with c_b = m_i^T b from L.cb (k_dgs_cb) and the
// L~x part in the same operation order.  Reads only x around the cell (radius 2).
template <class AX>
__device__ __forceinline__ double prev_core(const LevelK& L, AX X, int64_t i, double cbv);
template <class AX>
__device__ __forceinline__ double prev_value(const LevelK& L, AX X, int64_t i) {
    return prev_core(L, X, i, L.cb[i]);
}
template <class AX>
__device__ __forceinline__ double prev_core(const LevelK& L, AX X, int64_t i, double cbv) {
    const Geom& g = L.g;
    const int64_t fs = g.fs, sy = g.sy, sz = g.sz;
    const auto U = X, V = X + fs, W = X + 2 * fs, P = X + 3 * fs;
    const double luL = mom(L, U, P, i, 1);
    const double luR = mom(L, U, P, i + 1, 1);
    const double lvL = mom(L, V, P, i, sy);
    const double lvR = mom(L, V, P, i + sy, sy);
    const double lwL = mom(L, W, P, i, sz);
    const double lwR = mom(L, W, P, i + sz, sz);
    const double fl = ((luR - luL) + (lvR - lvL)) + (lwR - lwL);
    const double lc = cont(L, U, V, W, P, i, L.gamma);
    double s = cont(L, U, V, W, P, i - 1, L.gamma) + cont(L, U, V, W, P, i + 1, L.gamma);
    s = s + cont(L, U, V, W, P, i - sy, L.gamma);
    s = s + cont(L, U, V, W, P, i + sy, L.gamma);
    s = s + cont(L, U, V, W, P, i - sz, L.gamma);
    s = s + cont(L, U, V, W, P, i + sz, L.gamma);
    const double cl = fl * L.inv_h + L.eta_h2 * (6.0 * lc - s);
    return P[i] + (cbv - cl) / L.dp;
}
template <class AX>
__device__ __forceinline__ void dgs_prev_cell(const LevelK& L, AX X, const double* __restrict__ B, int64_t i) {
    (void)B;
    X[3 * L.g.fs + i] = prev_value(L, X, i);
}

// ---- lazy-gather forward pressure phases (single-part levels) ----
// Eager form: after phase c every cell K gets p_K += eta/h^2 (6 D_c[K] - sum_nbr D_c),
// which is a no-op unless colour(K) == c (self term) or colour(K) == c ^ bit
// (gather from the colour-c neighbours along one axis).  p_K is only read by
// K's own phase (its continuity residual) before the pressure sweep ends, so
// the gathers are applied when K is next read: those from phases c' < colour(K)
// at the start of K's phase, the others in a flush after phase 7 — the same
// additions in the same order, hence bit-identical.  One combined delta buffer
// holds delta_c at the V2 cells of colour c (band cells stay 0); a gather from
// phase c' masks the neighbour sum to colour-c' cells.
// The six delta neighbours of a cell (x-, x+, y-, y+, z-, z+), loaded once.
struct Nbr6 {
    double v[6];
};
template <class AD>
__device__ __forceinline__ Nbr6 load_nbr6(const Geom& g, AD D, int64_t i) {
    return Nbr6{{D[i - 1], D[i + 1], D[i - g.sy], D[i + g.sy], D[i - g.sz], D[i + g.sz]}};
}
__device__ __forceinline__ double masked_nbr_sum(const Nbr6& d, int x, int y, int zg, int cc) {
    // neighbour colours: x +-1 flips bit 1, y +-1 bit 2, z +-1 bit 4 of colour (x,y,zg)
    const int ck = (x & 1) + 2 * (y & 1) + 4 * (zg & 1);
    const bool mx = (ck ^ 1) == cc, my = (ck ^ 2) == cc, mz = (ck ^ 4) == cc;
    double s = (mx ? d.v[0] : 0.0) + (mx ? d.v[1] : 0.0);
    s = s + (my ? d.v[2] : 0.0);
    s = s + (my ? d.v[3] : 0.0);
    s = s + (mz ? d.v[4] : 0.0);
    s = s + (mz ? d.v[5] : 0.0);
    return s;
}

// p_K after the pending gathers (earlier colours if !later, the others if later).
__device__ __forceinline__ double apply_gathers(const LevelK& L, double p, const Nbr6& d, int x, int y, int zg,
                                                bool later) {
    const int k = (x & 1) + 2 * (y & 1) + 4 * (zg & 1);
    const int c1 = k ^ 1, c2 = k ^ 2, c4 = k ^ 4;  // ascending order among the three
    int cs[3] = {c1, c2, c4};
    if (cs[0] > cs[1]) { const int t = cs[0]; cs[0] = cs[1]; cs[1] = t; }
    if (cs[1] > cs[2]) { const int t = cs[1]; cs[1] = cs[2]; cs[2] = t; }
    if (cs[0] > cs[1]) { const int t = cs[0]; cs[0] = cs[1]; cs[1] = t; }
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const int cc = cs[q];
        if ((cc < k) == later) continue;
        const double sn = masked_nbr_sum(d, x, y, zg, cc);
        p = p + L.eta_h2 * (6.0 * 0.0 - sn);
    }
    return p;
}

// Split load / store forms of the lazy forward-pressure cell update and of
// the flush (same reasoning as VelUpd).
struct PfUpd {
    Nbr6 d;
    int64_t ii;
    double p0, uL, uR, vL, vR, wL, wR, bp;
    int x, y, zg;
    bool valid, band;
};
template <class AX, class AD>
__device__ __forceinline__ PfUpd pf_load(const LevelK& L, AX X, const double* __restrict__ B, AD D, int x, int y,
                                         int z, bool valid, bool flush) {
    const Geom& g = L.g;
    const int64_t fs = g.fs, sy = g.sy, sz = g.sz;
    PfUpd u;
    u.valid = valid;
    u.x = x;
    u.y = y;
    u.zg = g.gz(z);
    u.ii = valid ? g.slot(x, y, z) : 0;
    const int64_t ii = u.ii;
    u.band = flush || !valid || band_cell(L, x, y, z);
    u.uL = u.uR = u.vL = u.vR = u.wL = u.wR = u.bp = 0.0;
    u.p0 = 0.0;
    u.d = Nbr6{{0.0, 0.0, 0.0, 0.0, 0.0, 0.0}};
    if (valid) {
        u.d = load_nbr6(g, D, ii);
        u.p0 = X[3 * fs + ii];
    }
    if (!u.band) {
        u.uL = X[ii];
        u.uR = X[ii + 1];
        u.vL = X[fs + ii];
        u.vR = X[fs + ii + sy];
        u.wL = X[2 * fs + ii];
        u.wR = X[2 * fs + ii + sz];
        u.bp = B[3 * fs + ii];
    }
    return u;
}
template <bool FLUSH, class AX, class AD>
__device__ __forceinline__ void pf_store(const LevelK& L, AX X, AD D, const PfUpd& u) {
    if (!u.valid) return;
    const int64_t fs = L.g.fs, sy = L.g.sy, sz = L.g.sz, ii = u.ii;
    const double p = apply_gathers(L, u.p0, u.d, u.x, u.y, u.zg, FLUSH);
    if (FLUSH || u.band) {
        X[3 * fs + ii] = p;
        return;
    }
    if constexpr (!FLUSH) {
    // cont(): -((uR-uL) + (vR-vL) + (wR-wL)) / h - gamma p
    const double div = (u.uR - u.uL) + (u.vR - u.vL) + (u.wR - u.wL);
    const double rr = u.bp - (-div * L.inv_h - L.gamma * p);
    const double dc = rr / L.dp;
    D[ii] = dc;
    X[ii] = u.uL + (0.0 - dc) * L.inv_h;
    X[ii + 1] = u.uR + (dc - 0.0) * L.inv_h;
    X[fs + ii] = u.vL + (0.0 - dc) * L.inv_h;
    X[fs + ii + sy] = u.vR + (dc - 0.0) * L.inv_h;
    X[2 * fs + ii] = u.wL + (0.0 - dc) * L.inv_h;
    X[2 * fs + ii + sz] = u.wR + (dc - 0.0) * L.inv_h;
    // self term: the colour-c neighbour sum is a sum of six zeros
    double sn = 0.0 + 0.0;
    sn = sn + 0.0;
    sn = sn + 0.0;
    sn = sn + 0.0;
    sn = sn + 0.0;
    X[3 * fs + ii] = p + L.eta_h2 * (6.0 * dc - sn);
    }
}

// flush after phase 7: the gathers from the later colours (cell p only)
template <class AX, class AD>
__device__ __forceinline__ void flush_gathers(const LevelK& L, AX X, AD D, int x, int y, int z) {
    pf_store<true>(L, X, D, pf_load(L, X, nullptr, D, x, y, z, true, true));
}

template <class AX, class AD>
__device__ __forceinline__ void pf_lazy_cell(const LevelK& L, AX X, const double* __restrict__ B, AD D, int x, int y,
                                             int z) {
    pf_store<false>(L, X, D, pf_load(L, X, B, D, x, y, z, true, false));
}

// Colour groups of the 8-colour pressure phases.  A pressure phase of colour c
// reads what phase c' wrote only if c ^ c' is a single bit (axis neighbours
// share faces / pressures; diagonal neighbours share nothing), so colours of
// equal popcount commute and each popcount class runs as ONE step: forward
// 0 | 1,2,4 | 3,5,6 | 7, reverse 7 | 6,5,3 | 4,2,1 | 0.  Every dependent pair
// keeps its order, so results are bit-identical to the 8-step sequence.
// Packed as 3 bits per colour, count in bits 9..10.
__host__ __device__ constexpr int colour_group(int c0, int c1, int c2, int n) {
    return c0 | (c1 << 3) | (c2 << 6) | (n << 9);
}
__host__ __device__ constexpr int group_size(int grp) { return grp >> 9; }
__host__ __device__ constexpr int group_colour(int grp, int k) { return (grp >> (3 * k)) & 7; }
__host__ __device__ constexpr int fwd_group(int q) {
    return q == 0 ? colour_group(0, 0, 0, 1)
                  : q == 1 ? colour_group(1, 2, 4, 3) : q == 2 ? colour_group(3, 5, 6, 3) : colour_group(7, 0, 0, 1);
}
__host__ __device__ constexpr int rev_group(int q) {
    return q == 0 ? colour_group(7, 0, 0, 1)
                  : q == 1 ? colour_group(6, 5, 3, 3) : q == 2 ? colour_group(4, 2, 1, 3) : colour_group(0, 0, 0, 1);
}


// -------------------------------------- colour-compact per-phase DGS kernels ------
// For large levels: one kernel per phase (graph-captured; a kernel boundary is
// cheaper than a grid barrier), threads mapped onto the cells of the phase's
// colour only, so every thread works and only the needed rows are touched.
// Per-cell arithmetic is shared with the kernels above (bit-identical).
// Block coordinates, traversed in reverse order when rev (bit 16 of the step argument):
// consecutive steps alternate direction, so a step starts on the planes the previous
// one touched last, while they are still in L2.
struct BlkIdx {
    int x, y, z;
};
__device__ __forceinline__ BlkIdx blk_idx(bool rev) {
    if (!rev) return BlkIdx{static_cast<int>(blockIdx.x), static_cast<int>(blockIdx.y), static_cast<int>(blockIdx.z)};
    return BlkIdx{static_cast<int>(gridDim.x - 1 - blockIdx.x), static_cast<int>(gridDim.y - 1 - blockIdx.y),
                  static_cast<int>(gridDim.z - 1 - blockIdx.z)};
}
constexpr int kRevBit = 1 << 16;


// ZC independent cells per thread (planes z, z + gridDim.z, ...): more loads in flight
template <int ZC>
__global__ void __launch_bounds__(256) k_dgs_vel_c(LevelK L, double* __restrict__ X, const double* __restrict__ B,
                                                   int colour) {
    pdl_wait();
    const Geom& g = L.g;
    const BlkIdx bk = blk_idx(colour & kRevBit);
    colour &= 1;
    const int i = bk.x * 32 + threadIdx.x, y = bk.y * 8 + threadIdx.y;
#pragma unroll
    for (int q = 0; q < ZC; ++q) {
        const int z = bk.z + q * gridDim.z;
        const int x = 2 * i + ((y + g.gz(z) + colour) & 1);
        if (x < g.nx && y < g.ny && z < g.nz) dgs_vel_cell(L, X, B, x, y, z);
    }
}



__device__ __forceinline__ bool half_cell(const Geom& g, int c, int i, int j, int k, int& x, int& y, int& z) {
    x = 2 * i + (c & 1);
    y = 2 * j + ((c >> 1) & 1);
    z = 2 * k + (((c >> 2) ^ g.z0) & 1);  // local plane with global parity (c >> 2)
    return x < g.nx && y < g.ny && z < g.nz;
}

__global__ void __launch_bounds__(256) k_dgs_pf_delta_c(LevelK L, const double* __restrict__ X,
                                                        const double* __restrict__ B, double* __restrict__ D,
                                                        int c) {
    const Geom& g = L.g;
    const int i = blockIdx.x * 32 + threadIdx.x, j = blockIdx.y * 8 + threadIdx.y, k = blockIdx.z;
    int x, y, z;
    if (half_cell(g, (c + 6) & 7, i, j, k, x, y, z)) D[g.slot(x, y, z)] = 0.0;  // stale colour c-2
    if (!half_cell(g, c, i, j, k, x, y, z) || band_cell(L, x, y, z)) return;
    const int64_t fs = g.fs, ii = g.slot(x, y, z);
    const double rr = B[3 * fs + ii] - cont(L, X, X + fs, X + 2 * fs, X + 3 * fs, ii, L.gamma);
    D[ii] = rr / L.dp;
}

__device__ __forceinline__ void p_gather_update(const LevelK& L, double* __restrict__ X, const double* __restrict__ D,
                                                int64_t i) {
    const Geom& g = L.g;
    const int64_t fs = g.fs, sy = g.sy, sz = g.sz;
    double sn = D[i - 1] + D[i + 1];
    sn = sn + D[i - sy];
    sn = sn + D[i + sy];
    sn = sn + D[i - sz];
    sn = sn + D[i + sz];
    X[3 * fs + i] = X[3 * fs + i] + L.eta_h2 * (6.0 * D[i] - sn);
}

__global__ void __launch_bounds__(256) k_dgs_pf_apply_c(LevelK L, double* __restrict__ X, const double* __restrict__ D,
                                                        int c) {
    const Geom& g = L.g;
    const int i = blockIdx.x * 32 + threadIdx.x, j = blockIdx.y * 8 + threadIdx.y, k = blockIdx.z;
    const int64_t fs = g.fs, sy = g.sy, sz = g.sz;
    int x, y, z;
    if (half_cell(g, c, i, j, k, x, y, z) && !band_cell(L, x, y, z)) {
        const int64_t ii = g.slot(x, y, z);
        const double dc = D[ii];
        X[ii] = X[ii] + (0.0 - dc) * L.inv_h;
        X[ii + 1] = X[ii + 1] + (dc - 0.0) * L.inv_h;
        X[fs + ii] = X[fs + ii] + (0.0 - dc) * L.inv_h;
        X[fs + ii + sy] = X[fs + ii + sy] + (dc - 0.0) * L.inv_h;
        X[2 * fs + ii] = X[2 * fs + ii] + (0.0 - dc) * L.inv_h;
        // the top w face of a slab's top plane belongs to the next part (applied there, below)
        if (z + 1 < g.nz) X[2 * fs + ii + sz] = X[2 * fs + ii + sz] + (dc - 0.0) * L.inv_h;
        p_gather_update(L, X, D, ii);
    }
#pragma unroll
    for (int bit = 1; bit < 8; bit <<= 1)
        if (half_cell(g, c ^ bit, i, j, k, x, y, z)) p_gather_update(L, X, D, g.slot(x, y, z));
    // z-slab: colour-c cell in the halo plane below -> its top w face is this part's plane 0
    if (k == 0 && g.z0 > 0 && ((g.z0 - 1) & 1) == ((c >> 2) & 1)) {
        x = 2 * i + (c & 1);
        y = 2 * j + ((c >> 1) & 1);
        if (x < g.nx && y < g.ny && !band_cell(L, x, y, -1)) {
            const int64_t ih = g.slot(x, y, -1);
            X[2 * fs + ih + sz] = X[2 * fs + ih + sz] + (D[ih] - 0.0) * L.inv_h;
        }
    }
}

template <int ZC>
// grid.z = (z blocks) x (colours of the group), colour fastest so the group's
// colours of one plane pair run side by side
__global__ void __launch_bounds__(256) k_dgs_pf_lazy_c(LevelK L, double* __restrict__ X, const double* __restrict__ B,
                                                       double* __restrict__ D, int grp) {
    pdl_wait();
    const Geom& g = L.g;
    const BlkIdx bk = blk_idx(grp & kRevBit);
    grp &= kRevBit - 1;
    const int i = bk.x * 32 + threadIdx.x, j = bk.y * 8 + threadIdx.y;
    const int nc = group_size(grp), c = group_colour(grp, bk.z % nc);
    const int kz = bk.z / nc, nkz = gridDim.z / nc;
#pragma unroll
    for (int q = 0; q < ZC; ++q) {
        int x, y, z;
        if (half_cell(g, c, i, j, kz + q * nkz, x, y, z)) pf_lazy_cell(L, X, B, D, x, y, z);
    }
}

__global__ void __launch_bounds__(256) k_dgs_pf_flush(LevelK L, double* __restrict__ X, const double* __restrict__ D,
                                                      int rev) {
    pdl_wait();
    const BlkIdx bk = blk_idx(rev);
    const int x = bk.x * BX + threadIdx.x, y = bk.y * BY + threadIdx.y;
    if (x >= L.g.nx || y >= L.g.ny) return;
    flush_gathers(L, X, D, x, y, bk.z);
}

template <int ZC>
// build-time A/B: CTAs per SM the register allocation of k_dgs_prev_c targets.  The free allocation
// (104 registers, 2 CTAs/SM) measured best: 3 (80 registers, no spill) cfg 3 fine DGS sweep
// 20.74 -> 20.88 ms, 4 (64 registers, spills) 20.78 -> 21.44 ms (profiles/r1s5_prev_minb_ab.txt)
#ifndef SMG_PREV_MINB
#define SMG_PREV_MINB 1
#endif
__global__ void __launch_bounds__(256, SMG_PREV_MINB) k_dgs_prev_c(LevelK L, double* __restrict__ X, const double* __restrict__ B,
                                                    int grp) {
    pdl_wait();
    const Geom& g = L.g;
    const BlkIdx bk = blk_idx(grp & kRevBit);
    grp &= kRevBit - 1;
    const int i = bk.x * 32 + threadIdx.x, j = bk.y * 8 + threadIdx.y;
    const int nc = group_size(grp), c = group_colour(grp, bk.z % nc);
    const int kz = bk.z / nc, nkz = gridDim.z / nc;
#pragma unroll
    for (int q = 0; q < ZC; ++q) {
        int x, y, z;
        if (half_cell(g, c, i, j, kz + q * nkz, x, y, z) && !band_cell(L, x, y, z))
            dgs_prev_cell(L, X, B, g.slot(x, y, z));
    }
}


// ------------------------------------------------ SQMR device scalars ------
// Alg. 4 scalar recurrences evaluated on the device (same expressions and
// order as the oracle), so one SQMR iteration is a fixed kernel sequence that
// can be replayed as a CUDA graph.  sc[] layout: see SqmrSlot in smg_internal.h.

__device__ __forceinline__ void sqmr_alpha_from(double* sc, double sigma) {  // after sigma = q.t
    if (sc[S_STATUS] != 0.0) return;
    if (fabs(sigma) < 1e-300) { sc[S_STATUS] = 2.0; return; }
    sc[S_ALPHA] = sc[S_RHO] / sigma;
}
__device__ __forceinline__ void sqmr_alpha(double* sc) { sqmr_alpha_from(sc, sc[S_D0]); }



__device__ __forceinline__ void sqmr_beta(double* sc) {  // after ||b - L x||^2
    if (sc[S_STATUS] != 0.0) return;
    const double rel = sqrt(sc[S_D0]) / sc[S_BNORM];
    sc[S_REL] = rel;
    if (rel < sc[S_TOL]) { sc[S_STATUS] = 1.0; return; }  // converged
    const double rho_new = sc[S_RHONEW];
    if (fabs(rho_new) < 1e-300) { sc[S_STATUS] = 3.0; return; }
    sc[S_BETA] = rho_new / sc[S_RHO];
    sc[S_RHO] = rho_new;
    sc[S_NUOLD] = sc[S_NU];
}

// final combination of the block partials into sc[S_D0], sc[S_D1], then the Alg. 4 scalar update
// `which` (0 first: tau, rho; 1 alpha; 2 nu, c, tau, cd, cq; 3 rel, convergence, beta; -1 none)
__device__ __forceinline__ void sqmr_first(double* sc) {
    sc[S_TAU] = sqrt(sc[S_D0]);
    sc[S_NUOLD] = 0.0;
    sc[S_RHO] = sc[S_D1];
    sc[S_STATUS] = fabs(sc[S_RHO]) < 1e-300 ? 2.0 : 0.0;
}
__device__ __forceinline__ void sqmr_nu(double* sc) {
    if (sc[S_STATUS] != 0.0) return;
    const double nu = sqrt(sc[S_D0]) / sc[S_TAU];
    const double c = 1.0 / sqrt(1.0 + nu * nu);
    sc[S_TAU] = sc[S_TAU] * nu * c;
    const double c2 = c * c;
    sc[S_CD] = c2 * (sc[S_NUOLD] * sc[S_NUOLD]);
    sc[S_CQ] = c2 * sc[S_ALPHA];
    sc[S_NU] = nu;
    sc[S_RHONEW] = sc[S_D1];
    // beta_j = rho_j / rho_{j-1} already here: the q update of the next iteration runs before the
    // residual's final (sqmr_beta repeats the same division when it commits rho)
    sc[S_BETA] = sc[S_D1] / sc[S_RHO];
}
__global__ void __launch_bounds__(256) k_final_scalar(const double* __restrict__ partials, int64_t nblk,
                                                      double* __restrict__ sc, int which) {
    pdl_wait();
    if (which > 0 && sc[S_STATUS] != 0.0) return;
    final2(partials, nblk, sc + S_D0);
    if (threadIdx.x != 0) return;
    if (which == 0) sqmr_first(sc);
    else if (which == 1) sqmr_alpha(sc);
    else if (which == 2) sqmr_nu(sc);
    else if (which == 3) sqmr_beta(sc);
    else if (which == 4) {  // ||r_j||^2 in the first slot, sigma_{j+1} in the second: one reduction for both
        sqmr_beta(sc);
        sqmr_alpha_from(sc, sc[S_D1]);
    }
}

__global__ void k_axpy_s(double* __restrict__ s, const double* __restrict__ t, const double* __restrict__ sc,
                         int64_t n) {  // s = s - alpha t
    pdl_wait();
    if (sc[S_STATUS] != 0.0) return;
    const double a = sc[S_ALPHA];
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        s[k] = s[k] - a * t[k];
}

// ------------------------------------------- tile-ordered DGS (large levels) ------
// OD-1 rev. 2: a large level is cut into tiles of kTX x kTY x kTZ cells,
// coloured by tile parity T = (tx&1) + 2(ty&1) + 4(tz&1).  The symmetric sweep relaxes
// the tiles of colour 0..7 in turn (forward phases 0..9 inside each tile), then 7..0
// (reverse phases 10..19 inside each tile): "a given traversal order, then exactly the
// reverse", so the sweep stays symmetric.  Same-colour tiles are a whole
// tile apart, farther than any read (radius 2) plus write (radius 1) reach, so they run
// in parallel exactly as in sequence.  One CTA owns one tile: the tile's neighbourhood of x
// (all four fields), its b and (reverse half) its m^T b are staged in shared memory, every
// phase runs there with __syncthreads between phases, and only the DOFs a phase may change go
// back to HBM.  Per-point arithmetic is the per-step kernels' (same operand order) and the
// in-tile order is the oracle's: bit-identical.  A level vector is read once and written once
// per half sweep (plus the halo) instead of 13 passes of the per-step kernels.
//
// Shared-memory layout: every box row keeps its even-x and odd-x cells in two half-rows
// ("x-parity split"): a phase works on one parity class of cells at a time, so the 32 lanes of
// a warp read 8 consecutive words of 4 rows two apart (row stride 20 words: the two 8-word
// groups of a half-warp fall on disjoint banks) -- no bank conflicts, where the natural layout
// served stride-2 accesses in twice the wavefronts.  The x neighbours of a cell sit in the
// other half-row (offsets XM / XP, by the cell's x parity).  The box is filled by coalesced
// 128-bit loads (one even/odd pair each); m^T b, read once per cell, is staged by TMA.
//
// Two variants keep two CTAs per SM: FWD (phases 0..9; x box x [-2, TX+2), y, z [-1, T+1),
// the tile's b, pressure deltas on the tile + a zero ring) and REV (phases 10..19; x box y, z
// [-1, T+2) for the radius-2 reads of the reverse pressure update; b of u, v, w; m^T b).
constexpr int kTX = 16, kTY = 8, kTZ = 8;
constexpr int kTileThreads = 256;
constexpr int kTileCells = kTX * kTY * kTZ;
constexpr int kBX = kTX + 4, kHX = kBX / 2;  // box row (x from -2) and half-row
template <bool FWD>
struct TileBox {
    static constexpr int BY = FWD ? kTY + 2 : kTY + 3, BZ = FWD ? kTZ + 2 : kTZ + 3;
    static constexpr int SY = kBX, SZ = kBX * BY, BOX = kBX * BY * BZ;
    static constexpr int NB = FWD ? 4 : 3;  // fields of b staged
    // FWD: deltas on the tile plus a ring of zeros (natural layout, (T+2)^3); REV: m^T b of the
    // tile (natural, TMA) + the (lc, s) exchange of the split reverse update
    static constexpr int TS = FWD ? (kTX + 2) * (kTY + 2) * (kTZ + 2) : kTileCells + kTileCells / 4;
    static constexpr size_t SMEM = (4 * BOX + NB * kTileCells + TS) * sizeof(double) + 128 + 16;
    // cell (x, y, z) of the tile (x in [-2, TX + 2), y, z from -1) in the split box
    static __device__ __forceinline__ int li(int x, int y, int z) {
        return ((z + 1) * BY + (y + 1)) * kBX + (x & 1) * kHX + ((x + 2) >> 1);
    }
};
// x neighbours in the split layout of a cell of x parity p
__device__ __forceinline__ int xp_off(int p) { return p ? -kHX + 1 : kHX; }
template <int PX>
__host__ __device__ constexpr int XM() { return PX ? -kHX : kHX - 1; }
template <int PX>
__host__ __device__ constexpr int XP() { return PX ? -kHX + 1 : kHX; }
// b of the tile, split by x parity: rows of 16 = two half-rows of 8
__device__ __forceinline__ int tile_bi(int x, int y, int z) { return ((z * kTY + y) << 4) + (x & 1) * 8 + (x >> 1); }
// natural tile index (m^T b staged by TMA) and the delta box (tile plus a one-cell ring)
__device__ __forceinline__ int tile_ti(int x, int y, int z) { return (z * kTY + y) * kTX + x; }
constexpr int kDX = kTX + 2, kDXY = (kTX + 2) * (kTY + 2);
__device__ __forceinline__ int tile_td(int x, int y, int z) { return ((z + 1) * (kTY + 2) + (y + 1)) * kDX + (x + 1); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// The operators of the contract on the split box (operand order of mom / cont).
// PX: x parity of the evaluation point (warp-uniform in every phase: immediate offsets);
// KIND: normal axis of the face (0 u, 1 v, 2 w).
template <int SY, int SZ>
struct SplitOps {
    template <int PX, int KIND>
    static __device__ __forceinline__ double mom(const double* __restrict__ F, const double* __restrict__ P, int i,
                                                 double e2, double ih) {
        double s = F[i + XM<PX>()] + F[i + XP<PX>()];
        s = s + F[i - SY];
        s = s + F[i + SY];
        s = s + F[i - SZ];
        s = s + F[i + SZ];
        const double lap = 6.0 * F[i] - s;
        constexpr int PL = KIND == 0 ? XM<PX>() : (KIND == 1 ? -SY : -SZ);
        return e2 * lap + (P[i] - P[i + PL]) * ih;
    }
    template <int PX>
    static __device__ __forceinline__ double cont(const double* __restrict__ U, const double* __restrict__ V,
                                                  const double* __restrict__ W, const double* __restrict__ P, int i,
                                                  double gamma, double ih) {
        const double div = (U[i + XP<PX>()] - U[i]) + (V[i + SY] - V[i]) + (W[i + SZ] - W[i]);
        return -div * ih - gamma * P[i];
    }
};
template <int V>
using IC = std::integral_constant<int, V>;

// band test of a tile cell (IN: an interior tile, every cell V2)
template <bool IN>
__device__ __forceinline__ bool tile_v2(const LevelK& L, int x0, int y0, int z0, int lx, int ly, int lz) {
    if (IN) return lx >= 0 && ly >= 0 && lz >= 0 && lx < kTX && ly < kTY && lz < kTZ;
    return lx >= 0 && ly >= 0 && lz >= 0 && lx < kTX && ly < kTY && lz < kTZ &&
           !band_cell(L, x0 + lx, y0 + ly, z0 + lz);
}

// eta/h^2 (6 * 0 - s): the forward-pressure term of colour k ^ (1 << AX) on a cell K of colour k,
// s the six-neighbour delta sum in x-, x+, y-, y+, z-, z+ order whose nonzero entries are the two
// neighbours along AX (t: K's index in the delta box)
template <int AX>
__device__ __forceinline__ double gsum(const double* __restrict__ ts, int t) {
    constexpr int ST = AX == 0 ? 1 : (AX == 1 ? kDX : kDXY);
    const double a = ts[t - ST], b = ts[t + ST];
    double sn;
    if (AX == 0) {
        sn = a + b;
        sn = sn + 0.0;
        sn = sn + 0.0;
        sn = sn + 0.0;
        sn = sn + 0.0;
    } else if (AX == 1) {
        sn = 0.0 + 0.0;
        sn = sn + a;
        sn = sn + b;
        sn = sn + 0.0;
        sn = sn + 0.0;
    } else {
        sn = 0.0 + 0.0;
        sn = sn + 0.0;
        sn = sn + 0.0;
        sn = sn + a;
        sn = sn + b;
    }
    return sn;
}
// The pending terms of a cell of colour K over a full forward half: the colours below K (LOWER,
// added before K's own update) or above K (the flush), ascending.  Cells whose neighbours carry
// no delta get + 0 (the oracle skips them; the value is the same).
template <int K, bool LOWER>
__device__ __forceinline__ double gath(double p, const double* __restrict__ ts, int t, double e2) {
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
        const int bit = cc ^ K;
        if (bit != 1 && bit != 2 && bit != 4) continue;
        if (LOWER ? cc > K : cc < K) continue;
        const double sn = bit == 1 ? gsum<0>(ts, t) : (bit == 2 ? gsum<1>(ts, t) : gsum<2>(ts, t));
        p = p + e2 * (6.0 * 0.0 - sn);
    }
    return p;
}
template <bool LOWER>
__device__ __forceinline__ double gath_k(int k, double p, const double* __restrict__ ts, int t, double e2) {
    switch (k) {
        case 0: return gath<0, LOWER>(p, ts, t, e2);
        case 1: return gath<1, LOWER>(p, ts, t, e2);
        case 2: return gath<2, LOWER>(p, ts, t, e2);
        case 3: return gath<3, LOWER>(p, ts, t, e2);
        case 4: return gath<4, LOWER>(p, ts, t, e2);
        case 5: return gath<5, LOWER>(p, ts, t, e2);
        case 6: return gath<6, LOWER>(p, ts, t, e2);
        default: return gath<7, LOWER>(p, ts, t, e2);
    }
}
// Generic form (partial phase ranges, boundary tiles): p_K plus the terms of colours c' in
// [lo, hi] among k ^ 1, k ^ 2, k ^ 4 (ascending), each only if a neighbour along its axis is a
// V2 cell of the tile (the oracle touches no other K).
template <bool IN>
__device__ __forceinline__ double tile_gathers(const LevelK& L, const double* __restrict__ ts, double p, int x0,
                                               int y0, int z0, int lx, int ly, int lz, int k, int lo, int hi) {
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
        const int bit = cc ^ k;
        if (bit != 1 && bit != 2 && bit != 4) continue;
        if (cc < lo || cc > hi) continue;
        const int ax = bit == 1 ? 0 : (bit == 2 ? 1 : 2);
        const int dx = ax == 0, dy = ax == 1, dz = ax == 2;
        const bool m0 = tile_v2<IN>(L, x0, y0, z0, lx - dx, ly - dy, lz - dz);
        const bool m1 = tile_v2<IN>(L, x0, y0, z0, lx + dx, ly + dy, lz + dz);
        if (!m0 && !m1) continue;
        const int t = tile_td(lx, ly, lz), st = dx + dy * kDX + dz * kDXY;
        const double a = m0 ? ts[t - st] : 0.0, b = m1 ? ts[t + st] : 0.0;
        double sn;
        if (ax == 0) {
            sn = a + b;
            sn = sn + 0.0;
            sn = sn + 0.0;
            sn = sn + 0.0;
            sn = sn + 0.0;
        } else if (ax == 1) {
            sn = 0.0 + 0.0;
            sn = sn + a;
            sn = sn + b;
            sn = sn + 0.0;
            sn = sn + 0.0;
        } else {
            sn = 0.0 + 0.0;
            sn = sn + 0.0;
            sn = sn + 0.0;
            sn = sn + a;
            sn = sn + b;
        }
        p = p + L.eta_h2 * (6.0 * 0.0 - sn);
    }
    return p;
}

template <bool FWD, bool IN>
__device__ __forceinline__ void tile_phases(const LevelK& L, double* __restrict__ xs, const double* __restrict__ bs,
                                            double* __restrict__ ts, int x0, int y0, int z0, int ph0, int ph1) {
    using TB = TileBox<FWD>;
    constexpr int SY = TB::SY, SZ = TB::SZ, BOX = TB::BOX;
    using Ops = SplitOps<SY, SZ>;
    const Geom& g = L.g;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double e2 = L.eta_h2, ih = L.inv_h, dv = L.dv, dp = L.dp, gam = L.gamma;
    double *Us = xs, *Vs = xs + BOX, *Ws = xs + 2 * BOX, *Ps = xs + 3 * BOX;
    const int cfirst = ph0 > 2 ? ph0 - 2 : 0;  // first forward pressure colour of this launch
    const bool full = ph0 <= 2 && ph1 >= 10;    // all eight colours run in this launch
    // a parity-class cell of this lane: x = 2 m + cx, y = 2 r + cy (m = lane % 8, r = lane / 8)
    const int m8 = lane & 7, r4 = lane >> 3;
    for (int ph = ph0; ph < ph1; ++ph) {
        if (ph <= 1 || ph >= 18) {  // velocity colour: warp task (z, y parity a) -> 4 rows x 8 cells
            const int c = ph <= 1 ? ph : 19 - ph;
            int li[2], bi[2], px[2];
            bool du[2], dv_[2], dw[2];
            double nu[2], nv[2], nw[2];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int task = warp + 8 * k, lz = task >> 1, a = task & 1, ly = a + 2 * r4;
                px[k] = (c + a + lz + g.z0) & 1;  // x parity of the colour-c cells of these rows
                const int lx = 2 * m8 + px[k];
                li[k] = TB::li(lx, ly, lz);
                bi[k] = tile_bi(lx, ly, lz);
                du[k] = dv_[k] = dw[k] = true;
                if (!IN) {
                    const int gx = x0 + lx, gy = y0 + ly, zl = z0 + lz;
                    const bool here = band_cell(L, gx, gy, zl);
                    du[k] = gx >= 1 && !here && !band_cell(L, gx - 1, gy, zl);
                    dv_[k] = gy >= 1 && !here && !band_cell(L, gx, gy - 1, zl);
                    dw[k] = g.gz(zl) >= 1 && !here && !band_cell(L, gx, gy, zl - 1);
                }
            }
            // independent cells: every new value before any store (loads of all six face rows in flight)
            auto velc = [&](auto pxc, int k) {
                constexpr int PX = decltype(pxc)::value;
                nu[k] = Us[li[k]] + (bs[bi[k]] - Ops::template mom<PX, 0>(Us, Ps, li[k], e2, ih)) / dv;
                nv[k] = Vs[li[k]] + (bs[kTileCells + bi[k]] - Ops::template mom<PX, 1>(Vs, Ps, li[k], e2, ih)) / dv;
                nw[k] = Ws[li[k]] + (bs[2 * kTileCells + bi[k]] - Ops::template mom<PX, 2>(Ws, Ps, li[k], e2, ih)) / dv;
            };
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                if (px[k]) velc(IC<1>{}, k);
                else velc(IC<0>{}, k);
            }
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                if (du[k]) Us[li[k]] = nu[k];
                if (dv_[k]) Vs[li[k]] = nv[k];
                if (dw[k]) Ws[li[k]] = nw[k];
            }
            __syncthreads();
        } else if (FWD) {  // forward pressure colour c, lazy gathers; ts = deltas of the colours so far
            // Eager form (the oracle's): phase c adds eta/h^2 (6 delta_K - sum_nbr delta) to every
            // pressure K, nonzero only for K of colour c (self) or c ^ bit (the axis neighbours of a
            // colour-c cell).  p_K is read only by K's own phase before the pressure phases end, so
            // the neighbour terms are added when K is next read -- those of earlier colours at the
            // start of K's phase, the rest in the flush after the last colour: the same additions
            // in the same order, hence bit-identical.
            int c = ph - 2;
            // one colour-cc cell of this lane in warp slot s (z = 2 s + cz): load + compute, then store
            struct PNew {
                int li;
                int td;
                bool on;
                double dc, u0, u1, v0, v1, w0, w1, p;
            };
            auto pload = [&](int cc, int s) {
                PNew r;
                const int cx = cc & 1, cy = (cc >> 1) & 1, cz = cc >> 2;
                const int lx = 2 * m8 + cx, ly = 2 * r4 + cy, lz = 2 * s + cz;
                r.on = IN || tile_v2<false>(L, x0, y0, z0, lx, ly, lz);
                const int li = TB::li(lx, ly, lz), td = tile_td(lx, ly, lz);
                r.li = li;
                r.td = td;
                if (!r.on) return r;
                const double p = full ? gath_k<true>(cc, Ps[li], ts, td, e2)
                                      : tile_gathers<IN>(L, ts, Ps[li], x0, y0, z0, lx, ly, lz, cc, cfirst, cc);
                const int xp = li + xp_off(cx);
                const double uL = Us[li], uR = Us[xp], vL = Vs[li], vR = Vs[li + SY], wL = Ws[li], wR = Ws[li + SZ];
                const double div = (uR - uL) + (vR - vL) + (wR - wL);
                const double rr = bs[3 * kTileCells + tile_bi(lx, ly, lz)] - (-div * ih - gam * p);
                const double dc = rr / dp;
                r.dc = dc;
                r.u0 = uL + (0.0 - dc) * ih;
                r.u1 = uR + (dc - 0.0) * ih;
                r.v0 = vL + (0.0 - dc) * ih;
                r.v1 = vR + (dc - 0.0) * ih;
                r.w0 = wL + (0.0 - dc) * ih;
                r.w1 = wR + (dc - 0.0) * ih;
                double sn = 0.0 + 0.0;  // the colour-cc neighbour sum of a colour-cc cell: six zeros
                sn = sn + 0.0;
                sn = sn + 0.0;
                sn = sn + 0.0;
                sn = sn + 0.0;
                r.p = p + e2 * (6.0 * dc - sn);
                return r;
            };
            auto pstore = [&](const PNew& r, int cx) {
                if (!r.on) return;
                ts[r.td] = r.dc;
                Us[r.li] = r.u0;
                Us[r.li + xp_off(cx)] = r.u1;
                Vs[r.li] = r.v0;
                Vs[r.li + SY] = r.v1;
                Ws[r.li] = r.w0;
                Ws[r.li + SZ] = r.w1;
                Ps[r.li] = r.p;
            };
            const int s4 = warp & 3;
            if (full) {
                // Colours of equal popcount never touch each other's faces or pressures, nor does a
                // cell read a same-group colour's delta: 0 | 1,2,4 | 3,5,6 | 7 run as four steps
                // (per cell the same operations; bit-identical).  Warps 0-3 / 4-7 take z slots 0-3.
                const bool hi = warp >= 4;
                if (!hi) pstore(pload(0, s4), 0);
                __syncthreads();
                if (hi) {
                    pstore(pload(2, s4), 0);
                } else {
                    const PNew a = pload(1, s4), b = pload(4, s4);
                    pstore(a, 1);
                    pstore(b, 0);
                }
                __syncthreads();
                if (hi) {
                    pstore(pload(5, s4), 1);
                } else {
                    const PNew a = pload(3, s4), b = pload(6, s4);
                    pstore(a, 1);
                    pstore(b, 0);
                }
                __syncthreads();
                if (!hi) pstore(pload(7, s4), 1);
                __syncthreads();
                ph = 9;
                c = 7;
            } else {
                if (warp < 4) pstore(pload(c, s4), c & 1);
                __syncthreads();
            }
            if (ph == 9 || ph + 1 == ph1) {  // flush: the terms of colours [cfirst, c] still pending
                // tile cells by parity class (warp task: class k, z slot s), then the six face slabs
                // (ring edges and corners have no tile neighbour)
                for (int task = warp; task < 32; task += 8) {
                    const int k = task >> 2, s = task & 3;
                    const int lx = 2 * m8 + (k & 1), ly = 2 * r4 + ((k >> 1) & 1), lz = 2 * s + (k >> 2);
                    const int li = TB::li(lx, ly, lz), td = tile_td(lx, ly, lz);
                    if (full) {
                        // relaxed cell: the colours above k; a band cell of a boundary tile had no phase
                        // of its own: the colours below k first (ascending, as the generic form)
                        double p = Ps[li];
                        if (!IN && !tile_v2<false>(L, x0, y0, z0, lx, ly, lz)) p = gath_k<true>(k, p, ts, td, e2);
                        Ps[li] = gath_k<false>(k, p, ts, td, e2);
                    } else {
                        const bool relaxed = k >= cfirst && k <= c && tile_v2<IN>(L, x0, y0, z0, lx, ly, lz);
                        Ps[li] = tile_gathers<IN>(L, ts, Ps[li], x0, y0, z0, lx, ly, lz, k, relaxed ? k + 1 : cfirst, c);
                    }
                }
                constexpr int NSX = 2 * kTY * kTZ, NSY = 2 * kTX * kTZ, NSZ = 2 * kTX * kTY;
                for (int e = tid; e < NSX + NSY + NSZ; e += kTileThreads) {
                    int lx, ly, lz, ax;
                    if (e < NSX) {
                        ax = 0;
                        lx = (e & 1) ? kTX : -1;
                        ly = (e >> 1) % kTY;
                        lz = (e >> 1) / kTY;
                    } else if (e < NSX + NSY) {
                        const int f = e - NSX;
                        ax = 1;
                        lx = f % kTX;
                        ly = ((f / kTX) & 1) ? kTY : -1;
                        lz = f / (2 * kTX);
                    } else {
                        const int f = e - NSX - NSY;
                        ax = 2;
                        lx = f % kTX;
                        ly = (f / kTX) % kTY;
                        lz = (f / (kTX * kTY)) ? kTZ : -1;
                    }
                    if (!IN) {  // K must be an active cell of the level
                        const int gx = x0 + lx, gy = y0 + ly, gz = g.gz(z0 + lz);
                        if (gx < 0 || gy < 0 || gz < 0 || gx >= g.nx || gy >= g.ny || gz >= g.gnz) continue;
                    }
                    const int li = TB::li(lx, ly, lz), td = tile_td(lx, ly, lz);
                    const int k = (lx & 1) + 2 * (ly & 1) + 4 * (lz & 1);
                    if (full) {  // the one term of its inward neighbour's colour (a band neighbour carries delta 0)
                        const bool low = ax == 0 ? lx < 0 : (ax == 1 ? ly < 0 : lz < 0);
                        const int st = ax == 0 ? 1 : (ax == 1 ? kDX : kDXY);
                        const double d = ts[td + (low ? st : -st)];
                        const double a = low ? 0.0 : d, bb = low ? d : 0.0;  // the (-, +) pair
                        double sn;
                        if (ax == 0) {
                            sn = a + bb;
                            sn = sn + 0.0;
                            sn = sn + 0.0;
                            sn = sn + 0.0;
                            sn = sn + 0.0;
                        } else if (ax == 1) {
                            sn = 0.0 + 0.0;
                            sn = sn + a;
                            sn = sn + bb;
                            sn = sn + 0.0;
                            sn = sn + 0.0;
                        } else {
                            sn = 0.0 + 0.0;
                            sn = sn + 0.0;
                            sn = sn + 0.0;
                            sn = sn + a;
                            sn = sn + bb;
                        }
                        Ps[li] = Ps[li] + e2 * (6.0 * 0.0 - sn);
                    } else {
                        Ps[li] = tile_gathers<IN>(L, ts, Ps[li], x0, y0, z0, lx, ly, lz, k, cfirst, c);
                    }
                }
                __syncthreads();
            }
        } else {  // reverse (left-preconditioned) pressure colour c; ts = m^T b of the tile
            // Two warps per 32 colour-c cells: even warps evaluate the six momentum rows at the
            // cells' faces (flux part), odd warps the seven continuity rows (C and its six
            // neighbours) and hand (lc, s) over through shared memory; the even warps finish
            // prev_core's expression in its operand order.  Same-colour cells never read each
            // other's pressure, so the update goes in place.
            const int c = 17 - ph;
            const int half = warp & 1, s = warp >> 1, cell = (s << 5) | lane;
            const int cx = c & 1, lx = 2 * m8 + cx, ly = 2 * r4 + ((c >> 1) & 1), lz = 2 * s + (c >> 2);
            const bool v2 = IN || tile_v2<false>(L, x0, y0, z0, lx, ly, lz);
            const int i = TB::li(lx, ly, lz);
            double* xch = ts + kTileCells;  // [2][kTileCells / 8]: lc, s
            double fl = 0.0;
            auto rev = [&](auto pxc) {
                constexpr int PX = decltype(pxc)::value, QX = 1 - PX;
                if (half == 0) {
                    const int ir = i + XP<PX>();  // the u face on the right: x parity 1 - PX
                    const double luL = Ops::template mom<PX, 0>(Us, Ps, i, e2, ih);
                    const double luR = Ops::template mom<QX, 0>(Us, Ps, ir, e2, ih);
                    const double lvL = Ops::template mom<PX, 1>(Vs, Ps, i, e2, ih);
                    const double lvR = Ops::template mom<PX, 1>(Vs, Ps, i + SY, e2, ih);
                    const double lwL = Ops::template mom<PX, 2>(Ws, Ps, i, e2, ih);
                    const double lwR = Ops::template mom<PX, 2>(Ws, Ps, i + SZ, e2, ih);
                    fl = ((luR - luL) + (lvR - lvL)) + (lwR - lwL);
                } else {
                    const double lc = Ops::template cont<PX>(Us, Vs, Ws, Ps, i, gam, ih);
                    double sn = Ops::template cont<QX>(Us, Vs, Ws, Ps, i + XM<PX>(), gam, ih) +
                                Ops::template cont<QX>(Us, Vs, Ws, Ps, i + XP<PX>(), gam, ih);
                    sn = sn + Ops::template cont<PX>(Us, Vs, Ws, Ps, i - SY, gam, ih);
                    sn = sn + Ops::template cont<PX>(Us, Vs, Ws, Ps, i + SY, gam, ih);
                    sn = sn + Ops::template cont<PX>(Us, Vs, Ws, Ps, i - SZ, gam, ih);
                    sn = sn + Ops::template cont<PX>(Us, Vs, Ws, Ps, i + SZ, gam, ih);
                    xch[cell] = lc;
                    xch[kTileCells / 8 + cell] = sn;
                }
            };
            if (v2) {
                if (cx) rev(IC<1>{});
                else rev(IC<0>{});
            }
            __syncthreads();
            if (v2 && half == 0) {
                const double cl = fl * ih + e2 * (6.0 * xch[cell] - xch[kTileCells / 8 + cell]);
                Ps[i] = Ps[i] + (ts[tile_ti(lx, ly, lz)] - cl) / dp;
            }
            __syncthreads();
        }
    }
}

__device__ __forceinline__ void tma_load(void* dst, const CUtensorMap* m, int c0, int c1, int c2, int c3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}

// contiguous global -> shared bulk copy against the same mbarrier (16-byte aligned, size % 16 == 0)
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// L2 prefetch of a box (no shared-memory destination, no barrier): a hint only, always safe
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* m, int c0, int c1, int c2, int c3) {
    asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(
                     reinterpret_cast<uint64_t>(m)),
                 "r"(c0), "r"(c1), "r"(c2), "r"(c3)
                 : "memory");
}

// FWD: phases [ph0, ph1) within 0..9; REV: within 10..19 -- on the tiles of colour T.
// pf > 0: the CTA also prefetches into L2 the boxes of tile blockIdx.x + pf (the CTA most likely to
// take this SM slot next: pf = resident CTAs of the device), so that tile's TMA loads hit L2
// while this tile computes.
// tmx: x box map; tmb: b (tile box, NB fields); tmc: m^T b (tile box, one field; REV only).
template <bool FWD>
__global__ void __launch_bounds__(kTileThreads, 2)
    k_dgs_tile(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmb,
               const __grid_constant__ CUtensorMap tmc, LevelK L, double* __restrict__ X, int T, int ph0, int ph1,
               int ntx, int nty, int pf, int kz0, int kzs, const double* __restrict__ bpk) {
    using TB = TileBox<FWD>;
    extern __shared__ __align__(128) double tsm_raw[];
    // 128-byte aligned by pointer arithmetic on the shared array (an integer round trip would hide
    // the address space and turn every box access into a generic LD/ST)
    double* xs = tsm_raw + (((128u - (smem_u32(tsm_raw) & 127u)) & 127u) >> 3);
    double* bs = xs + 4 * TB::BOX;          // b of the tile, NB fields (split rows)
    double* ts = bs + TB::NB * kTileCells;  // deltas (FWD) / m^T b + exchange (REV)
    uint64_t* bar = reinterpret_cast<uint64_t*>(ts + TB::TS);
    const Geom& g = L.g;
    const int tid = threadIdx.x;
    // tile of colour T for this CTA (z parity on global tile indices: slab parts start on a tile)
    const int pz = ((T >> 2) ^ (g.z0 / kTZ)) & 1;
    const int hx = (ntx - (T & 1) + 1) >> 1, hy = (nty - ((T >> 1) & 1) + 1) >> 1;
    // pf < 0: this launch walks its tiles backwards, so it starts where the previous launch (the
    // neighbouring tile colour, walked forwards) ended -- on data still in L2
    const int bi = pf < 0 ? static_cast<int>(gridDim.x) - 1 - static_cast<int>(blockIdx.x) : static_cast<int>(blockIdx.x);
    // tile layers of this launch: the colour's layers kz0, kz0 + kzs, ... (all of them: 0, 1; a slab
    // part's boundary / interior layers when the halo transfer overlaps the interior tiles)
    const int tx = 2 * (bi % hx) + (T & 1), ty = 2 * ((bi / hx) % hy) + ((T >> 1) & 1),
              tz = 2 * (kz0 + kzs * (bi / (hx * hy))) + pz;
    const int x0 = tx * kTX, y0 = ty * kTY, z0 = tz * kTZ;  // z0: local plane of the part
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_wait();  // the previous kernel's writes are visible from here on
    if (tid == 0) {  // TMA: the x box (4 fields), the tile's b (NB fields), m^T b (REV)
        const uint32_t bytes = (4u * TB::BOX + (TB::NB + (FWD ? 0 : 1)) * kTileCells) * sizeof(double);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                     : "memory");
        tma_load(xs, &tmx, x0 - 2 + g.xo, y0, z0 - 1 + g.zg, 0, bar);
        if (bpk) {  // tile-major packed b / c_b (k_dgs_cb<true>): contiguous, already parity-split
            const double* tb = bpk + (static_cast<int64_t>(tz * (g.ny / kTY) + ty) * ntx + tx) * (5 * kTileCells);
            bulk_load(bs, tb, TB::NB * kTileCells * sizeof(double), bar);
            if (!FWD) bulk_load(ts, tb + 4 * kTileCells, kTileCells * sizeof(double), bar);
        } else {
            tma_load(bs, &tmb, x0 + g.xo, y0 + 1, z0 + g.zg, 0, bar);
            if (!FWD) tma_load(ts, &tmc, x0 + g.xo, y0 + 1, z0 + g.zg, 0, bar);
        }
        const int bn = bi + pf;
        if (pf > 0 && bn < static_cast<int>(gridDim.x)) {
            const int nx0 = (2 * (bn % hx) + (T & 1)) * kTX, ny0 = (2 * ((bn / hx) % hy) + ((T >> 1) & 1)) * kTY,
                      nz0 = (2 * (kz0 + kzs * (bn / (hx * hy))) + pz) * kTZ;
            tma_prefetch(&tmx, nx0 - 2 + g.xo, ny0, nz0 - 1 + g.zg, 0);
            tma_prefetch(&tmb, nx0 + g.xo, ny0 + 1, nz0 + g.zg, 0);
            if (!FWD) tma_prefetch(&tmc, nx0 + g.xo, ny0 + 1, nz0 + g.zg, 0);
        }
    }
    if (FWD)
        for (int k = tid; k < TB::TS; k += kTileThreads) ts[k] = 0.0;
    if (tid == 0) {  // one waiter (with a suspend hint), the others wait at the barrier
        const uint32_t ba = smem_u32(bar);
        asm volatile(
            "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0, 1000000;\n @!p bra "
            "WAIT_%=;\n}" ::"r"(ba)
            : "memory");
    }
    __syncthreads();
    {  // x-parity split of every staged row, in place (a warp reads its rows' pairs, then writes)
        const int lane = tid & 31, warp = tid >> 5;
        constexpr int ROWS = 4 * TB::BZ * TB::BY;
        const int lr = lane / kHX, lq = lane % kHX;  // 3 rows of 10 pairs per warp step
        for (int r0 = warp * 3; r0 < ROWS; r0 += 24) {
            const int r = r0 + lr;
            const bool ok = lane < 3 * kHX && r < ROWS;
            double2 v = make_double2(0.0, 0.0);
            if (ok) v = *reinterpret_cast<const double2*>(&xs[r * kBX + 2 * lq]);
            __syncwarp();
            if (ok) {
                xs[r * kBX + lq] = v.x;
                xs[r * kBX + kHX + lq] = v.y;
            }
            __syncwarp();
        }
        constexpr int BROWS = TB::NB * kTZ * kTY;  // rows of 16: 4 rows of 8 pairs per warp step
        for (int r0 = warp * 4; r0 < (bpk ? 0 : BROWS); r0 += 32) {
            const int r = r0 + (lane >> 3), q = lane & 7;
            const bool ok = r < BROWS;
            double2 v = make_double2(0.0, 0.0);
            if (ok) v = *reinterpret_cast<const double2*>(&bs[(r << 4) + 2 * q]);
            __syncwarp();
            if (ok) {
                bs[(r << 4) + q] = v.x;
                bs[(r << 4) + 8 + q] = v.y;
            }
            __syncwarp();
        }
    }
    __syncthreads();
    const int64_t fs = g.fs;
    // interior: every cell of the tile and of the cell layer around it is a V2 cell of the level
    const int gz0 = g.gz(z0), bw = L.bw;
    const bool interior = x0 - 1 >= bw && y0 - 1 >= bw && gz0 - 1 >= bw && x0 + kTX + 1 <= g.nx - bw &&
                          y0 + kTY + 1 <= g.ny - bw && gz0 + kTZ + 1 <= g.gnz - bw;
    if (interior) tile_phases<FWD, true>(L, xs, bs, ts, x0, y0, z0, ph0, ph1);
    else tile_phases<FWD, false>(L, xs, bs, ts, x0, y0, z0, ph0, ph1);
    // Write back the DOFs the phases may have changed: the tile's own, plus (after forward
    // pressure phases) its high faces and the pressures of the six neighbouring slabs.  Rows of
    // 16 go out as 16-byte stores (an even/odd pair each; the lanes of a half-warp read rows two
    // apart).  Every slot written was loaded by this CTA and no other CTA touches it during the
    // launch; wall and ghost slots were loaded as 0 and never changed.
    const int hw = (FWD && ph1 > 2) ? 1 : 0;  // a forward pressure phase ran
    auto rows = [&](int f, int ylo, int nyr, int zlo, int nzr) {
        const int n = nyr * nzr * (kTX / 2);
        for (int e = tid; e < n; e += kTileThreads) {
            const int q = e & 7, r = e >> 3;
            // rows in the order y = 0, 2, 4, ..., 1, 3, ... within each z (nyr even) for conflict-free reads
            const int ry = r % nyr, lz = zlo + r / nyr;
            const int ly = ylo + ((nyr & 1) ? ry : (ry < nyr / 2 ? 2 * ry : 2 * (ry - nyr / 2) + 1));
            const int li = TB::li(2 * q, ly, lz);
            const double2 v = make_double2(xs[f * TB::BOX + li], xs[f * TB::BOX + li + kHX]);
            *reinterpret_cast<double2*>(&X[f * fs + g.slot(x0 + 2 * q, y0 + ly, z0 + lz)]) = v;
        }
    };
    auto col = [&](int f, int lx) {  // one x column of the tile's rows
        for (int e = tid; e < kTY * kTZ; e += kTileThreads) {
            const int ly = e % kTY, lz = e / kTY;
            X[f * fs + g.slot(x0 + lx, y0 + ly, z0 + lz)] = xs[f * TB::BOX + TB::li(lx, ly, lz)];
        }
    };
    rows(0, 0, kTY, 0, kTZ);
    rows(1, 0, kTY + hw, 0, kTZ);
    rows(2, 0, kTY, 0, kTZ + hw);
    rows(3, 0, kTY, 0, kTZ);
    if (hw) {
        col(0, kTX);
        col(3, -1);
        col(3, kTX);
        rows(3, -1, 1, 0, kTZ);
        rows(3, kTY, 1, 0, kTZ);
        rows(3, 0, kTY, -1, 1);
        rows(3, 0, kTY, kTZ, 1);
    }
}

// ------------------------------------------ z-slab halo frames ------
// A Vanka phase changes only band DOFs.  On the two boundary planes of a z-slab that is a frame
// around the plane's perimeter (rows / columns within bw + 1 slots of the x and y walls) as long as
// the planes are not themselves within reach of a z wall, so the halo refresh after a Vanka phase
// moves the frames of the 2 planes x 4 fields (a few 10 KB at 512^2) instead of the planes.
// Frame of one padded plane (py rows of px columns): rows [0, RL) and [py - RH, py) whole, and of
// the rows in between the columns [0, CL) and [px - CH, px).
struct FrameDims {
    int RL, RH, CL, CH, px, py;
    __host__ __device__ int mid_rows() const { return py - RL - RH; }
    __host__ __device__ int64_t count() const {
        return static_cast<int64_t>(RL + RH) * px + static_cast<int64_t>(mid_rows()) * (CL + CH);
    }
};
static FrameDims frame_dims(const Geom& g, int bw) {
    FrameDims f;
    f.px = g.px;
    f.py = g.py;
    f.RL = bw + 2;                      // y slots -1 .. bw (a block at cell y updates faces y and y + 1)
    f.RH = bw + 1;                      // y slots ny - bw .. ny
    f.CL = g.xo + bw + 1;               // x slots .. bw
    f.CH = g.px - g.xo - g.nx + bw;     // x slots nx - bw ..
    return f;
}
// to_buf: buf <- frames of the padded planes zs, zs + 1 of the 4 fields; else the reverse
// blockIdx.z picks the plane pair: (buf0, zs0) or (buf1, zs1); a null buffer means no neighbour there
__global__ void __launch_bounds__(256) k_frame_copy(Geom g, FrameDims f, double* __restrict__ X,
                                                    double* __restrict__ buf0, int zs0, double* __restrict__ buf1,
                                                    int zs1, int to_buf) {
    double* __restrict__ buf = blockIdx.z ? buf1 : buf0;
    const int zs = blockIdx.z ? zs1 : zs0;
    if (!buf) return;
    const int64_t n = f.count();
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= n) return;
    int row, col;
    const int64_t top = static_cast<int64_t>(f.RL) * f.px, bot = static_cast<int64_t>(f.RH) * f.px;
    if (e < top) {
        row = static_cast<int>(e / f.px);
        col = static_cast<int>(e % f.px);
    } else if (e < top + bot) {
        row = f.py - f.RH + static_cast<int>((e - top) / f.px);
        col = static_cast<int>((e - top) % f.px);
    } else {
        const int64_t r = e - top - bot;
        const int w = f.CL + f.CH, c = static_cast<int>(r % w);
        row = f.RL + static_cast<int>(r / w);
        col = c < f.CL ? c : f.px - f.CH + (c - f.CL);
    }
    const int pf = blockIdx.y;  // plane (0, 1) x field (0..3)
    const int64_t xi = static_cast<int64_t>(pf >> 1) * g.fs + static_cast<int64_t>(zs + (pf & 1)) * g.sz +
                       static_cast<int64_t>(row) * g.sy + col;
    double* b = buf + static_cast<int64_t>(pf) * n + e;
    if (to_buf) *b = X[xi];
    else X[xi] = *b;
}

// ------------------------------------------ general labelled domains ------
// SPEC:17-97 (domain), 124/176 (dropped Neumann legs), 245-251 (Vanka signature classes):
// Dirichlet / Interior / Exterior cells inside the implicit Dirichlet ring.  The padded layout is
// the box's: Dirichlet-valued and Inactive slots hold 0 forever (never written), so every stencil
// sum is already right; what changes is WHICH slots are DOFs (L.cls bits instead of coordinate
// tests), the momentum diagonal 6 - dropped legs (cls_diag), band membership (a mask, not a
// distance to the wall) and the Vanka class table (kidx -> ktab).  One kernel per phase, per-point
// arithmetic in the contract's operand order: bit-identical to the oracle on any labelling, and to
// the box kernels when every cell is Interior.
__global__ void k_apply_m(LevelK L, const double* __restrict__ X, const double* __restrict__ B,
                          double* __restrict__ Y, double gamma) {
    pdl_wait();
    Cell c;
    if (!thread_cell(L.g, c)) return;
    const Geom& g = L.g;
    const int64_t fs = g.fs, i = c.i;
    const uint32_t m = L.cls[i];
    if (!(m & (CLS_P | CLS_U | CLS_V | CLS_W))) return;
    const double *U = X, *V = X + fs, *W = X + 2 * fs, *P = X + 3 * fs;
    if (m & CLS_U) {
        const double y = mom_d(L, U, P, i, 1, cls_diag(m, 0));
        Y[i] = B ? B[i] - y : y;
    }
    if (m & CLS_V) {
        const double y = mom_d(L, V, P, i, g.sy, cls_diag(m, 1));
        Y[fs + i] = B ? B[fs + i] - y : y;
    }
    if (m & CLS_W) {
        const double y = mom_d(L, W, P, i, g.sz, cls_diag(m, 2));
        Y[2 * fs + i] = B ? B[2 * fs + i] - y : y;
    }
    if (m & CLS_P) {
        const double y = cont(L, U, V, W, P, i, gamma);
        Y[3 * fs + i] = B ? B[3 * fs + i] - y : y;
    }
}

// DGS velocity phase on the V2 faces of one red-black colour (their stencils are full: diagonal 6).
// Threads only on the colour's cells: x = 2 i + ((y + z + colour) & 1).
__global__ void k_dgs_vel_m(LevelK L, double* __restrict__ X, const double* __restrict__ B, int colour) {
    const Geom& g = L.g;
    Cell c;
    c.y = blockIdx.y * BY + threadIdx.y;
    c.z = blockIdx.z;
    c.x = 2 * (blockIdx.x * BX + threadIdx.x) + ((c.y + g.gz(c.z) + colour) & 1);
    if (c.x >= g.nx || c.y >= g.ny) return;
    c.i = g.slot(c.x, c.y, c.z);
    const int64_t fs = g.fs, i = c.i;
    const uint32_t m = L.cls[i];
    if (!(m & (CLS_U2 | CLS_V2 | CLS_W2))) return;
    double *U = X, *V = X + fs, *W = X + 2 * fs;
    const double* P = X + 3 * fs;
    if (m & CLS_U2) {
        const double r = B[i] - mom(L, U, P, i, 1);
        U[i] = U[i] + r / L.dv;
    }
    if (m & CLS_V2) {
        const double r = B[fs + i] - mom(L, V, P, i, g.sy);
        V[i] = V[i] + r / L.dv;
    }
    if (m & CLS_W2) {
        const double r = B[2 * fs + i] - mom(L, W, P, i, g.sz);
        W[i] = W[i] + r / L.dv;
    }
}

// Threads only on the cells of one parity colour (labelled levels are single parts: local = global planes).
__device__ __forceinline__ bool colour_cell(const Geom& g, int colour, Cell& c) {
    c.x = 2 * (blockIdx.x * BX + threadIdx.x) + (colour & 1);
    c.y = 2 * (blockIdx.y * BY + threadIdx.y) + ((colour >> 1) & 1);
    c.z = 2 * blockIdx.z + (colour >> 2);
    if (c.x >= g.nx || c.y >= g.ny || c.z >= g.nz) return false;
    c.i = g.slot(c.x, c.y, c.z);
    return true;
}
inline dim3 colour_grid(const Geom& g) {
    return dim3(((g.nx + 1) / 2 + BX - 1) / BX, ((g.ny + 1) / 2 + BY - 1) / BY, (g.nz + 1) / 2);
}
inline dim3 redblack_grid(const Geom& g) { return dim3(((g.nx + 1) / 2 + BX - 1) / BX, (g.ny + BY - 1) / BY, g.nz); }

// Forward pressure phase of parity colour `colour`, part 1: delta at the colour's cells only (0 on
// its band cells); D at cells of other colours is never read as this phase's delta (part 2 knows
// every neighbour's colour from its coordinates), so nothing else is written.
__global__ void k_dgs_pdelta_m(LevelK L, const double* __restrict__ X, const double* __restrict__ B,
                               double* __restrict__ D, int colour) {
    Cell c;
    if (!colour_cell(L.g, colour, c)) return;
    const int64_t fs = L.g.fs, i = c.i;
    const uint32_t m = L.cls[i];
    double d = 0.0;
    if ((m & (CLS_P | CLS_BAND)) == CLS_P) {
        const double r = B[3 * fs + i] - cont(L, X, X + fs, X + 2 * fs, X + 3 * fs, i, L.gamma);
        d = r / L.dp;
    }
    D[i] = d;
}

// Part 2: x += sum_C delta_C M_.C in gather form.  Only cells of the colour itself (self term,
// their low faces) or of a colour one parity bit away (the neighbours of a colour cell along that
// axis: one low face and the pressure) are touched -- exactly the DOFs the oracle updates; a
// neighbour of any other colour contributes the literal 0.0 of the reference sum.
__global__ void k_dgs_papply_m(LevelK L, double* __restrict__ X, const double* __restrict__ D, int colour) {
    Cell c;
    if (!thread_cell(L.g, c)) return;
    const Geom& g = L.g;
    const int bit = pcolour(g, c) ^ colour;
    if (bit != 0 && bit != 1 && bit != 2 && bit != 4) return;
    const int64_t fs = g.fs, i = c.i, sy = g.sy, sz = g.sz;
    const uint32_t m = L.cls[i];
    if (bit == 0) {  // a cell of the colour: its three low faces see (0 - delta), its pressure 6 delta
        const double dc = D[i];
        if (m & CLS_U) X[i] = X[i] + (0.0 - dc) * L.inv_h;
        if (m & CLS_V) X[fs + i] = X[fs + i] + (0.0 - dc) * L.inv_h;
        if (m & CLS_W) X[2 * fs + i] = X[2 * fs + i] + (0.0 - dc) * L.inv_h;
        if (m & CLS_P) {
            double s = 0.0 + 0.0;
            s = s + 0.0;
            s = s + 0.0;
            s = s + 0.0;
            s = s + 0.0;
            X[3 * fs + i] = X[3 * fs + i] + L.eta_h2 * (6.0 * dc - s);
        }
        return;
    }
    // the two neighbours along the differing axis carry the colour
    const int64_t st = bit == 1 ? 1 : (bit == 2 ? sy : sz);
    const double dm = D[i - st], dp = D[i + st];
    const uint32_t fbit = bit == 1 ? CLS_U : (bit == 2 ? CLS_V : CLS_W);
    const int64_t fo = bit == 1 ? 0 : (bit == 2 ? fs : 2 * fs);
    if (m & fbit) X[fo + i] = X[fo + i] + (dm - 0.0) * L.inv_h;  // the low face along that axis
    if (m & CLS_P) {
        double s;
        if (bit == 1) {
            s = dm + dp;
            s = s + 0.0;
            s = s + 0.0;
            s = s + 0.0;
            s = s + 0.0;
        } else if (bit == 2) {
            s = 0.0 + 0.0;
            s = s + dm;
            s = s + dp;
            s = s + 0.0;
            s = s + 0.0;
        } else {
            s = 0.0 + 0.0;
            s = s + 0.0;
            s = s + 0.0;
            s = s + dm;
            s = s + dp;
        }
        X[3 * fs + i] = X[3 * fs + i] + L.eta_h2 * (6.0 * 0.0 - s);
    }
}

// Reverse pressure phase on V2 cells: prev_core with the six face rows' own diagonals (a face of a
// V2 cell may be a V1 face with a dropped leg one cell further out).
__global__ void k_dgs_prev_m(LevelK L, double* __restrict__ X, int colour) {
    Cell c;
    if (!colour_cell(L.g, colour, c)) return;
    const Geom& g = L.g;
    const int64_t fs = g.fs, sy = g.sy, sz = g.sz, i = c.i;
    const uint32_t m0 = L.cls[i];
    if ((m0 & (CLS_P | CLS_BAND)) != CLS_P) return;
    const uint32_t mx = L.cls[i + 1], my = L.cls[i + sy], mz = L.cls[i + sz];
    const double *U = X, *V = X + fs, *W = X + 2 * fs, *P = X + 3 * fs;
    const double luL = mom_d(L, U, P, i, 1, cls_diag(m0, 0));
    const double luR = mom_d(L, U, P, i + 1, 1, cls_diag(mx, 0));
    const double lvL = mom_d(L, V, P, i, sy, cls_diag(m0, 1));
    const double lvR = mom_d(L, V, P, i + sy, sy, cls_diag(my, 1));
    const double lwL = mom_d(L, W, P, i, sz, cls_diag(m0, 2));
    const double lwR = mom_d(L, W, P, i + sz, sz, cls_diag(mz, 2));
    const double fl = ((luR - luL) + (lvR - lvL)) + (lwR - lwL);
    const double lc = cont(L, U, V, W, P, i, L.gamma);
    double s = cont(L, U, V, W, P, i - 1, L.gamma) + cont(L, U, V, W, P, i + 1, L.gamma);
    s = s + cont(L, U, V, W, P, i - sy, L.gamma);
    s = s + cont(L, U, V, W, P, i + sy, L.gamma);
    s = s + cont(L, U, V, W, P, i - sz, L.gamma);
    s = s + cont(L, U, V, W, P, i + sz, L.gamma);
    const double cl = fl * L.inv_h + L.eta_h2 * (6.0 * lc - s);
    X[3 * fs + i] = P[i] + (L.cb[i] - cl) / L.dp;
}

// Residual slot s8 (0..5 the faces uL, uR, vL, vR, wL, wR; 6 the pressure) of the Vanka block at cell
// slot i with active-face mask m: the momentum row with the face's own diagonal (labelled levels: from
// the DofMap bits of the face's cell; else 6) or the continuity row; 0 for an inactive face.
template <bool M>
__device__ __forceinline__ double vanka_slot_residual_m(const LevelK& L, const double* __restrict__ X,
                                                        const double* __restrict__ B, int64_t i, int m, int s8) {
    const Geom& g = L.g;
    const int64_t fs = g.fs, sy = g.sy, sz = g.sz;
    const bool mom_row = s8 < 6;
    if (mom_row && !((m >> s8) & 1)) return 0.0;
    const double *U = X, *V = X + fs, *W = X + 2 * fs, *P = X + 3 * fs;
    if (!mom_row) return B[3 * fs + i] - cont(L, U, V, W, P, i, L.gamma);
    const int d = s8 >> 1;
    const int64_t st = d == 0 ? 1 : (d == 1 ? sy : sz);
    const int64_t jj = i + ((s8 & 1) ? st : 0);  // face slot
    const double diag = M ? cls_diag(L.cls[jj], d) : 6.0;
    return B[d * fs + jj] - mom_d(L, X + d * fs, P, jj, st, diag);
}

// One Vanka colour list (a parity colour or a merged complementary pair), part 1: 8 lanes per block,
// lane s < 7 computes residual slot s (the momentum row with the face's own diagonal / the continuity
// row) and the correction of DOF s, delta_s = sum_q K[s][q] r_q with r_q gathered by warp shuffles in
// ascending q (the oracle's order); kidx picks the block's signature class in ktab on labelled levels.
// Part 2 (k_vanka_apply8 / k_vanka_apply) adds the corrections: Jacobi within the list.
// M: labelled level (face diagonals from L.cls, class index from kidx); else the box (diagonal 6,
// the class is the face mask).
template <bool M>
__global__ void __launch_bounds__(256) k_vanka_delta8(LevelK L, const double* __restrict__ X,
                                                        const double* __restrict__ B,
                                                        const int32_t* __restrict__ cells,
                                                        const uint8_t* __restrict__ masks,
                                                        const uint16_t* __restrict__ kidx, int n,
                                                        const double* __restrict__ ktab, double* __restrict__ delta) {
    pdl_wait();
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, lane = threadIdx.x & 31, s8 = lane & 7;
    const int t = tid >> 3;
    const bool act = t < n;
    const Geom& g = L.g;
    const int64_t fs = g.fs, sy = g.sy, sz = g.sz;
    double r = 0.0;
    int ki = 0;
    if (act && s8 < 7) {
        const int m = masks[t];
        ki = M ? kidx[t] : m;
        r = vanka_slot_residual_m<M>(L, X, B, cells[t], m, s8);
    }
    const double* K = ktab + static_cast<int64_t>(ki) * 49 + (s8 < 7 ? s8 : 0) * 7;
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < 7; ++q) {
        const double rq = __shfl_sync(0xffffffffu, r, (lane & ~7) + q);
        acc = acc + K[q] * rq;
    }
    if (act && s8 < 7) delta[static_cast<int64_t>(t) * 8 + s8] = acc;
}
__global__ void __launch_bounds__(256) k_vanka_apply8(LevelK L, double* __restrict__ X,
                                                      const int32_t* __restrict__ cells,
                                                      const uint8_t* __restrict__ masks, int n,
                                                      const double* __restrict__ delta) {
    pdl_wait();
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, s8 = tid & 7, t = tid >> 3;
    if (t >= n || s8 == 7) return;
    const Geom& g = L.g;
    const int64_t fs = g.fs, i = cells[t];
    const int m = masks[t];
    if (s8 < 6 && !((m >> s8) & 1)) return;
    const int64_t offs = s8 == 0 ? 0 : s8 == 1 ? 1 : s8 == 2 ? fs : s8 == 3 ? fs + g.sy : s8 == 4 ? 2 * fs
                         : s8 == 5 ? 2 * fs + g.sz : 3 * fs;
    X[i + offs] = X[i + offs] + delta[static_cast<int64_t>(t) * 8 + s8];
}

// Restriction / prolongation with the coarse / fine DofMap bits deciding which DOFs exist; legs
// into Dirichlet or Inactive slots read 0 (dropped, no renormalisation).
__global__ void k_restrict_m(LevelK F, LevelK C, const double* __restrict__ R, double* __restrict__ BC) {
    pdl_wait();
    const Geom &fg = F.g, &cg = C.g;
    Cell c;
    if (!thread_cell(cg, c)) return;
    const uint32_t m = C.cls[c.i];
    if (!(m & (CLS_P | CLS_U | CLS_V | CLS_W))) return;
    const int64_t ffs = fg.fs, cfs = cg.fs;
    const int64_t fb = fg.slot(2 * c.x, 2 * c.y, 2 * c.z);
    const int64_t sx = 1, sy = fg.sy, sz = fg.sz;
    if (m & CLS_U) BC[c.i] = restrict_face(R, fb, sx, sy, sz);
    if (m & CLS_V) BC[cfs + c.i] = restrict_face(R + ffs, fb, sy, sx, sz);
    if (m & CLS_W) BC[2 * cfs + c.i] = restrict_face(R + 2 * ffs, fb, sz, sx, sy);
    if (m & CLS_P) {
        const double* RP = R + 3 * ffs;
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int ii = 0; ii < 2; ++ii) s = s + RP[fb + k * sz + j * sy + ii];
        BC[3 * cfs + c.i] = 0.125 * s;
    }
}

__global__ void k_prolong_add_m(LevelK F, LevelK C, const double* __restrict__ E, double* __restrict__ X) {
    pdl_wait();
    Cell c;
    if (!thread_cell(F.g, c)) return;
    const Geom &fg = F.g, &cg = C.g;
    const uint32_t m = F.cls[c.i];
    if (!(m & (CLS_P | CLS_U | CLS_V | CLS_W))) return;
    const int64_t ffs = fg.fs, cfs = cg.fs;
    const int z = c.z;
    if (m & CLS_U) X[c.i] = X[c.i] + prolong_face<0>(E, cg, c.x, c.y, z);
    if (m & CLS_V) X[ffs + c.i] = X[ffs + c.i] + prolong_face<1>(E + cfs, cg, c.x, c.y, z);
    if (m & CLS_W) X[2 * ffs + c.i] = X[2 * ffs + c.i] + prolong_face<2>(E + 2 * cfs, cg, c.x, c.y, z);
    if (m & CLS_P) X[3 * ffs + c.i] = X[3 * ffs + c.i] + E[3 * cfs + cg.slot(c.x >> 1, c.y >> 1, z >> 1)];
}

// compact FieldVector <-> padded layout through the level's slot list (SPEC:48 numbering)
__global__ void k_gather(const int32_t* __restrict__ slots, int64_t n, const double* __restrict__ X,
                         double* __restrict__ out) {
    pdl_wait();
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        out[k] = X[slots[k]];
}
__global__ void k_scatter(const int32_t* __restrict__ slots, int64_t n, const double* __restrict__ in,
                          double* __restrict__ X) {
    pdl_wait();
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        X[slots[k]] = in[k];
}

inline int stream_blocks(int64_t n) {
    const int64_t b = (n + 255) / 256;
    return static_cast<int>(b < 148 * 16 ? b : 148 * 16);
}

}  // namespace

// ----------------------------------------------------------- launchers ------
static int env_int(const char* name, int dflt);
static int num_sms();
// Launch with the programmatic-stream-serialization attribute (SMG_PDL=0 disables):
// the kernel's launch and block scheduling overlap the previous kernel's tail.
// use_pdl = false: an ordinary launch (the kernel's griddepcontrol.wait is then a no-op).
template <typename... KArgs, typename... Args>
static void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args);
template <typename... KArgs, typename... Args>
static void launch_plain(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    note(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}
template <typename... KArgs, typename... Args>
static void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
    static const int pdl = env_int("SMG_PDL", 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    note(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}
void launch_apply(const LevelK& L, const double* x, const double* b, double* y, double gamma, cudaStream_t s) {
    if (L.cls) launch_k(k_apply_m, cell_grid(L.g), dim3(BX, BY), 0, s, L, x, b, y, gamma);
    else launch_k(k_apply, cell_grid(L.g), dim3(BX, BY), 0, s, L, x, b, y, gamma);
    count();
}
void launch_dgs_vel(const LevelK& L, double* x, const double* b, int colour, cudaStream_t s) {
    if (L.cls) k_dgs_vel_m<<<redblack_grid(L.g), dim3(BX, BY), 0, s>>>(L, x, b, colour);
    else k_dgs_vel<<<cell_grid(L.g), dim3(BX, BY), 0, s>>>(L, x, b, colour);
    count();
}
void launch_dgs_pdelta(const LevelK& L, const double* x, const double* b, double* delta, int colour,
                       cudaStream_t s) {
    if (L.cls) k_dgs_pdelta_m<<<colour_grid(L.g), dim3(BX, BY), 0, s>>>(L, x, b, delta, colour);
    else k_dgs_pdelta<<<cell_grid(L.g), dim3(BX, BY), 0, s>>>(L, x, b, delta, colour);
    count();
}
void launch_dgs_papply(const LevelK& L, double* x, const double* delta, cudaStream_t s, int colour) {
    if (L.cls) k_dgs_papply_m<<<cell_grid(L.g), dim3(BX, BY), 0, s>>>(L, x, delta, colour);
    else k_dgs_papply<<<cell_grid(L.g), dim3(BX, BY), 0, s>>>(L, x, delta);
    count();
}
void launch_dgs_cb(const LevelK& L, const double* b, cudaStream_t s) {
    if (L.bp) launch_k(k_dgs_cb<true>, cell_grid(L.g), dim3(BX, BY), 0, s, L, b, L.cb);
    else launch_k(k_dgs_cb<false>, cell_grid(L.g), dim3(BX, BY), 0, s, L, b, L.cb);
    count();
}
void launch_dgs_prev(const LevelK& L, double* x, const double* b, int colour, cudaStream_t s) {
    if (L.cls) k_dgs_prev_m<<<colour_grid(L.g), dim3(BX, BY), 0, s>>>(L, x, colour);
    else k_dgs_prev<<<cell_grid(L.g), dim3(BX, BY), 0, s>>>(L, x, b, colour);
    count();
}
void launch_vanka_delta(const LevelK& L, const double* x, const double* b, const int32_t* cells,
                        const uint8_t* masks, int ncells, const double* ktab, double* delta, cudaStream_t s,
                        const uint16_t* kidx) {
    if (ncells <= 0) return;
    // ordinary launches (no PDL): next to the tile DGS kernel early-scheduled dependents cost more
    // than they hide (SMG_VANKA_PDL=1 restores PDL; profiles/r2d_experiments.md)
    const int blocks = static_cast<int>((8 * static_cast<int64_t>(ncells) + 255) / 256);
    static const int vpdl = env_int("SMG_VANKA_PDL", 0);
    if (L.cls) {
        if (vpdl) launch_k(k_vanka_delta8<true>, blocks, 256, 0, s, L, x, b, cells, masks, kidx, ncells, ktab, delta);
        else k_vanka_delta8<true><<<blocks, 256, 0, s>>>(L, x, b, cells, masks, kidx, ncells, ktab, delta);
    } else {
        if (vpdl) launch_k(k_vanka_delta8<false>, blocks, 256, 0, s, L, x, b, cells, masks, kidx, ncells, ktab, delta);
        else k_vanka_delta8<false><<<blocks, 256, 0, s>>>(L, x, b, cells, masks, kidx, ncells, ktab, delta);
    }
    count();
}
void launch_vanka_apply(const LevelK& L, double* x, const int32_t* cells, const uint8_t* masks, int ncells,
                        const double* delta, cudaStream_t s, const uint8_t* amask) {
    if (ncells <= 0) return;
    if (!amask) {
        const int blocks = static_cast<int>((8 * static_cast<int64_t>(ncells) + 255) / 256);
        static const int vpdl = env_int("SMG_VANKA_PDL", 0);
        if (vpdl) launch_k(k_vanka_apply8, blocks, 256, 0, s, L, x, cells, masks, ncells, delta);
        else k_vanka_apply8<<<blocks, 256, 0, s>>>(L, x, cells, masks, ncells, delta);
    } else {  // z-slab parts: per-block ownership masks
        k_vanka_apply<<<(ncells + 127) / 128, 128, 0, s>>>(L, x, cells, masks, ncells, delta, amask);
    }
    count();
}
void launch_restrict(const LevelK& F, const LevelK& C, const double* rf, double* bc, cudaStream_t s, int zc_lo,
                     int nzc) {
    dim3 grid = cell_grid(C.g);
    if (F.cls) {  // labelled levels (single part): one thread per coarse cell
        launch_k(k_restrict_m, grid, dim3(BX, BY), 0, s, F, C, rf, bc);
        count();
        return;
    }
    grid.z = nzc < 0 ? C.g.nz : nzc;
    if (grid.z == 0) return;
    // z-marching variant (SMG_RESTRICT_ZM, default on) when the columns alone leave segments of
    // >= 2 coarse planes at ~one full-occupancy wave; otherwise one thread per coarse cell
    const int zm = env_int("SMG_RESTRICT_ZM", 1);
    const int64_t cols = static_cast<int64_t>(grid.x) * grid.y * BX * BY;
    const int64_t target = static_cast<int64_t>(num_sms()) * 2048;
    int nseg = static_cast<int>(std::min<int64_t>(grid.z, (target + cols - 1) / cols));
    const int force_zseg = env_int("SMG_RESTRICT_ZSEG", 0);  // tests: segment length on every level
    const int zseg = force_zseg > 0 ? force_zseg : (static_cast<int>(grid.z) + nseg - 1) / nseg;
    if (zm && zseg >= 2) {
        nseg = (static_cast<int>(grid.z) + zseg - 1) / zseg;
        launch_k(k_restrict_zm, dim3(grid.x, grid.y, nseg), dim3(BX, BY), 0, s, F, C, rf, bc, zc_lo,
                 zc_lo + static_cast<int>(grid.z), zseg);
    } else {
        launch_k(k_restrict, grid, dim3(BX, BY), 0, s, F, C, rf, bc, zc_lo);
    }
    count();
}

void launch_prolong_add(const LevelK& F, const LevelK& C, const double* xc, double* xf, cudaStream_t s) {
    if (F.cls) launch_k(k_prolong_add_m, cell_grid(F.g), dim3(BX, BY), 0, s, F, C, xc, xf);
    else launch_k(k_prolong_add, cell_grid(F.g), dim3(BX, BY), 0, s, F, C, xc, xf);
    count();
}
void launch_coarse_gemv(const double* ksym, const int32_t* slots, int n, const double* b, double* x,
                        cudaStream_t s, bool accumulate) {
    const int nchunks = (n + 63) / 64;
    const size_t smem = static_cast<size_t>(nchunks) * CG_ROWS * sizeof(double);
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_coarse_gemv, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_set = true;
    }
    launch_k(k_coarse_gemv, (n + CG_ROWS - 1) / CG_ROWS, dim3(CG_ROWS, CG_LANES), smem, s, ksym, slots, n, b, x,
             accumulate ? 1 : 0);
    count();
}
void launch_pack(const LevelK& L, const double* padded, double* compact, cudaStream_t s) {
    launch_k(k_pack, cell_grid(L.g), dim3(BX, BY), 0, s, L, padded, compact, 0);
    count();
}
void launch_unpack(const LevelK& L, const double* compact, double* padded, cudaStream_t s) {
    launch_k(k_pack, cell_grid(L.g), dim3(BX, BY), 0, s, L, padded, const_cast<double*>(compact), 1);
    count();
}
void launch_gather(const int32_t* slots, int64_t n, const double* padded, double* compact, cudaStream_t s) {
    if (n <= 0) return;
    launch_k(k_gather, dim3(stream_blocks(n)), dim3(256), 0, s, slots, n, padded, compact);
    count();
}
void launch_scatter(const int32_t* slots, int64_t n, const double* compact, double* padded, cudaStream_t s) {
    if (n <= 0) return;
    launch_k(k_scatter, dim3(stream_blocks(n)), dim3(256), 0, s, slots, n, compact, padded);
    count();
}
static dim3 dot_grid(const Geom& g) {
    return dim3((g.nx + 31) / 32, (g.ny + 7) / 8, (g.nz + kDotZB - 1) / kDotZB);
}
int64_t dot_partials(const Geom& g) { return 2 * dot_nblk(g); }
void launch_cdot_planes(const Geom& g, const double* a, const double* b, const double* c, const double* d,
                        double* partials, cudaStream_t s) {
    launch_k(k_cdot, dot_grid(g), dim3(32, 8), 0, s, g, a, b, c, d, partials);
    count();
}
void launch_cdot_final(const Geom& g, const double* partials, double* out, cudaStream_t s) {
    launch_k(k_cdot_final, 1, 256, 0, s, partials, dot_nblk(g), out);
    count();
}
void launch_cdot2(const Geom& g, const double* a, const double* b, const double* c, const double* d,
                  double* partials, double* out, cudaStream_t s) {
    launch_cdot_planes(g, a, b, c, d, partials, s);
    launch_cdot_final(g, partials, out, s);
}
void launch_final_scalar(const Geom& g, const double* partials, double* sc, int which, cudaStream_t s) {
    launch_k(k_final_scalar, 1, 256, 0, s, partials, dot_nblk(g), sc, which);
    count();
}
void launch_apply_q(const LevelK& L, const double* t, const double* q0, double* q1, double* tn, const double* sc,
                    double* partials, int halo_lo, int halo_hi, cudaStream_t s, int second) {
    // SMG_SQMR_SPLIT (default 1): the vector update as its own streaming pass, then the stencil + dot
    // kernel on the stored vector; 0: one kernel evaluating the update at every stencil point
    const int split = env_int("SMG_SQMR_SPLIT", 1);  // read per launch: tests toggle it in-process
    if (split) {
        dim3 ug = cell_grid(L.g);
        ug.z = L.g.nz + halo_lo + halo_hi;
        launch_k(k_q_upd, ug, dim3(BX, BY), 0, s, L.g, t, q0, q1, sc, halo_lo, halo_hi);
        count();
        if (L.cls) launch_k(k_apply_q<true, false>, dot_grid(L.g), dim3(32, 8), 0, s, L, t, q0, q1, tn, sc, partials, halo_lo, halo_hi, second);
        else launch_k(k_apply_q<false, false>, dot_grid(L.g), dim3(32, 8), 0, s, L, t, q0, q1, tn, sc, partials, halo_lo, halo_hi, second);
    } else if (L.cls) {
        launch_k(k_apply_q<true, true>, dot_grid(L.g), dim3(32, 8), 0, s, L, t, q0, q1, tn, sc, partials, halo_lo, halo_hi, second);
    } else {
        launch_k(k_apply_q<false, true>, dot_grid(L.g), dim3(32, 8), 0, s, L, t, q0, q1, tn, sc, partials, halo_lo, halo_hi, second);
    }
    count();
}
void launch_apply_x(const LevelK& L, const double* x0, const double* d0, const double* q, const double* b, double* x1,
                    double* d1, const double* sc, double* partials, int halo_lo, int halo_hi, cudaStream_t s) {
    const int split = env_int("SMG_SQMR_SPLIT", 1);  // read per launch: tests toggle it in-process
    if (split) {
        dim3 ug = cell_grid(L.g);
        ug.z = L.g.nz + halo_lo + halo_hi;
        launch_k(k_xd_upd, ug, dim3(BX, BY), 0, s, L.g, x0, d0, q, x1, d1, sc, halo_lo, halo_hi);
        count();
        if (L.cls) launch_k(k_apply_x<true, false>, dot_grid(L.g), dim3(32, 8), 0, s, L, x0, d0, q, b, x1, d1, sc, partials, halo_lo, halo_hi);
        else launch_k(k_apply_x<false, false>, dot_grid(L.g), dim3(32, 8), 0, s, L, x0, d0, q, b, x1, d1, sc, partials, halo_lo, halo_hi);
    } else if (L.cls) {
        launch_k(k_apply_x<true, true>, dot_grid(L.g), dim3(32, 8), 0, s, L, x0, d0, q, b, x1, d1, sc, partials, halo_lo, halo_hi);
    } else {
        launch_k(k_apply_x<false, true>, dot_grid(L.g), dim3(32, 8), 0, s, L, x0, d0, q, b, x1, d1, sc, partials, halo_lo, halo_hi);
    }
    count();
}
static int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

static int num_sms() {
    static int sms = 0;
    if (!sms) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    return sms;
}

// Co-resident block capacity of a cooperative kernel at `threads` per block.
static int64_t coop_capacity_blocks(const void* fn, int threads) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, 0);
    const int cap = env_int("SMG_COOP_BLOCKS_PER_SM", 0);  // tuning knob
    if (cap > 0 && cap < per_sm) per_sm = cap;
    return static_cast<int64_t>(num_sms()) * (per_sm > 0 ? per_sm : 0);
}

// Grid size of a cooperative launch: enough blocks for `work` threads, capped at co-residency.
static int coop_blocks(const void* fn, int64_t work, int threads) {
    const int64_t maxb = coop_capacity_blocks(fn, threads);
    const int64_t want = (work + threads - 1) / threads;
    return static_cast<int>(want < 1 ? 1 : (want < maxb ? want : maxb));
}

constexpr int kClusterCTAs = 16, kClusterThreads = 512;
// CTA size of the cooperative sweeps (tuning knob): 256 measured faster than 512 on the cfg-1
// iteration (2.43 -> 2.34 ms; fine-level Vanka sweep 0.093 -> 0.075 ms: 4 CTAs/SM instead of 2)
static int coop_threads() { return env_int("SMG_COOP_THREADS", 256) == 512 ? 512 : 256; }

// Launch either as one cooperative grid (MODE 0) or as a single cluster of
// kClusterCTAs CTAs (MODE 1) whose phases are separated by cluster barriers.
static void launch_sweep(const void* fn_grid, const void* fn_cluster, bool cluster, int64_t work, void** args,
                         cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cluster) {
        note(cudaFuncSetAttribute(fn_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        cfg.gridDim = dim3(kClusterCTAs);
        cfg.blockDim = dim3(kClusterThreads);
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = kClusterCTAs;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        note(cudaLaunchKernelExC(&cfg, fn_cluster, args));
    } else {
        // spread the work evenly: k blocks on every SM (k as small as fits), block size
        // trimmed to the per-SM share, so no SM carries twice the lanes of another
        const int bt = coop_threads();
        const int sms = num_sms();
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn_grid, bt, 0);
        const int cap = env_int("SMG_COOP_BLOCKS_PER_SM", 0);
        if (cap > 0 && cap < per_sm) per_sm = cap;
        const int64_t need = (work + sms - 1) / sms;  // threads per SM
        int k = static_cast<int>((need + bt - 1) / bt);
        int threads = bt;
        if (per_sm > 0 && k <= per_sm && env_int("SMG_EVEN_GRID", 1)) {
            k = k < 1 ? 1 : k;
            const int64_t per_block = (work + static_cast<int64_t>(sms) * k - 1) / (static_cast<int64_t>(sms) * k);
            threads = static_cast<int>((per_block + 31) / 32 * 32);
            threads = threads < 32 ? 32 : (threads > bt ? bt : threads);
            cfg.gridDim = dim3(sms * k);
        } else {
            cfg.gridDim = dim3(coop_blocks(fn_grid, work, bt));
        }
        cfg.blockDim = dim3(threads);
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        note(cudaLaunchKernelExC(&cfg, fn_grid, args));
    }
    count();
}

static void set_pairs(VankaLists& vl, const VankaPairs& pr) {
    vl.pairs = pr.pairs;
    for (int m = 0; m < 4; ++m) vl.first[m] = pr.first[m];
}
// host twin of vanka_phase_list
static int host_phase_list(const VankaPairs& pr, int k) {
    const int j = k < 8 ? k : 15 - k;
    const int p = vanka_order(j);
    return ((j & 1) && ((pr.pairs >> (7 - p)) & 1)) ? -1 : p;
}

template <int CPT>
static void launch_vanka8(bool cl, int64_t threads, void** args, cudaStream_t s) {
    launch_sweep(reinterpret_cast<const void*>(k_vanka8<0, CPT>), reinterpret_cast<const void*>(k_vanka8<1, CPT>), cl,
                 threads, args, s);
}

template <int CPT>
static void launch_vanka_pp(bool cl, int64_t threads, void** args, cudaStream_t s) {
    launch_sweep(reinterpret_cast<const void*>(k_vanka_pp<0, CPT>), reinterpret_cast<const void*>(k_vanka_pp<1, CPT>),
                 cl, threads, args, s);
}

void launch_vanka_sym_coop(const LevelK& L, double* x, const double* b, const int32_t* const* cells,
                           const uint8_t* const* masks, const int* n, const double* ktab, double* delta, int nu,
                           cudaStream_t s, double* xb, const int32_t* refresh, int64_t nrefresh,
                           const VankaPairs& pr) {
    VankaLists vl;
    set_pairs(vl, pr);
    int maxn = 1;
    for (int c = 0; c < 8; ++c) {
        vl.cells[c] = cells[c];
        vl.masks[c] = masks[c];
        vl.n[c] = n[c];
        maxn = n[c] > maxn ? n[c] : maxn;
    }
    LevelK Lc = L;
    void* args[] = {&Lc, &x, const_cast<double**>(&b), &vl, const_cast<double**>(&ktab), &nu};
    const int64_t lanes = 8 * static_cast<int64_t>(maxn);
    const int64_t cl_threads = static_cast<int64_t>(kClusterCTAs) * kClusterThreads;
    const int mode = env_int("SMG_SYNC_MODE", 0);
    // tuning knob: a cluster also takes levels needing up to SMG_CL_CPT blocks per lane group
    const bool cl = mode == 2 || (mode == 0 && lanes <= cl_threads * std::max(1, env_int("SMG_CL_CPT", 1)));
    // every block of a colour must be held in registers by some lane group:
    // threads * CPT >= lanes with threads = co-resident capacity of THAT instance
    auto fits = [&](const void* fn, int cpt) {
        const int64_t threads = cl ? cl_threads : coop_capacity_blocks(fn, coop_threads()) * coop_threads();
        return threads * cpt >= lanes;
    };
    auto refresh_xb = [&] {
        if (nrefresh <= 0) return;
        const int64_t blocks = (nrefresh + 255) / 256;
        launch_k(k_refresh, static_cast<int>(blocks < 4096 ? blocks : 4096), 256, 0, s, refresh, nrefresh, x, xb);
        count();
    };
    // ping-pong, one launch per phase: forced (SMG_VANKA_KERNELS=1), or on levels whose phases
    // fit none of the persistent sweeps below (there a kernel boundary per phase is cheap next
    // to the phase's work; SMG_VANKA_KERNELS=0 falls back to per-phase delta/apply launches)
    const int vk_kernels = env_int("SMG_VANKA_KERNELS", -1);
    auto ppk = [&] {
        refresh_xb();
        const int64_t blocks = (8 * static_cast<int64_t>(maxn) + 255) / 256;  // one lane group per block
        int ph = 0, pcol = -1;
        for (int kk = 0; kk < 16 * nu; ++kk) {
            const int c0 = host_phase_list(pr, kk & 15);
            if (c0 < 0) continue;
            const double* xc = (ph & 1) ? xb : x;
            double* xn = (ph & 1) ? x : xb;
            launch_k(k_vanka_ppk<1>, static_cast<int>(blocks), 256, 0, s, L, xc, xn, b, vl, ktab, c0, pcol);
            count();
            pcol = c0;
            ++ph;
        }
    };
    if (xb && vk_kernels == 1) { ppk(); return; }
    const bool phases = env_int("SMG_VANKA_PHASES", 0) != 0;  // 1: per-phase delta/apply launches (tests)
    bool big = false;  // the level's phases fit no persistent ping-pong sweep
    if (!phases && xb && !cl && env_int("SMG_VANKA_PP", 1)) {  // ping-pong (grid mode): one barrier per phase
        const bool rin = env_int("SMG_VANKA_REFRESH_IN", 1) != 0;
        if (!rin) refresh_xb();
        const int32_t* rl = refresh;
        int64_t rn = rin && nrefresh > 0 ? nrefresh : 0;
        void* pargs[] = {args[0], &x, &xb, args[2], args[3], args[4], args[5], &rl, &rn};
        if (fits(reinterpret_cast<const void*>(k_vanka_pp<0, 1>), 1)) {
            launch_vanka_pp<1>(cl, lanes, pargs, s);
            return;
        }
        if (fits(reinterpret_cast<const void*>(k_vanka_pp<0, 2>), 2)) {
            launch_vanka_pp<2>(cl, (lanes + 1) / 2, pargs, s);
            return;
        }
        if (fits(reinterpret_cast<const void*>(k_vanka_pp<0, 4>), 4)) {
            launch_vanka_pp<4>(cl, (lanes + 3) / 4, pargs, s);
            return;
        }
        // beyond the persistent ping-pong sweep (256^3 and up): a delta and an apply launch per merged
        // phase, 8 lanes per block.  Measured on one box (round 2, session 5; cfg 2 / cfg 3 fine
        // symmetric sweep): persistent CPT-8 sweep 0.339 ms / --, ping-pong launch per phase (ppk,
        // SMG_VANKA_KERNELS=1) 0.304 / 1.36 ms, delta + apply launches 0.245 / 1.27 ms and no
        // k_refresh of the ping-pong copy per sweep (smooth 3.14 -> 2.57 / 18.2 -> 16.5 ms)
        if (vk_kernels == 1) {
            ppk();
            return;
        }
        big = true;
    }
    bool done = !phases && !big;
    if (!done) {
    } else if (fits(reinterpret_cast<const void*>(k_vanka8<0, 1>), 1)) launch_vanka8<1>(cl, lanes, args, s);
    else if (fits(reinterpret_cast<const void*>(k_vanka8<0, 2>), 2)) launch_vanka8<2>(cl, (lanes + 1) / 2, args, s);
    else if (fits(reinterpret_cast<const void*>(k_vanka8<0, 4>), 4)) launch_vanka8<4>(cl, (lanes + 3) / 4, args, s);
    else if (fits(reinterpret_cast<const void*>(k_vanka8<0, 8>), 8)) launch_vanka8<8>(cl, (lanes + 7) / 8, args, s);
    else if (xb && vk_kernels != 0) { ppk(); return; }
    else done = false;
    if (!done) {
        for (int sweep = 0; sweep < nu; ++sweep)
            for (int k = 0; k < 16; ++k) {
                const int col = host_phase_list(pr, k);
                if (col < 0) continue;  // folded into the list of its complementary colour
                launch_vanka_delta(L, x, b, cells[col], masks[col], n[col], ktab, delta, s);
                launch_vanka_apply(L, x, cells[col], masks[col], n[col], delta, s);
            }
    }
}

// Merging a complementary pair halves the dependent phases and doubles each phase's lanes.
// Mask of the pairs to merge: SMG_VANKA_PAIRS = 0 none, 2 all, 1 (default) all unless the
// merged phases would leave the persistent ping-pong sweep (> 2 blocks per lane group) while
// the unmerged ones still fit it at 1 block per lane group.  Levels beyond the persistent
// sweep run one kernel per phase, where merging always pays (half the launches, same work).
int vanka_pairs_pay(const int* n) {
    const int mode = env_int("SMG_VANKA_PAIRS", 1);
    if (mode == 0) return 0;
    if (mode == 2) return 0xf;
    int maxn = 0, maxm = 0;
    for (int c = 0; c < 8; ++c) maxn = n[c] > maxn ? n[c] : maxn;
    for (int m = 0; m < 4; ++m) maxm = n[m] + n[7 - m] > maxm ? n[m] + n[7 - m] : maxm;
    const int64_t cap = coop_capacity_blocks(reinterpret_cast<const void*>(k_vanka_pp<0, 2>), coop_threads()) *
                        coop_threads();
    const int64_t cl = static_cast<int64_t>(kClusterCTAs) * kClusterThreads;
    const int64_t lm = 8 * static_cast<int64_t>(maxm), lu = 8 * static_cast<int64_t>(maxn);
    const bool merged_fits = lm <= cl || lm <= 2 * cap;
    const bool unmerged_cpt1 = lu <= cl || lu <= cap;
    return (merged_fits || !unmerged_cpt1) ? 0xf : 0;
}

// Single phases of the colour-compact DGS (the z-slab path exchanges halos between them).
static dim3 dgs_grid_v(const Geom& g) { return dim3((((g.nx + 1) / 2) + 31) / 32, (g.ny + 7) / 8, g.nz); }
static dim3 dgs_grid_h(const Geom& g) {
    return dim3((((g.nx + 1) / 2) + 31) / 32, (((g.ny + 1) / 2) + 7) / 8, (g.nz + 1) / 2);
}
void launch_dgs_vel_c(const LevelK& L, double* x, const double* b, int colour, cudaStream_t s) {
    launch_k(k_dgs_vel_c<1>, dgs_grid_v(L.g), dim3(32, 8), 0, s, L, x, b, colour);
    count();
}
void launch_dgs_pf_delta_c(const LevelK& L, const double* x, const double* b, double* d, int c, cudaStream_t s) {
    k_dgs_pf_delta_c<<<dgs_grid_h(L.g), dim3(32, 8), 0, s>>>(L, x, b, d, c);
    count();
}
void launch_dgs_pf_apply_c(const LevelK& L, double* x, const double* d, int c, cudaStream_t s) {
    k_dgs_pf_apply_c<<<dgs_grid_h(L.g), dim3(32, 8), 0, s>>>(L, x, d, c);
    count();
}
void launch_dgs_prev_c(const LevelK& L, double* x, const double* b, int c, cudaStream_t s) {
    launch_k(k_dgs_prev_c<1>, dgs_grid_h(L.g), dim3(32, 8), 0, s, L, x, b, colour_group(c, 0, 0, 1));
    count();
}


// Per-step launches of a symmetric DGS sweep (OD-1): velocity red, black, the 4 forward
// pressure groups (lazy gathers into the delta buffer d0), the flush, then the 4 reverse
// pressure groups and velocity black, red -- 13 kernels for the 20 phases.
void launch_dgs_sym_coop(const LevelK& L, double* x, const double* b, double* d0, double* d1, int nph,
                         cudaStream_t s, double* xb) {
    (void)d1;
    (void)xb;
    const Geom& g = L.g;
    const dim3 blk(32, 8);
    const dim3 gv = dgs_grid_v(g), gh = dgs_grid_h(g);
    auto groups_grid = [&](int grp) { return dim3(gh.x, gh.y, gh.z * group_size(grp)); };
    // consecutive steps alternate the traversal direction (kRevBit): L2 reuse between steps
    const int alt = env_int("SMG_DGS_ALT", 1) ? kRevBit : 0;
    launch_k(k_dgs_vel_c<1>, gv, blk, 0, s, L, x, b, 0);
    launch_k(k_dgs_vel_c<1>, gv, blk, 0, s, L, x, b, 1 | alt);
    for (int q = 0; q < 4; ++q)
        launch_k(k_dgs_pf_lazy_c<1>, groups_grid(fwd_group(q)), blk, 0, s, L, x, b, d0, fwd_group(q) | (q & 1 ? alt : 0));
    launch_k(k_dgs_pf_flush, cell_grid(g), blk, 0, s, L, x, d0, 0);
    for (int k = 0; k < 7; ++k) count();
    if (nph <= 10) return;
    for (int q = 0; q < 4; ++q)
        launch_k(k_dgs_prev_c<1>, groups_grid(rev_group(q)), blk, 0, s, L, x, b, rev_group(q) | (q & 1 ? 0 : alt));
    launch_k(k_dgs_vel_c<1>, gv, blk, 0, s, L, x, b, 1 | alt);
    launch_k(k_dgs_vel_c<1>, gv, blk, 0, s, L, x, b, 0);
    for (int k = 0; k < 6; ++k) count();
}


// ---- tile-ordered DGS sweep (OD-1 rev. 2) ----
typedef CUresult (*TmapEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static TmapEncodeFn tmap_encode() {
    static TmapEncodeFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<TmapEncodeFn>(p);
    }
    return fn;
}

bool dgs_tiled(int nx, int ny, int nz, int64_t tile_min) {
    if (tile_min == 0) tile_min = int64_t{1} << 24;  // 256^3 (the oracle's kTileMinDefault)
    if (tile_min < 0) return false;
    if (static_cast<int64_t>(nx) * ny * nz < tile_min) return false;
    return nx % kTX == 0 && ny % kTY == 0 && nz % kTZ == 0 && nx / kTX >= 2 && ny / kTY >= 2 && nz / kTZ >= 2;
}
int dgs_tile_dim(int axis) { return axis == 0 ? kTX : (axis == 1 ? kTY : kTZ); }

// 4-D tensor map (x, y, z slots of the padded boxes, nf fields) of a level vector with box
// (bx, by, bz, nf); OOB coordinates (beyond the ghost ring) read as 0.
static bool level_tmap(const Geom& g, const double* x, int nf, int bx, int by, int bz, CUtensorMap* m) {
    TmapEncodeFn enc = tmap_encode();
    if (!enc) return false;
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(g.px), static_cast<cuuint64_t>(g.py),
                                static_cast<cuuint64_t>(g.pz), static_cast<cuuint64_t>(nf)};
    const cuuint64_t strides[3] = {static_cast<cuuint64_t>(g.sy) * 8, static_cast<cuuint64_t>(g.sz) * 8,
                                   static_cast<cuuint64_t>(g.fs) * 8};
    const cuuint32_t box[4] = {static_cast<cuuint32_t>(bx), static_cast<cuuint32_t>(by), static_cast<cuuint32_t>(bz),
                               static_cast<cuuint32_t>(nf)};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(x), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Phases [ph0, ph1) on the tiles of colour T (a range within one half: 0..9 or 10..19).
// zsel: 0 = every tile layer of the part; 1 = only the part's bottom and top tile layers (the tiles
// whose updates reach the 2 planes a halo exchange sends and the ghost planes a push reads);
// 2 = only the layers in between (they touch nothing a halo transfer reads or writes: z-slab
// parts run them while the transfer is in flight on the comm stream).
// packed: L.bp holds this b (launch_dgs_cb ran on it): the tiles stage b / c_b from there.
void launch_dgs_tile_phases(const LevelK& L, double* x, const double* b, int T, int ph0, int ph1, cudaStream_t s,
                            int zsel, bool packed) {
    const Geom& g = L.g;
    const int ntx = g.nx / kTX, nty = g.ny / kTY, ntz = g.nz / kTZ;
    const int pz = ((T >> 2) ^ (g.z0 / kTZ)) & 1;
    const int hx = (ntx - (T & 1) + 1) >> 1, hy = (nty - ((T >> 1) & 1) + 1) >> 1;
    int hz = (ntz - pz + 1) >> 1;  // layers of this colour: tz = pz, pz + 2, ...
    if (hx * hy * hz == 0 || ph1 <= ph0) return;
    const bool fwd = ph1 <= 10;
    if (!fwd && ph0 < 10) {  // split at the half boundary
        launch_dgs_tile_phases(L, x, b, T, ph0, 10, s, zsel, packed);
        launch_dgs_tile_phases(L, x, b, T, 10, ph1, s, zsel, packed);
        return;
    }
    int kz0 = 0, kzs = 1;
    if (zsel != 0) {
        const bool bot = pz == 0, top = hz > (bot ? 1 : 0) && ((ntz - 1 - pz) & 1) == 0;  // top != bottom layer
        if (zsel == 1) {
            kz0 = bot ? 0 : hz - 1;
            kzs = hz > 1 ? hz - 1 : 1;
            hz = (bot ? 1 : 0) + (top ? 1 : 0);
        } else {
            kz0 = bot ? 1 : 0;
            hz -= (bot ? 1 : 0) + (top ? 1 : 0);
        }
        if (hz <= 0) return;
    }
    CUtensorMap mx, mb, mc;
    bool ok;
    if (fwd) {
        using TB = TileBox<true>;
        ok = level_tmap(g, x, 4, kBX, TB::BY, TB::BZ, &mx) && level_tmap(g, b, 4, kTX, kTY, kTZ, &mb);
        mc = mb;
    } else {
        using TB = TileBox<false>;
        ok = level_tmap(g, x, 4, kBX, TB::BY, TB::BZ, &mx) && level_tmap(g, b, 3, kTX, kTY, kTZ, &mb) &&
             level_tmap(g, L.cb, 1, kTX, kTY, kTZ, &mc);
    }
    if (!ok) {
        note(cudaErrorNotSupported);
        return;
    }
    static bool attr = false;
    if (!attr) {
        note(cudaFuncSetAttribute(k_dgs_tile<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(TileBox<true>::SMEM)));
        note(cudaFuncSetAttribute(k_dgs_tile<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(TileBox<false>::SMEM)));
        attr = true;
    }
    // SMG_TILE_PF: L2 prefetch distance in CTAs (0 = off, the default: measured 2.19 (off) / 2.16 (148) /
    // 2.30 (296) / 2.40 ms (592) per cfg-2 fine sweep -- the loads are not latency-exposed)
    static const int pf0 = env_int("SMG_TILE_PF", 0);
    // SMG_TILE_ALT (default 1): consecutive launches of a sweep alternate their traversal direction
    static const int alt = env_int("SMG_TILE_ALT", 1);
    const int seq = fwd ? T : 15 - T;  // position of this launch in the symmetric sweep
    const int pf = (alt && (seq & 1)) ? -1 : pf0;
    // Ordinary launches (SMG_TILE_PDL=1 restores programmatic dependent launch): with PDL the next
    // colour's CTAs take the SM's shared memory slots early and the cfg-2 fine sweep measured
    // 2.185 ms against 2.04 ms without (round 2, session 5)
    static const int tile_pdl = env_int("SMG_TILE_PDL", 0);
    // SMG_TILE_BPACK=0: stage b from the level vector even when the packed copy is valid (A/B, tests)
    const char* bpe = std::getenv("SMG_TILE_BPACK");
    const double* bpk = (packed && L.bp && !(bpe && std::atoi(bpe) == 0)) ? L.bp : nullptr;
    if (fwd && tile_pdl)
        launch_k(k_dgs_tile<true>, dim3(hx * hy * hz), dim3(kTileThreads), TileBox<true>::SMEM, s, mx, mb, mc, L, x, T,
                 ph0, ph1, ntx, nty, pf, kz0, kzs, bpk);
    else if (fwd)
        launch_plain(k_dgs_tile<true>, dim3(hx * hy * hz), dim3(kTileThreads), TileBox<true>::SMEM, s, mx, mb, mc, L, x,
                     T, ph0, ph1, ntx, nty, pf, kz0, kzs, bpk);
    else if (tile_pdl)
        launch_k(k_dgs_tile<false>, dim3(hx * hy * hz), dim3(kTileThreads), TileBox<false>::SMEM, s, mx, mb, mc, L, x,
                 T, ph0, ph1, ntx, nty, pf, kz0, kzs, bpk);
    else
        launch_plain(k_dgs_tile<false>, dim3(hx * hy * hz), dim3(kTileThreads), TileBox<false>::SMEM, s, mx, mb, mc, L,
                     x, T, ph0, ph1, ntx, nty, pf, kz0, kzs, bpk);
    count();
}

// Symmetric sweep (nph = 20) or its forward half (nph = 10): tile colours 0..7 forward, then
// 7..0 reverse (16 launches; the two halves use different kernel variants).
void launch_dgs_tiled(const LevelK& L, double* x, const double* b, int nph, cudaStream_t s, bool packed) {
    for (int T = 0; T < 8; ++T) launch_dgs_tile_phases(L, x, b, T, 0, 10, s, 0, packed);
    if (nph <= 10) return;
    for (int T = 7; T >= 0; --T) launch_dgs_tile_phases(L, x, b, T, 10, 20, s, 0, packed);
}

void launch_vanka_additive(const LevelK& L, double* x, const double* b, const int32_t* cells, const uint8_t* masks,
                           int n, const double* ktab, double* d7, double omega, cudaStream_t s, const uint16_t* kidx) {
    if (n <= 0) return;
    const dim3 gd(static_cast<unsigned>((8 * static_cast<int64_t>(n) + 255) / 256)), ga(static_cast<unsigned>((n + 255) / 256));
    if (L.cls) {
        launch_k(k_vadd_delta<true>, gd, dim3(256), 0, s, L, x, b, cells, masks, kidx, n, ktab, d7);
        launch_k(k_vadd_apply<true>, ga, dim3(256), 0, s, L, x, cells, masks, n, d7, omega);
    } else {
        launch_k(k_vadd_delta<false>, gd, dim3(256), 0, s, L, x, b, cells, masks, kidx, n, ktab, d7);
        launch_k(k_vadd_apply<false>, ga, dim3(256), 0, s, L, x, cells, masks, n, d7, omega);
    }
    count();
    count();
}

void launch_axpy_s(double* s_, const double* t, const double* sc, int64_t n, cudaStream_t s) {
    launch_k(k_axpy_s, stream_blocks(n), 256, 0, s, s_, t, sc, n);
    count();
}
// Frames of the padded plane pairs zs0, zs0 + 1 and zs1, zs1 + 1 (all four fields) of a slab vector <->
// two contiguous buffers of frame_doubles(g, bw) doubles each (z-slab halo refresh after a Vanka phase);
// a null buffer skips its pair.
int64_t frame_doubles(const Geom& g, int bw) { return 8 * frame_dims(g, bw).count(); }
void launch_frame_copy(const Geom& g, int bw, double* x, double* buf0, int zs0, double* buf1, int zs1, bool to_buf,
                       cudaStream_t s) {
    if (!buf0 && !buf1) return;
    const FrameDims f = frame_dims(g, bw);
    const dim3 grid(static_cast<unsigned>((f.count() + 255) / 256), 8, 2);  // both plane pairs in one launch
    k_frame_copy<<<grid, 256, 0, s>>>(g, f, x, buf0, zs0, buf1, zs1, to_buf ? 1 : 0);
    count();
}
void launch_axpy(double* y, const double* x, double alpha, int64_t n, cudaStream_t s) {
    k_axpy<<<stream_blocks(n), 256, 0, s>>>(y, x, alpha, n);
    count();
}
void launch_xpby(double* y, const double* x, double beta, int64_t n, cudaStream_t s) {
    k_xpby<<<stream_blocks(n), 256, 0, s>>>(y, x, beta, n);
    count();
}
void launch_dx_update(double* d, double* x, const double* q, double cd, double cq, int64_t n, cudaStream_t s) {
    k_dx_update<<<stream_blocks(n), 256, 0, s>>>(d, x, q, cd, cq, n);
    count();
}

}  // namespace smg

#ifdef SMG_TRACE
extern "C" int smg_trace_enable(long long n) {
    unsigned long long* p = nullptr;
    if (cudaMalloc(&p, n * sizeof(unsigned long long)) != cudaSuccess) return -1;
    cudaMemset(p, 0, n * sizeof(unsigned long long));
    return cudaMemcpyToSymbol(smg::g_trace, &p, sizeof(p)) == cudaSuccess ? 0 : -1;
}
extern "C" int smg_trace_read(unsigned long long* host, long long n) {
    unsigned long long* p = nullptr;
    cudaMemcpyFromSymbol(&p, smg::g_trace, sizeof(p));
    return cudaMemcpy(host, p, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : -1;
}
#endif
