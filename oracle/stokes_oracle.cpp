// =============================================================================
// oracle/stokes_oracle.cpp — TEST INFRASTRUCTURE ONLY.
//
// CPU fp64 restatement of the reference's MG-preconditioned SQMR Stokes path
// (arXiv 2312.10615).  The reference ships no solver code: this file
// restates SPEC.md (modules domain, discretization, transfer, smoothers,
// multigrid, krylov) and PAPER.md (Alg. 1-4, App. A-D), fixing every point the
// reference leaves open as recorded in DESIGN.md §"Open decisions" (OD-1..OD-12
// of SURVEY §8).  It is the parity checker for the CUDA path and the CPU
// baseline ("port") — it is never linked into, or called by, the product.
//
// Independence from the product: the oracle works on the SPEC's compact
// FieldVector (active DOFs numbered u-lex, v-lex, w-lex, p-lex)
// over a generic labelled CellGrid with neighbour tables, whereas the GPU works
// on padded SoA boxes with analytic indexing.  Per-point arithmetic follows the
// arithmetic contract in DESIGN.md §4 so results can be compared bit-for-bit
// (compile with -ffp-contract=off; the GPU side uses -fmad=false).
//
// Parity pins ("parity unpinned" by the reference for residual histories: no reference artifact
// pins them; the committed goldens are self-pinned):
//   * Table-1 DOF census, exact — tests/test_oracle_census.py
//   * structural KATs of SPEC AC 3-6, 8, 9, 11, 12, on the walled box and on labelled domains with
//     obstacles and Exterior cells — tests/test_oracle_*.py, tests/test_labeled_host.py
//   * dense / sparse direct solves at small sizes — tests/test_oracle_direct.py, test_labeled_host.py
//   * the reference's only compiled code, util.hpp (which this file includes through the drop-in
//     header), against the reference's own header — tests/golden/util_probe_reference.txt
// =============================================================================
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../include/stokesmg/util.hpp"

namespace orc {

using stokesmg::parallel_for;
using vec = std::vector<double>;

// ---------------------------------------------------------------- domain ----
// CellLabel.  Cells outside the labelled box are an implicit
// Dirichlet ring (OD-5).
enum : uint8_t { LAB_D = 0, LAB_I = 1, LAB_E = 2 };

struct CellGrid {
    int dim = 3;
    int n[3] = {1, 1, 1};
    double h = 1.0;
    std::vector<uint8_t> lab;  // row-major, x fastest (OD-10)
    uint8_t at(int x, int y, int z) const {
        if (x < 0 || y < 0 || z < 0 || x >= n[0] || y >= n[1] || z >= n[2]) return LAB_D;
        return lab[(static_cast<size_t>(z) * n[1] + y) * n[0] + x];
    }
};

// coarsen_grid: coarse label D if any child D, else I if any
// child I, else E.  Odd extents are padded with E.
static CellGrid coarsen(const CellGrid& f) {
    CellGrid c;
    c.dim = f.dim;
    for (int a = 0; a < 3; ++a) c.n[a] = (a < f.dim) ? (f.n[a] + 1) / 2 : 1;
    for (int a = 0; a < f.dim; ++a)
        if (f.n[a] < 2) throw std::runtime_error("coarsen: extent 1");
    c.h = 2.0 * f.h;
    c.lab.assign(static_cast<size_t>(c.n[0]) * c.n[1] * c.n[2], LAB_E);
    const int dz = f.dim == 3 ? 2 : 1;
    for (int z = 0; z < c.n[2]; ++z)
        for (int y = 0; y < c.n[1]; ++y)
            for (int x = 0; x < c.n[0]; ++x) {
                bool anyD = false, anyI = false;
                for (int k = 0; k < dz; ++k)
                    for (int j = 0; j < 2; ++j)
                        for (int i = 0; i < 2; ++i) {
                            const int fx = 2 * x + i, fy = 2 * y + j, fz = dz * z + k;
                            if (fx >= f.n[0] || fy >= f.n[1] || fz >= f.n[2]) continue;  // E pad
                            const uint8_t l = f.at(fx, fy, fz);
                            anyD |= (l == LAB_D);
                            anyI |= (l == LAB_I);
                        }
                c.lab[(static_cast<size_t>(z) * c.n[1] + y) * c.n[0] + x] =
                    anyD ? LAB_D : (anyI ? LAB_I : LAB_E);
            }
    return c;
}

// Status codes of a face/cell in the DofMap.
constexpr int32_t ST_DIRICHLET = -1;
constexpr int32_t ST_INACTIVE = -2;

// classify_dofs + partition_band.
struct DofMap {
    int dim = 3;
    int n[3] = {1, 1, 1};
    // face index arrays per component c: extents n[a] + (a == c), x fastest
    std::vector<int32_t> fid[3];
    int fext[3][3] = {};
    std::vector<int32_t> cid;  // per cell: active index or status
    int64_t N = 0;
    int64_t off[4] = {0, 0, 0, 0}, cnt[4] = {0, 0, 0, 0};
    std::vector<uint8_t> band_cell;  // per cell
    std::vector<uint8_t> v1;         // per active DOF
    std::vector<int32_t> comp;       // per active DOF: 0..2 velocity, 3 pressure
    std::vector<std::array<int32_t, 3>> pos;  // storage coordinates per active DOF

    int32_t face(int c, int x, int y, int z) const {
        if (x < 0 || y < 0 || z < 0 || x >= fext[c][0] || y >= fext[c][1] || z >= fext[c][2])
            return ST_DIRICHLET;  // faces of ring cells: Dirichlet
        return fid[c][(static_cast<size_t>(z) * fext[c][1] + y) * fext[c][0] + x];
    }
    int32_t cell(int x, int y, int z) const {
        if (x < 0 || y < 0 || z < 0 || x >= n[0] || y >= n[1] || z >= n[2]) return ST_INACTIVE;
        return cid[(static_cast<size_t>(z) * n[1] + y) * n[0] + x];
    }
    bool is_band(int x, int y, int z) const {
        return band_cell[(static_cast<size_t>(z) * n[1] + y) * n[0] + x] != 0;
    }
};

static DofMap classify(const CellGrid& g, int band_width) {
    DofMap m;
    m.dim = g.dim;
    for (int a = 0; a < 3; ++a) m.n[a] = g.n[a];
    const int nc = g.dim;  // velocity components
    int64_t next = 0;
    for (int c = 0; c < 3; ++c) {
        for (int a = 0; a < 3; ++a) m.fext[c][a] = g.n[a] + ((a == c && c < nc) ? 1 : 0);
        m.off[c] = next;
        if (c >= nc) { m.cnt[c] = 0; continue; }
        const size_t sz = static_cast<size_t>(m.fext[c][0]) * m.fext[c][1] * m.fext[c][2];
        m.fid[c].assign(sz, ST_INACTIVE);
        for (int z = 0; z < m.fext[c][2]; ++z)
            for (int y = 0; y < m.fext[c][1]; ++y)
                for (int x = 0; x < m.fext[c][0]; ++x) {
                    // face (x,y,z) of component c lies between cell (x,y,z)-e_c and (x,y,z)
                    int lx = x, ly = y, lz = z;
                    if (c == 0) lx -= 1;
                    if (c == 1) ly -= 1;
                    if (c == 2) lz -= 1;
                    const uint8_t a = g.at(lx, ly, lz), b = g.at(x, y, z);
                    int32_t st;
                    if (a == LAB_D || b == LAB_D) st = ST_DIRICHLET;
                    else if (a == LAB_I && b == LAB_I) st = static_cast<int32_t>(next++);
                    else st = ST_INACTIVE;
                    m.fid[c][(static_cast<size_t>(z) * m.fext[c][1] + y) * m.fext[c][0] + x] = st;
                }
        m.cnt[c] = next - m.off[c];
    }
    m.off[3] = next;
    const size_t ncell = static_cast<size_t>(g.n[0]) * g.n[1] * g.n[2];
    m.cid.assign(ncell, ST_INACTIVE);
    for (size_t q = 0; q < ncell; ++q)
        if (g.lab[q] == LAB_I) m.cid[q] = static_cast<int32_t>(next++);
    m.cnt[3] = next - m.off[3];
    m.N = next;

    // partition_band: Chebyshev distance <= width to any non-Interior cell
    m.band_cell.assign(ncell, 0);
    const int wz = g.dim == 3 ? band_width : 0;
    for (int z = 0; z < g.n[2]; ++z)
        for (int y = 0; y < g.n[1]; ++y)
            for (int x = 0; x < g.n[0]; ++x) {
                bool band = false;
                for (int k = -wz; k <= wz && !band; ++k)
                    for (int j = -band_width; j <= band_width && !band; ++j)
                        for (int i = -band_width; i <= band_width && !band; ++i)
                            if (g.at(x + i, y + j, z + k) != LAB_I) band = true;
                m.band_cell[(static_cast<size_t>(z) * g.n[1] + y) * g.n[0] + x] = band;
            }

    // per-DOF component, storage coordinates and V1 membership
    m.comp.assign(m.N, 0);
    m.pos.assign(m.N, {0, 0, 0});
    m.v1.assign(m.N, 0);
    for (int c = 0; c < nc; ++c)
        for (int z = 0; z < m.fext[c][2]; ++z)
            for (int y = 0; y < m.fext[c][1]; ++y)
                for (int x = 0; x < m.fext[c][0]; ++x) {
                    const int32_t id = m.face(c, x, y, z);
                    if (id < 0) continue;
                    m.comp[id] = c;
                    m.pos[id] = {x, y, z};
                    int lx = x, ly = y, lz = z;
                    if (c == 0) lx -= 1;
                    if (c == 1) ly -= 1;
                    if (c == 2) lz -= 1;
                    // V1 = active DOFs on faces of band cells
                    m.v1[id] = (m.is_band(lx, ly, lz) || m.is_band(x, y, z)) ? 1 : 0;
                }
    for (int z = 0; z < g.n[2]; ++z)
        for (int y = 0; y < g.n[1]; ++y)
            for (int x = 0; x < g.n[0]; ++x) {
                const int32_t id = m.cell(x, y, z);
                if (id < 0) continue;
                m.comp[id] = 3;
                m.pos[id] = {x, y, z};
                m.v1[id] = m.is_band(x, y, z) ? 1 : 0;
            }
    return m;
}

// ------------------------------------------------------ discretization ------
// One multigrid level: LevelOperator with the neighbour tables
// the matrix-free apply needs.  3-D only (every BASELINE config is 3-D).
struct Level {
    CellGrid grid;
    DofMap map;
    double h = 1, eta = 1, gamma = 0;
    double eta_h2 = 1, inv_h = 1, dv = 6, dp = -6;
    // velocity DOF: [x-, x+, y-, y+, z-, z+] same-component neighbours, then
    // [p_left, p_right]; entries < 0 contribute value 0 (Dirichlet).
    std::vector<std::array<int32_t, 8>> vnb;
    std::vector<double> vdiag;  // neighbour-leg count (6 in the cube; SPEC:124 drops Neumann legs)
    // pressure DOF: faces [uL, uR, vL, vR, wL, wR] and neighbour cells [x-, x+, y-, y+, z-, z+]
    std::vector<std::array<int32_t, 6>> pface, pcell;
    // DGS sets (V2) by DGS tile colour T (OD-1 rev. 2): large levels are cut
    // into tiles of kTile cells whose parity colour (tx&1)+2(ty&1)+4(tz&1) orders the sweep
    // (forward: T = 0..7, each tile's DOFs in the in-tile order; reverse: T = 7..0, each in
    // the exact reverse in-tile order); small levels are one tile (ntc = 1).  In a tile:
    // velocities by red-black parity, pressures by the 8 parity colours (i&1)+2(j&1)+4(k&1).
    int ntc = 1;
    int tile[3] = {0, 0, 0};
    std::vector<int32_t> dgs_vel[8][2], dgs_p[8][8];
    // every active pressure by parity colour (targets of the distributive pressure update)
    std::vector<int32_t> all_p[8];
    // SPEC-literal order (Hierarchy::order = 1): V2 DOFs ascending
    std::vector<int32_t> v2_lex;
    // Vanka blocks (band cells with an active pressure), by colour (OD-2)
    struct Block { std::array<int32_t, 7> dof; int mask; };
    std::vector<Block> vk[8];
    std::vector<Block> vk_all;  // every block, ascending cell index (additive Vanka's summation order)
    // factorisation cache keyed by the block's signature class ("keyed by neighbor-label
    // signature"): the active-face mask (bits 0-5) and, per active face, its dropped Neumann legs
    // 6 - vdiag (3 bits each from bit 6) -- everything the local matrix depends on
    std::map<int, std::array<double, 49>> vk_inv;
    // face -> (left cell, right cell) pressure ids, for the distributive update
    std::vector<std::array<int32_t, 2>> fcells;
    // direct-on-V1 mode: the V1 DOFs ascending and, built on first use, the exactly
    // symmetrised dense inverse of the V1 x V1 principal sub-block of L~
    std::vector<int32_t> v1_ids;
    mutable std::vector<double> v1_inv;
};

static inline double val(const vec& x, int32_t id) { return id >= 0 ? x[id] : 0.0; }

// L̃ x at one velocity DOF (arithmetic contract).
static inline double mom_row(const Level& L, const vec& x, int32_t f) {
    const auto& nb = L.vnb[f];
    double s = val(x, nb[0]) + val(x, nb[1]);
    s = s + val(x, nb[2]);
    s = s + val(x, nb[3]);
    s = s + val(x, nb[4]);
    s = s + val(x, nb[5]);
    const double lap = L.vdiag[f] * x[f] - s;
    return L.eta_h2 * lap + (val(x, nb[7]) - val(x, nb[6])) * L.inv_h;
}
// L̃ x at one pressure DOF: -(div u)/h - gamma p.
static inline double cont_row(const Level& L, const vec& x, int32_t c, double gamma) {
    const auto& fc = L.pface[c];
    const double div = (val(x, fc[1]) - val(x, fc[0])) + (val(x, fc[3]) - val(x, fc[2])) +
                       (val(x, fc[5]) - val(x, fc[4]));
    return -div * L.inv_h - gamma * x[c];
}

static int g_threads = 1;

// apply: y = L x (penalized = 0) or L̃ x (penalized = 1).
static void apply(const Level& L, const vec& x, vec& y, bool penalized) {
    const double gam = penalized ? L.gamma : 0.0;
    y.assign(L.map.N, 0.0);
    const int64_t nv = L.map.off[3];
    parallel_for(g_threads, g_threads, [&](int64_t t) {
        const int64_t lo = L.map.N * t / g_threads, hi = L.map.N * (t + 1) / g_threads;
        for (int64_t q = lo; q < hi; ++q)
            y[q] = (q < nv) ? mom_row(L, x, static_cast<int32_t>(q))
                            : cont_row(L, x, static_cast<int32_t>(q), gam);
    });
}

static void residual(const Level& L, const vec& x, const vec& b, vec& r) {
    const int64_t nv = L.map.off[3];
    r.assign(L.map.N, 0.0);
    parallel_for(g_threads, g_threads, [&](int64_t t) {
        const int64_t lo = L.map.N * t / g_threads, hi = L.map.N * (t + 1) / g_threads;
        for (int64_t q = lo; q < hi; ++q)
            r[q] = b[q] - ((q < nv) ? mom_row(L, x, static_cast<int32_t>(q))
                                    : cont_row(L, x, static_cast<int32_t>(q), L.gamma));
    });
}

// Sparse row of L̃ (used for dense assembly and the Vanka local matrices).
static void ltilde_row(const Level& L, int32_t r, std::vector<std::pair<int32_t, double>>& out) {
    out.clear();
    if (r < L.map.off[3]) {
        const auto& nb = L.vnb[r];
        out.push_back({r, L.vdiag[r] * L.eta_h2});
        for (int k = 0; k < 6; ++k)
            if (nb[k] >= 0) out.push_back({nb[k], -L.eta_h2});
        if (nb[6] >= 0) out.push_back({nb[6], -L.inv_h});
        if (nb[7] >= 0) out.push_back({nb[7], L.inv_h});
    } else {
        const auto& fc = L.pface[r];
        for (int a = 0; a < 3; ++a) {
            if (fc[2 * a] >= 0) out.push_back({fc[2 * a], L.inv_h});        // left face: +1/h
            if (fc[2 * a + 1] >= 0) out.push_back({fc[2 * a + 1], -L.inv_h});  // right face
        }
        out.push_back({r, -L.gamma});
    }
}

// ------------------------------------------------------- dense helpers ------
// LU with partial pivoting, then the explicit inverse column by column, then
// exact symmetrisation (OD-4).  Row-major n x n.
static std::vector<double> dense_inverse_sym(std::vector<double> a, int n, int threads) {
    std::vector<int> piv(n);
    for (int k = 0; k < n; ++k) {
        int p = k;
        double best = std::fabs(a[static_cast<size_t>(k) * n + k]);
        for (int i = k + 1; i < n; ++i) {
            const double v = std::fabs(a[static_cast<size_t>(i) * n + k]);
            if (v > best) { best = v; p = i; }
        }
        if (best == 0.0) throw std::runtime_error("dense LU: singular matrix");
        piv[k] = p;
        if (p != k)
            for (int j = 0; j < n; ++j) std::swap(a[static_cast<size_t>(k) * n + j], a[static_cast<size_t>(p) * n + j]);
        const double d = a[static_cast<size_t>(k) * n + k];
        parallel_for(n - k - 1, threads, [&](int64_t t) {
            const int i = k + 1 + static_cast<int>(t);
            double* ri = &a[static_cast<size_t>(i) * n];
            const double* rk = &a[static_cast<size_t>(k) * n];
            const double m = ri[k] / d;
            ri[k] = m;
            if (m != 0.0)
                for (int j = k + 1; j < n; ++j) ri[j] = ri[j] - m * rk[j];
        });
    }
    std::vector<double> inv(static_cast<size_t>(n) * n, 0.0);  // column-major solve results
    parallel_for(n, threads, [&](int64_t col) {
        std::vector<double> y(n, 0.0);
        y[col] = 1.0;
        // apply the row permutation to e_col
        for (int k = 0; k < n; ++k)
            if (piv[k] != k) std::swap(y[k], y[piv[k]]);
        for (int i = 0; i < n; ++i) {  // forward (unit lower)
            double s = y[i];
            const double* ri = &a[static_cast<size_t>(i) * n];
            for (int j = 0; j < i; ++j) s = s - ri[j] * y[j];
            y[i] = s;
        }
        for (int i = n - 1; i >= 0; --i) {  // backward
            double s = y[i];
            const double* ri = &a[static_cast<size_t>(i) * n];
            for (int j = i + 1; j < n; ++j) s = s - ri[j] * y[j];
            y[i] = s / ri[i];
        }
        for (int i = 0; i < n; ++i) inv[static_cast<size_t>(col) * n + i] = y[i];  // inv[col][i] = (A^-1)_{i,col}
    });
    // symmetrise: K_ij = 0.5 * ((A^-1)_ij + (A^-1)_ji)
    std::vector<double> k(static_cast<size_t>(n) * n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            k[static_cast<size_t>(i) * n + j] =
                0.5 * (inv[static_cast<size_t>(j) * n + i] + inv[static_cast<size_t>(i) * n + j]);
    return k;
}

// Small dense inverse (Gauss-Jordan with partial pivoting) for Vanka blocks.
static std::array<double, 49> small_inverse(const std::vector<double>& m, int n) {
    std::vector<double> a(m), e(static_cast<size_t>(n) * n, 0.0);
    for (int i = 0; i < n; ++i) e[i * n + i] = 1.0;
    for (int k = 0; k < n; ++k) {
        int p = k;
        double best = std::fabs(a[k * n + k]);
        for (int i = k + 1; i < n; ++i)
            if (std::fabs(a[i * n + k]) > best) { best = std::fabs(a[i * n + k]); p = i; }
        if (best == 0.0) throw std::runtime_error("vanka: singular local matrix (SPEC:288)");
        if (p != k)
            for (int j = 0; j < n; ++j) { std::swap(a[k * n + j], a[p * n + j]); std::swap(e[k * n + j], e[p * n + j]); }
        const double d = a[k * n + k];
        for (int j = 0; j < n; ++j) { a[k * n + j] = a[k * n + j] / d; e[k * n + j] = e[k * n + j] / d; }
        for (int i = 0; i < n; ++i) {
            if (i == k) continue;
            const double f = a[i * n + k];
            if (f == 0.0) continue;
            for (int j = 0; j < n; ++j) { a[i * n + j] = a[i * n + j] - f * a[k * n + j]; e[i * n + j] = e[i * n + j] - f * e[k * n + j]; }
        }
    }
    std::array<double, 49> out{};
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) out[i * 7 + j] = e[i * n + j];
    return out;
}

// ------------------------------------------------------- level builder ------
// DGS tiling rule (OD-1 rev. 2), shared with the GPU (csrc/smg_internal.h dgs_tiled):
// a level is tiled iff its cell count is at least tile_min and every extent is a
// multiple of the tile extent with at least two tiles per axis.
constexpr int kTile[3] = {16, 8, 8};
constexpr int64_t kTileMinDefault = int64_t{1} << 24;  // 256^3
static bool dgs_tiled(const int* n, int64_t tile_min) {
    if (tile_min <= 0) tile_min = kTileMinDefault;
    const int64_t cells = static_cast<int64_t>(n[0]) * n[1] * n[2];
    if (cells < tile_min) return false;
    for (int a = 0; a < 3; ++a)
        if (n[a] % kTile[a] || n[a] / kTile[a] < 2) return false;
    return true;
}

static void build_level(Level& L, const CellGrid& g, double eta, double gamma, int band_width,
                        int64_t tile_min = 0) {
    if (g.dim != 3) throw std::runtime_error("operator is 3-D only");
    L.grid = g;
    L.map = classify(g, band_width);
    L.h = g.h;
    L.eta = eta;
    L.gamma = gamma;
    L.eta_h2 = eta / (g.h * g.h);
    L.inv_h = 1.0 / g.h;
    L.dv = 6.0 * L.eta_h2;                                  // d_j velocity (SPEC:154, 3-D)
    L.dp = -6.0 * (1.0 + gamma * eta) / (g.h * g.h);       // d_j = L̃_j. M_.j, pressure
    const DofMap& m = L.map;
    L.vnb.assign(m.off[3], {0, 0, 0, 0, 0, 0, 0, 0});
    L.vdiag.assign(m.off[3], 6.0);
    L.fcells.assign(m.off[3], {ST_INACTIVE, ST_INACTIVE});
    for (int c = 0; c < 3; ++c)
        for (int z = 0; z < m.fext[c][2]; ++z)
            for (int y = 0; y < m.fext[c][1]; ++y)
                for (int x = 0; x < m.fext[c][0]; ++x) {
                    const int32_t id = m.face(c, x, y, z);
                    if (id < 0) continue;
                    auto& nb = L.vnb[id];
                    const int d[6][3] = {{-1, 0, 0}, {1, 0, 0}, {0, -1, 0}, {0, 1, 0}, {0, 0, -1}, {0, 0, 1}};
                    double diag = 6.0;
                    for (int k = 0; k < 6; ++k) {
                        const int32_t s = m.face(c, x + d[k][0], y + d[k][1], z + d[k][2]);
                        if (s == ST_INACTIVE) { diag -= 1.0; nb[k] = ST_INACTIVE; }  // dropped Neumann leg
                        else nb[k] = s;                                               // active or Dirichlet(0)
                    }
                    L.vdiag[id] = diag;
                    int lx = x, ly = y, lz = z;
                    if (c == 0) lx -= 1;
                    if (c == 1) ly -= 1;
                    if (c == 2) lz -= 1;
                    nb[6] = m.cell(lx, ly, lz);
                    nb[7] = m.cell(x, y, z);
                    L.fcells[id] = {nb[6], nb[7]};
                }
    const int64_t np = m.cnt[3];
    L.pface.assign(np + m.off[3], {-1, -1, -1, -1, -1, -1});
    L.pcell.assign(np + m.off[3], {-1, -1, -1, -1, -1, -1});
    for (int z = 0; z < g.n[2]; ++z)
        for (int y = 0; y < g.n[1]; ++y)
            for (int x = 0; x < g.n[0]; ++x) {
                const int32_t id = m.cell(x, y, z);
                if (id < 0) continue;
                L.pface[id] = {m.face(0, x, y, z), m.face(0, x + 1, y, z), m.face(1, x, y, z),
                               m.face(1, x, y + 1, z), m.face(2, x, y, z), m.face(2, x, y, z + 1)};
                L.pcell[id] = {m.cell(x - 1, y, z), m.cell(x + 1, y, z), m.cell(x, y - 1, z),
                               m.cell(x, y + 1, z), m.cell(x, y, z - 1), m.cell(x, y, z + 1)};
            }
    // DGS sets: V2 velocities split by red-black parity of their storage
    // coordinates, V2 pressures by the 8 parity colours (OD-1), both by the DGS tile
    // colour of the owning cell (a face at storage (x,y,z) is the low face of cell (x,y,z))
    const bool tiled = dgs_tiled(g.n, tile_min);
    L.ntc = tiled ? 8 : 1;
    for (int a = 0; a < 3; ++a) L.tile[a] = tiled ? kTile[a] : 0;
    auto tcol = [&](const std::array<int32_t, 3>& p) {
        if (!tiled) return 0;
        return ((p[0] / kTile[0]) & 1) + 2 * ((p[1] / kTile[1]) & 1) + 4 * ((p[2] / kTile[2]) & 1);
    };
    for (int t = 0; t < 8; ++t) {
        for (int k = 0; k < 2; ++k) L.dgs_vel[t][k].clear();
        for (int k = 0; k < 8; ++k) L.dgs_p[t][k].clear();
    }
    for (int k = 0; k < 8; ++k) L.all_p[k].clear();
    L.v2_lex.clear();
    for (int64_t q = 0; q < m.N; ++q) {
        const auto& p = m.pos[q];
        const int pc = (p[0] & 1) + 2 * (p[1] & 1) + 4 * (p[2] & 1);
        if (q >= m.off[3]) L.all_p[pc].push_back(static_cast<int32_t>(q));
        if (m.v1[q]) continue;
        L.v2_lex.push_back(static_cast<int32_t>(q));
        if (q < m.off[3]) L.dgs_vel[tcol(p)][(p[0] + p[1] + p[2]) & 1].push_back(static_cast<int32_t>(q));
        else L.dgs_p[tcol(p)][pc].push_back(static_cast<int32_t>(q));
    }
    // Vanka blocks: one per band cell with an active
    // pressure; slots [uL,uR,vL,vR,wL,wR,p]; colour (i&1)+2(j&1)+4(k&1).
    for (int k = 0; k < 8; ++k) L.vk[k].clear();
    L.v1_ids.clear();
    for (int64_t q = 0; q < m.N; ++q)
        if (m.v1[q]) L.v1_ids.push_back(static_cast<int32_t>(q));
    L.vk_all.clear();
    L.vk_inv.clear();
    std::vector<std::pair<int32_t, double>> row;
    for (int z = 0; z < g.n[2]; ++z)
        for (int y = 0; y < g.n[1]; ++y)
            for (int x = 0; x < g.n[0]; ++x) {
                const int32_t pid = m.cell(x, y, z);
                if (pid < 0 || !m.is_band(x, y, z)) continue;
                Level::Block blk;
                const auto& f = L.pface[pid];
                int mask = 0;
                for (int s = 0; s < 6; ++s) {
                    blk.dof[s] = f[s] >= 0 ? f[s] : -1;
                    if (f[s] >= 0) mask |= 1 << s;
                }
                blk.dof[6] = pid;
                for (int s = 0; s < 6; ++s)
                    if (f[s] >= 0) mask |= static_cast<int>(6.0 - L.vdiag[f[s]]) << (6 + 3 * s);
                blk.mask = mask;
                const int col = (x & 1) + 2 * (y & 1) + 4 * (z & 1);
                L.vk[col].push_back(blk);
                L.vk_all.push_back(blk);
                if (!L.vk_inv.count(mask)) {
                    // local matrix C_i L̃ C_i^T over the active slots, in slot order
                    std::vector<int32_t> act;
                    for (int s = 0; s < 7; ++s)
                        if (blk.dof[s] >= 0) act.push_back(blk.dof[s]);
                    const int nb = static_cast<int>(act.size());
                    std::vector<double> lm(static_cast<size_t>(nb) * nb, 0.0);
                    for (int a = 0; a < nb; ++a) {
                        ltilde_row(L, act[a], row);
                        for (auto& e : row)
                            for (int b2 = 0; b2 < nb; ++b2)
                                if (e.first == act[b2]) lm[a * nb + b2] = e.second;
                    }
                    std::array<double, 49> red = small_inverse(lm, nb);
                    // scatter to the fixed 7-slot layout (inactive slots: zero rows/cols)
                    std::array<double, 49> full{};
                    std::vector<int> slot;
                    for (int s = 0; s < 7; ++s)
                        if (blk.dof[s] >= 0) slot.push_back(s);
                    for (int a = 0; a < nb; ++a)
                        for (int b2 = 0; b2 < nb; ++b2) full[slot[a] * 7 + slot[b2]] = red[a * 7 + b2];
                    L.vk_inv[mask] = full;
                }
            }
}

// ----------------------------------------------------------- smoothers ------
// DGS velocity phase (Alg. 2 velocity rows: M_.j = e_j): one red-black
// colour of DGS tile colour T.
static void dgs_vel(const Level& L, vec& x, const vec& b, int T, int col) {
    const auto& lst = L.dgs_vel[T][col];
    parallel_for(static_cast<int64_t>(lst.size()), g_threads > 1 ? g_threads : 1, [&](int64_t t) {
        const int32_t f = lst[t];
        const double r = b[f] - mom_row(L, x, f);
        x[f] = x[f] + r / L.dv;
    });
}

// DGS forward pressure phase (Alg. 2 pressure rows, gather form, OD-1/OD-3) on the V2
// cells C of parity colour col in tile colour T: delta_C = r_C / d_p, then
// x += sum_C delta_C M_.C.  Only DOFs with a nonzero contribution are touched: the six
// faces of every C (x_f += (delta_left - delta_right) / h; M_{f,C} = +1/h on C's right
// face) and the pressures of C and of its axis neighbours (x_K += eta/h^2 (6 delta_K -
// sum_nbr delta); M_{K,C} = eta (B B^T)_{KC}).  `delta` (np entries) and `inset` are
// zero on entry and on exit.
static void dgs_p_fwd(const Level& L, vec& x, const vec& b, int T, int col, vec& delta,
                      std::vector<uint8_t>& inset) {
    const DofMap& m = L.map;
    const int64_t np = m.cnt[3], p0 = m.off[3];
    if (static_cast<int64_t>(delta.size()) != np) delta.assign(np, 0.0);
    if (static_cast<int64_t>(inset.size()) != np) inset.assign(np, 0);
    const auto& lst = L.dgs_p[T][col];
    parallel_for(static_cast<int64_t>(lst.size()), g_threads, [&](int64_t t) {
        const int32_t c = lst[t];
        delta[c - p0] = (b[c] - cont_row(L, x, c, L.gamma)) / L.dp;
        inset[c - p0] = 1;
    });
    auto dl = [&](int32_t id) { return id >= 0 ? delta[id - p0] : 0.0; };
    auto pupd = [&](int32_t k) {  // eager pressure update of cell k (operand order of the contract)
        const auto& nc = L.pcell[k];
        double s = dl(nc[0]) + dl(nc[1]);
        s = s + dl(nc[2]);
        s = s + dl(nc[3]);
        s = s + dl(nc[4]);
        s = s + dl(nc[5]);
        x[k] = x[k] + L.eta_h2 * (6.0 * delta[k - p0] - s);
    };
    // faces: every face of a colour-col cell borders exactly one such cell
    parallel_for(static_cast<int64_t>(lst.size()), g_threads, [&](int64_t t) {
        const auto& fc = L.pface[lst[t]];
        for (int q = 0; q < 6; ++q) {
            const int32_t f = fc[q];
            if (f < 0) continue;
            const auto& lr = L.fcells[f];
            x[f] = x[f] + (dl(lr[0]) - dl(lr[1])) * L.inv_h;
        }
        pupd(lst[t]);  // self term (its neighbours carry no delta)
    });
    // neighbour pressures: colours col ^ 1, col ^ 2, col ^ 4, gathered (several C may share one)
    for (int bit = 1; bit <= 4; bit <<= 1) {
        const auto& kl = L.all_p[col ^ bit];
        const int ax = bit == 1 ? 0 : (bit == 2 ? 2 : 4);
        parallel_for(static_cast<int64_t>(kl.size()), g_threads, [&](int64_t t) {
            const int32_t k = kl[t];
            const auto& nc = L.pcell[k];
            const bool hit = (nc[ax] >= 0 && inset[nc[ax] - p0]) || (nc[ax + 1] >= 0 && inset[nc[ax + 1] - p0]);
            if (hit) pupd(k);
        });
    }
    for (int32_t c : lst) {
        delta[c - p0] = 0.0;
        inset[c - p0] = 0;
    }
}

// DGS reverse (left-preconditioned) pressure phase:
// x_C += m_C^T (b - L̃ x) / d_p for V2 cells C of colour col in tile colour T,
// evaluated as (m_C^T b - m_C^T (L̃ x)) / d_p: the b part is fixed while b is (the GPU
// computes it once per V-cycle level visit), the L̃x part from the 6 momentum rows at C's
// faces and the 7 continuity rows around C, each part with the same operation order
// (DESIGN.md §4).  Same-colour cells never read each other's pressure: one pass.
static double m_col_dot(const Level& L, const vec& v, int32_t c) {
    const auto& f = L.pface[c];
    const auto& nc = L.pcell[c];
    const double fl = ((v[f[1]] - v[f[0]]) + (v[f[3]] - v[f[2]])) + (v[f[5]] - v[f[4]]);
    double s = v[nc[0]] + v[nc[1]];
    s = s + v[nc[2]];
    s = s + v[nc[3]];
    s = s + v[nc[4]];
    s = s + v[nc[5]];
    return fl * L.inv_h + L.eta_h2 * (6.0 * v[c] - s);
}
static double m_col_dot_lx(const Level& L, const vec& x, int32_t c) {
    const auto& f = L.pface[c];
    const auto& nc = L.pcell[c];
    double lf[6], ln[6];
    for (int q = 0; q < 6; ++q) lf[q] = mom_row(L, x, f[q]);
    for (int q = 0; q < 6; ++q) ln[q] = cont_row(L, x, nc[q], L.gamma);
    const double lc = cont_row(L, x, c, L.gamma);
    const double fl = ((lf[1] - lf[0]) + (lf[3] - lf[2])) + (lf[5] - lf[4]);
    double s = ln[0] + ln[1];
    s = s + ln[2];
    s = s + ln[3];
    s = s + ln[4];
    s = s + ln[5];
    return fl * L.inv_h + L.eta_h2 * (6.0 * lc - s);
}
static void dgs_p_rev(const Level& L, vec& x, const vec& b, int T, int col) {
    const auto& lst = L.dgs_p[T][col];
    std::vector<double> nv(lst.size());
    parallel_for(static_cast<int64_t>(lst.size()), g_threads, [&](int64_t t) {
        const int32_t c = lst[t];
        const double cb = m_col_dot(L, b, c), cl = m_col_dot_lx(L, x, c);
        nv[t] = x[c] + (cb - cl) / L.dp;
    });
    for (size_t t = 0; t < lst.size(); ++t) x[lst[t]] = nv[t];
}

// Phase ids (test harness and GPU share them): forward 0,1 velocity colours
// 0,1; 2..9 pressure colours 0..7; reverse 10..17 pressure colours 7..0;
// 18,19 velocity colours 1,0 -- the exact reverse traversal.  On a tiled
// level a phase acts on one DGS tile colour T (argument phase + 32 T).
constexpr int kDgsPhases = 20;
struct DgsScratch {
    vec delta;
    std::vector<uint8_t> inset;
};
static void dgs_phase(const Level& L, vec& x, const vec& b, int phase, int T, DgsScratch& sc) {
    if (T < 0 || T >= L.ntc) throw std::runtime_error("bad dgs tile colour");
    if (phase == 0 || phase == 1) dgs_vel(L, x, b, T, phase);
    else if (phase >= 2 && phase <= 9) dgs_p_fwd(L, x, b, T, phase - 2, sc.delta, sc.inset);
    else if (phase >= 10 && phase <= 17) dgs_p_rev(L, x, b, T, 17 - phase);
    else if (phase == 18 || phase == 19) dgs_vel(L, x, b, T, 19 - phase);
    else throw std::runtime_error("bad dgs phase");
}

// SPEC-literal DGS (Hierarchy::order = 1, comparison mode): V2 DOFs relaxed one at a
// time in ascending global DOF index (velocities u, v, w lexicographic, then pressures;
// SPEC:261, 332), the reverse in strictly descending order.  Velocity j:
// x_j += r_j / d_v.  Pressure j forward: x += (r_j / d_p) M_.j; reverse: x_j += m_j^T (b -
// L̃x) / d_p.  Strictly sequential (no colouring): the reference's own traversal.
static void dgs_lex(const Level& L, vec& x, const vec& b, bool forward) {
    const int64_t nv = L.map.off[3];
    const int64_t n = static_cast<int64_t>(L.v2_lex.size());
    for (int64_t t0 = 0; t0 < n; ++t0) {
        const int32_t j = L.v2_lex[forward ? t0 : n - 1 - t0];
        if (j < nv) {
            x[j] = x[j] + (b[j] - mom_row(L, x, j)) / L.dv;
        } else if (forward) {
            const double d = (b[j] - cont_row(L, x, j, L.gamma)) / L.dp;
            const auto& f = L.pface[j];
            for (int q = 0; q < 6; ++q)
                if (f[q] >= 0) x[f[q]] = x[f[q]] + ((q & 1) ? d : -d) * L.inv_h;
            x[j] = x[j] + L.eta_h2 * 6.0 * d;
            for (int32_t k : L.pcell[j])
                if (k >= 0) x[k] = x[k] - L.eta_h2 * d;
        } else {
            x[j] = x[j] + (m_col_dot(L, b, j) - m_col_dot_lx(L, x, j)) / L.dp;
        }
    }
}

// symmetric_dgs: forward phases then their exact reverse.
static void symmetric_dgs(const Level& L, vec& x, const vec& b, bool skip_reverse = false, int order = 0) {
    if (order == 1) {
        dgs_lex(L, x, b, true);
        if (!skip_reverse) dgs_lex(L, x, b, false);
        return;
    }
    DgsScratch sc;
    for (int T = 0; T < L.ntc; ++T)
        for (int ph = 0; ph < kDgsPhases / 2; ++ph) dgs_phase(L, x, b, ph, T, sc);
    if (skip_reverse) return;
    for (int T = L.ntc - 1; T >= 0; --T)
        for (int ph = kDgsPhases / 2; ph < kDgsPhases; ++ph) dgs_phase(L, x, b, ph, T, sc);
}

// One Vanka colour phase, Jacobi within the colour (OD-2): every block reads
// the pre-phase state; writes of same-colour blocks are disjoint.
static void vanka_colour(const Level& L, vec& x, const vec& b, int col) {
    const auto& blocks = L.vk[col];
    std::vector<std::array<double, 7>> dl(blocks.size());
    parallel_for(static_cast<int64_t>(blocks.size()), g_threads, [&](int64_t t) {
        const auto& blk = blocks[t];
        double r[7];
        for (int s = 0; s < 7; ++s) {
            const int32_t id = blk.dof[s];
            if (id < 0) { r[s] = 0.0; continue; }
            r[s] = b[id] - (s < 6 ? mom_row(L, x, id) : cont_row(L, x, id, L.gamma));
        }
        const auto& K = L.vk_inv.at(blk.mask);
        for (int s = 0; s < 7; ++s) {
            double acc = 0.0;
            for (int q = 0; q < 7; ++q) acc = acc + K[s * 7 + q] * r[q];
            dl[t][s] = acc;
        }
    });
    parallel_for(static_cast<int64_t>(blocks.size()), g_threads, [&](int64_t t) {
        const auto& blk = blocks[t];
        for (int s = 0; s < 7; ++s)
            if (blk.dof[s] >= 0) x[blk.dof[s]] = x[blk.dof[s]] + dl[t][s];
    });
}

// vanka_multiplicative_symmetric: the 8 parity colours in
// the order kVankaOrder, then exactly reversed (SPEC: "reverse multiplicative
// sweep reverses both block order and color order").  The SPEC fixes only the
// 2^d parity colouring, not the order of the colours (OD-2); this order puts
// complementary parities (p, 7 - p) next to each other.  Two such colours never
// touch each other's DOFs (every residual stencil reaches along one axis, so a
// block reads DOFs of cells differing in at most two parities), hence each
// adjacent pair commutes and a GPU may run it as ONE Jacobi phase with
// bit-identical results: 8 dependent phases per symmetric sweep instead of 16.
// Measured MG/SQMR convergence equals the 0..7 order.
static const int kVankaOrder[8] = {0, 7, 1, 6, 2, 5, 3, 4};
// SPEC-literal comparison mode (order = 1): blocks strictly one after another, colour-major
// 0..7 and ascending cell index within a colour, each block seeing every
// earlier update; the reverse sweep reverses block and colour order.
static void vanka_block_seq(const Level& L, vec& x, const vec& b, const Level::Block& blk) {
    double r[7];
    for (int s = 0; s < 7; ++s) {
        const int32_t id = blk.dof[s];
        r[s] = id < 0 ? 0.0 : b[id] - (s < 6 ? mom_row(L, x, id) : cont_row(L, x, id, L.gamma));
    }
    const auto& K = L.vk_inv.at(blk.mask);
    double dl[7];
    for (int s = 0; s < 7; ++s) {
        double acc = 0.0;
        for (int q = 0; q < 7; ++q) acc = acc + K[s * 7 + q] * r[q];
        dl[s] = acc;
    }
    for (int s = 0; s < 7; ++s)
        if (blk.dof[s] >= 0) x[blk.dof[s]] = x[blk.dof[s]] + dl[s];
}
static void vanka_symmetric(const Level& L, vec& x, const vec& b, int order = 0) {
    if (order == 1) {
        for (int c = 0; c < 8; ++c)
            for (const auto& blk : L.vk[c]) vanka_block_seq(L, x, b, blk);
        for (int c = 7; c >= 0; --c)
            for (auto it = L.vk[c].rbegin(); it != L.vk[c].rend(); ++it) vanka_block_seq(L, x, b, *it);
        return;
    }
    for (int c = 0; c < 8; ++c) vanka_colour(L, x, b, kVankaOrder[c]);
    for (int c = 7; c >= 0; --c) vanka_colour(L, x, b, kVankaOrder[c]);
}

// vanka_additive (Eq. S_AV): r = b - L~x once; every block solves
// against that same residual; each V1 DOF gets omega times the sum of the
// corrections of the blocks containing it, added in ascending block (cell lex)
// order starting from 0.0 -- a fixed order, so the result is deterministic and
// independent of how the block solves are scheduled.
static void vanka_additive(const Level& L, vec& x, const vec& b, double omega) {
    const auto& blocks = L.vk_all;
    std::vector<std::array<double, 7>> dl(blocks.size());
    parallel_for(static_cast<int64_t>(blocks.size()), g_threads, [&](int64_t t) {
        const auto& blk = blocks[t];
        double r[7];
        for (int s = 0; s < 7; ++s) {
            const int32_t id = blk.dof[s];
            if (id < 0) { r[s] = 0.0; continue; }
            r[s] = b[id] - (s < 6 ? mom_row(L, x, id) : cont_row(L, x, id, L.gamma));
        }
        const auto& K = L.vk_inv.at(blk.mask);
        for (int s = 0; s < 7; ++s) {
            double acc = 0.0;
            for (int q = 0; q < 7; ++q) acc = acc + K[s * 7 + q] * r[q];
            dl[t][s] = acc;
        }
    });
    vec acc(x.size(), 0.0);
    std::vector<uint8_t> hit(x.size(), 0);
    for (size_t t = 0; t < blocks.size(); ++t)
        for (int s = 0; s < 7; ++s) {
            const int32_t id = blocks[t].dof[s];
            if (id < 0) continue;
            acc[id] = acc[id] + dl[t][s];
            hit[id] = 1;
        }
    for (size_t q = 0; q < x.size(); ++q)
        if (hit[q]) x[q] = x[q] + omega * acc[q];
}

// Direct-on-V1 (PAPER section 6 "the ideal scenario where a direct solver is employed
// for the boundary domains"): x_V1 <- x_V1 + A11^{-1} (b - L~x)_V1 with A11 the V1 x V1 principal
// sub-block of L~, i.e. the exact solve of the V1 equations with x_V2 frozen.  A11^{-1} is a dense
// symmetric inverse (the coarsest solve's LU + exact symmetrisation, OD-4) applied with the coarse
// GEMV's summation order (64-column chunks, ascending); capped like the coarsest system.
static void vanka_direct(const Level& L, vec& x, const vec& b) {
    const auto& ids = L.v1_ids;
    const int64_t n = static_cast<int64_t>(ids.size());
    if (n == 0) return;
    if (L.v1_inv.empty()) {
        if (n > 20000) throw std::runtime_error("direct-on-V1: |V1| above the dense cap 20000 (SPEC:365)");
        std::vector<int32_t> loc(L.map.N, -1);
        for (int64_t k = 0; k < n; ++k) loc[ids[k]] = static_cast<int32_t>(k);
        std::vector<double> a(static_cast<size_t>(n) * n, 0.0);
        std::vector<std::pair<int32_t, double>> row;
        for (int64_t k = 0; k < n; ++k) {
            ltilde_row(L, ids[k], row);
            for (auto& e : row)
                if (loc[e.first] >= 0) a[static_cast<size_t>(k) * n + loc[e.first]] += e.second;
        }
        L.v1_inv = dense_inverse_sym(std::move(a), static_cast<int>(n), std::max(1, g_threads));
    }
    vec r(n);
    const int64_t nv = L.map.off[3];
    parallel_for(n, g_threads, [&](int64_t k) {
        const int32_t id = ids[k];
        r[k] = b[id] - (id < nv ? mom_row(L, x, id) : cont_row(L, x, id, L.gamma));
    });
    parallel_for(n, g_threads, [&](int64_t i) {
        const double* kk = &L.v1_inv[static_cast<size_t>(i) * n];
        double sum = 0.0;
        for (int64_t j0 = 0; j0 < n; j0 += 64) {
            double part = 0.0;
            const int64_t j1 = std::min<int64_t>(n, j0 + 64);
            for (int64_t j = j0; j < j1; ++j) part = part + kk[j] * r[j];
            sum = sum + part;
        }
        x[ids[i]] = x[ids[i]] + sum;
    });
}

// Vanka flavour of the smoother (SmootherConfig).
struct VankaCfg {
    int kind = 0;        // 0 symmetric multiplicative, 1 additive, 2 direct solve on V1
    double omega = 1.0;  // additive damping
};
static VankaCfg g_vanka_default;

static void vanka_apply(const Level& L, vec& x, const vec& b, const VankaCfg& vc, int order = 0) {
    if (vc.kind == 1) vanka_additive(L, x, b, vc.omega);
    else if (vc.kind == 2) vanka_direct(L, x, b);
    else vanka_symmetric(L, x, b, order);
}

// smooth, Alg. 3: nu x Vanka(V1), symmetric DGS(V2), nu x Vanka(V1).
static void smooth(const Level& L, vec& x, const vec& b, int nu, bool skip_reverse = false,
                   const VankaCfg& vc = g_vanka_default, int order = 0) {
    const int reps = vc.kind == 2 ? 1 : nu;  // an exact V1 solve is idempotent: once per side
    for (int k = 0; k < reps; ++k) vanka_apply(L, x, b, vc, order);
    symmetric_dgs(L, x, b, skip_reverse, order);
    for (int k = 0; k < reps; ++k) vanka_apply(L, x, b, vc, order);
}

// ------------------------------------------------------------ transfer ------
// Shared 1-D weight tables (OD-6).  Normal direction: a fine face at
// even index I coincides with coarse face I/2 (weight 1); odd I sits midway
// (1/2, 1/2).  Tangential: fine cell J has parent J>>1 with weight 3/4 and the
// nearer second coarse cell (J even: parent-1, J odd: parent+1) with 1/4.
// Legs to non-active coarse DOFs are dropped, no renormalisation.
struct Leg { int idx; double w; };
static int normal_legs(int I, Leg* out) {
    if ((I & 1) == 0) { out[0] = {I / 2, 1.0}; return 1; }
    out[0] = {(I - 1) / 2, 0.5};
    out[1] = {(I + 1) / 2, 0.5};
    return 2;
}
static int tangent_legs(int J, Leg* out) {
    const int p = J >> 1;
    out[0] = {p, 0.75};
    out[1] = {(J & 1) ? p + 1 : p - 1, 0.25};
    return 2;
}

// prolong: xf = P xc (values, not increments).
static void prolong(const Level& F, const Level& C, const vec& xc, vec& xf) {
    const DofMap& fm = F.map;
    const DofMap& cm = C.map;
    xf.assign(fm.N, 0.0);
    parallel_for(fm.N, g_threads, [&](int64_t q) {
        const int comp = fm.comp[q];
        const auto& p = fm.pos[q];
        if (comp == 3) {
            xf[q] = val(xc, cm.cell(p[0] >> 1, p[1] >> 1, p[2] >> 1));
            return;
        }
        // separable gather: normal axis innermost, then the tangential axes in x,y,z order
        const int ta = comp == 0 ? 1 : 0, tb = comp == 2 ? 1 : 2;
        Leg ln[2], la[2], lb[2];
        const int nn = normal_legs(p[comp], ln);
        tangent_legs(p[ta], la);
        tangent_legs(p[tb], lb);
        double sb = 0.0;
        for (int ib = 0; ib < 2; ++ib) {
            double sa = 0.0;
            for (int ia = 0; ia < 2; ++ia) {
                double sn = 0.0;
                for (int in = 0; in < nn; ++in) {
                    int c3[3];
                    c3[comp] = ln[in].idx;
                    c3[ta] = la[ia].idx;
                    c3[tb] = lb[ib].idx;
                    sn = sn + ln[in].w * val(xc, cm.face(comp, c3[0], c3[1], c3[2]));
                }
                sa = sa + la[ia].w * sn;
            }
            sb = sb + lb[ib].w * sa;
        }
        xf[q] = sb;
    });
}

// restrict: rc = (1/8) P^T rf through the same weight tables.
static void restrict_(const Level& F, const Level& C, const vec& rf, vec& rc) {
    const DofMap& fm = F.map;
    const DofMap& cm = C.map;
    rc.assign(cm.N, 0.0);
    parallel_for(cm.N, g_threads, [&](int64_t q) {
        const int comp = cm.comp[q];
        const auto& p = cm.pos[q];
        if (comp == 3) {
            double s = 0.0;
            for (int k = 0; k < 2; ++k)
                for (int j = 0; j < 2; ++j)
                    for (int i = 0; i < 2; ++i)
                        s = s + val(rf, fm.cell(2 * p[0] + i, 2 * p[1] + j, 2 * p[2] + k));
            rc[q] = 0.125 * s;
            return;
        }
        // fine faces with a nonzero weight to coarse face p: normal 2I-1 (1/2), 2I (1), 2I+1 (1/2);
        // tangential 2J-1 (1/4), 2J (3/4), 2J+1 (3/4), 2J+2 (1/4).
        const int ta = comp == 0 ? 1 : 0, tb = comp == 2 ? 1 : 2;
        const int nI[3] = {2 * p[comp] - 1, 2 * p[comp], 2 * p[comp] + 1};
        const double wI[3] = {0.5, 1.0, 0.5};
        const double wT[4] = {0.25, 0.75, 0.75, 0.25};
        double sb = 0.0;
        for (int ib = 0; ib < 4; ++ib) {
            double sa = 0.0;
            for (int ia = 0; ia < 4; ++ia) {
                double sn = 0.0;
                for (int in = 0; in < 3; ++in) {
                    int c3[3];
                    c3[comp] = nI[in];
                    c3[ta] = 2 * p[ta] - 1 + ia;
                    c3[tb] = 2 * p[tb] - 1 + ib;
                    sn = sn + wI[in] * val(rf, fm.face(comp, c3[0], c3[1], c3[2]));
                }
                sa = sa + wT[ia] * sn;
            }
            sb = sb + wT[ib] * sa;
        }
        rc[q] = 0.125 * sb;
    });
}

// ----------------------------------------------------------- multigrid ------
struct Hierarchy {
    std::vector<std::unique_ptr<Level>> lv;
    std::vector<double> coarse_inv;  // symmetric dense inverse of the coarsest L̃, row-major
    int nu = 1;
    int cycle = 0;              // 0 V-cycle, 1 W-cycle
    bool skip_reverse = false;  // fault injection for the symmetry negative control
    VankaCfg vanka;             // multiplicative (default) or additive Vanka on V1
    int order = 0;              // 0: the GPU's order (OD-1/OD-2); 1: SPEC-literal sequential order
};

static std::vector<double> assemble_dense(const Level& L, bool penalized) {
    const int64_t n = L.map.N;
    std::vector<double> a(static_cast<size_t>(n) * n, 0.0);
    std::vector<std::pair<int32_t, double>> row;
    for (int64_t r = 0; r < n; ++r) {
        ltilde_row(L, static_cast<int32_t>(r), row);
        for (auto& e : row) {
            double v = e.second;
            if (!penalized && r >= L.map.off[3] && e.first == r) v = 0.0;
            a[static_cast<size_t>(r) * n + e.first] += v;
        }
    }
    return a;
}

// build_hierarchy.
static std::unique_ptr<Hierarchy> build_hierarchy(const CellGrid& g, double eta, double gamma, int levels,
                                                  int nu, int band_width, int64_t tile_min = 0) {
    if (levels < 1) throw std::runtime_error("levels < 1");
    auto H = std::make_unique<Hierarchy>();
    H->nu = nu;
    CellGrid cur = g;
    for (int l = 0; l < levels; ++l) {
        if (l > 0) cur = coarsen(cur);
        for (int a = 0; a < 3; ++a)
            if (cur.n[a] < 2) throw std::runtime_error("coarsened extent below 2 (SPEC:82)");
        auto L = std::make_unique<Level>();
        build_level(*L, cur, eta, gamma, band_width, tile_min);
        H->lv.push_back(std::move(L));
    }
    const Level& C = *H->lv.back();
    if (C.map.N > 20000) throw std::runtime_error("coarsest system above dense cap 20000 (SPEC:365)");
    H->coarse_inv = dense_inverse_sym(assemble_dense(C, true), static_cast<int>(C.map.N), std::max(1, g_threads));
    return H;
}

static void coarse_solve(const Hierarchy& H, const vec& b, vec& x) {
    const int64_t n = H.lv.back()->map.N;
    x.assign(n, 0.0);
    // Fixed summation order: partial sums over 64-column chunks,
    // chunks accumulated in ascending order.
    parallel_for(n, g_threads, [&](int64_t i) {
        const double* k = &H.coarse_inv[static_cast<size_t>(i) * n];
        double s = 0.0;
        for (int64_t j0 = 0; j0 < n; j0 += 64) {
            double part = 0.0;
            const int64_t j1 = std::min<int64_t>(n, j0 + 64);
            for (int64_t j = j0; j < j1; ++j) part = part + k[j] * b[j];
            s = s + part;
        }
        x[i] = s;
    });
}

// cycle, Alg. 1 with x0 = 0.
static void vcycle(const Hierarchy& H, int l, const vec& b, vec& x) {
    const Level& L = *H.lv[l];
    if (l == static_cast<int>(H.lv.size()) - 1) { coarse_solve(H, b, x); return; }
    x.assign(L.map.N, 0.0);
    smooth(L, x, b, H.nu, H.skip_reverse, H.vanka, H.order);
    vec r, rc, ec, ef;
    residual(L, x, b, r);
    restrict_(L, *H.lv[l + 1], r, rc);
    vcycle(H, l + 1, rc, ec);
    // W-cycle: a second recursive call at every level below the finest, on the
    // residual of the first; skipped when the child is the exact coarsest solve.
    if (H.cycle == 1 && l >= 1 && l + 2 < static_cast<int>(H.lv.size())) {
        vec r2, e2;
        residual(*H.lv[l + 1], ec, rc, r2);
        vcycle(H, l + 1, r2, e2);
        for (size_t q = 0; q < ec.size(); ++q) ec[q] = ec[q] + e2[q];
    }
    prolong(L, *H.lv[l + 1], ec, ef);
    for (int64_t q = 0; q < L.map.N; ++q) x[q] = x[q] + ef[q];
    smooth(L, x, b, H.nu, H.skip_reverse, H.vanka, H.order);
}

// ----------------------------------------------------- canonical dot -------
// Fixed reduction order of every SQMR inner product (OD-12 rev. 2), the one the
// GPU's fused kernels produce natively (kernels.cu k_cdot / k_apply_q / k_apply_x / final2):
//   * blocks of 32 x-lanes x 8 y-rows x 4 z-planes; a lane adds, over its cell's planes in
//     ascending z, ((p_u + p_v) + p_w) + p_p, the products of the four DOFs stored at the cell
//     (the u, v, w faces on the cell's low side and its pressure; an inactive one gives +0);
//   * the 32 lanes of a row combine by the tree acc[l] += acc[l + o], o = 16..1 (lane 0), the 8
//     rows are added in ascending order: the block partial, at ((zb GY + by) GX + bx);
//   * final: 256 accumulators take partials k = t, t + 256, ... ascending, each warp of 32
//     combines by the same tree, the 8 warp sums are added in ascending order.
static double lane_tree(double* acc) {
    for (int o = 16; o > 0; o >>= 1)
        for (int l = 0; l < o; ++l) acc[l] = acc[l] + acc[l + o];
    return acc[0];
}

static double cdot(const Level& L, const vec& a, const vec& b) {
    const DofMap& m = L.map;
    const int nx = m.n[0], ny = m.n[1], nz = m.n[2];
    const int GX = (nx + 31) / 32, GY = (ny + 7) / 8, GZ = (nz + 3) / 4;
    std::vector<double> part(static_cast<size_t>(GX) * GY * GZ);
    auto prod = [&](int32_t id) { return id >= 0 ? a[id] * b[id] : 0.0 * 0.0; };
    parallel_for(GZ, g_threads, [&](int64_t zb) {
        for (int by = 0; by < GY; ++by)
            for (int bx = 0; bx < GX; ++bx) {
                double ws[8];
                for (int w = 0; w < 8; ++w) {
                    double acc[32];
                    for (int l = 0; l < 32; ++l) {
                        const int x = bx * 32 + l, y = by * 8 + w;
                        double v = 0.0;
                        if (x < nx && y < ny)
                            for (int z = static_cast<int>(zb) * 4; z < std::min(nz, static_cast<int>(zb) * 4 + 4); ++z) {
                                const double pu = prod(m.face(0, x, y, z)), pv = prod(m.face(1, x, y, z));
                                const double pw = prod(m.face(2, x, y, z)), pp = prod(m.cell(x, y, z));
                                v = v + (((pu + pv) + pw) + pp);
                            }
                        acc[l] = v;
                    }
                    ws[w] = lane_tree(acc);
                }
                double s = ws[0];
                for (int w = 1; w < 8; ++w) s = s + ws[w];
                part[(static_cast<size_t>(zb) * GY + by) * GX + bx] = s;
            }
    });
    double acc[256];
    for (int t = 0; t < 256; ++t) acc[t] = 0.0;
    for (size_t k = 0; k < part.size(); ++k) acc[k & 255] = acc[k & 255] + part[k];
    double ws[8];
    for (int w = 0; w < 8; ++w) ws[w] = lane_tree(acc + 32 * w);
    double s = ws[0];
    for (int w = 1; w < 8; ++w) s = s + ws[w];
    return s;
}

// -------------------------------------------------------------- krylov ------
enum { ST_CONVERGED = 0, ST_MAXIT = 1, ST_BREAKDOWN = 2 };

// sqmr_solve, Alg. 4 verbatim; x0 = 0; true
// relative residual recomputed every iteration.
static int sqmr(const Hierarchy& H, const vec& b, vec& x, double tol, int maxit, int precond,
                std::vector<double>& hist, std::vector<double>& secs) {
    const Level& L0 = *H.lv[0];
    const int64_t n = L0.map.N;
    auto t0 = std::chrono::steady_clock::now();
    hist.clear();
    secs.clear();
    x.assign(n, 0.0);
    const double bnorm = std::sqrt(cdot(L0, b, b));
    if (bnorm == 0.0) return ST_CONVERGED;
    auto M = [&](const vec& in, vec& out) {
        if (precond) vcycle(H, 0, in, out);
        else out = in;
    };
    vec s = b, t, q, d(n, 0.0), r;
    M(s, t);
    q = t;
    double tau = std::sqrt(cdot(L0, t, t)), nu_old = 0.0, rho = cdot(L0, s, q);
    if (std::fabs(rho) < 1e-300) return ST_BREAKDOWN;
    for (int j = 1; j <= maxit; ++j) {
        apply(L0, q, t, false);
        const double sigma = cdot(L0, q, t);
        if (std::fabs(sigma) < 1e-300) return ST_BREAKDOWN;
        const double alpha = rho / sigma;
        for (int64_t i = 0; i < n; ++i) s[i] = s[i] - alpha * t[i];
        M(s, t);
        const double nu = std::sqrt(cdot(L0, t, t)) / tau;
        const double c = 1.0 / std::sqrt(1.0 + nu * nu);
        tau = tau * nu * c;
        const double c2 = c * c;
        const double cd = c2 * (nu_old * nu_old), cq = c2 * alpha;
        for (int64_t i = 0; i < n; ++i) {
            d[i] = cd * d[i] + cq * q[i];
            x[i] = x[i] + d[i];
        }
        vec lx;
        apply(L0, x, lx, false);
        for (int64_t i = 0; i < n; ++i) lx[i] = b[i] - lx[i];
        const double rel = std::sqrt(cdot(L0, lx, lx)) / bnorm;
        hist.push_back(rel);
        secs.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
        if (rel < tol) return ST_CONVERGED;
        const double rho_new = cdot(L0, s, t);
        if (std::fabs(rho_new) < 1e-300) return ST_BREAKDOWN;
        const double beta = rho_new / rho;
        for (int64_t i = 0; i < n; ++i) q[i] = t[i] + beta * q[i];
        rho = rho_new;
        nu_old = nu;
    }
    return ST_MAXIT;
}

// mg_solve: x_j = x_{j-1} + cycle(b - L~ x_{j-1}), x_0 = 0, history of
// the true relative residual ||b - L~ x_j|| / ||b|| (canonical inner product).
static int mg_solve(const Hierarchy& H, const vec& b, vec& x, double tol, int maxit, std::vector<double>& hist,
                    std::vector<double>& secs) {
    const Level& L0 = *H.lv[0];
    const int64_t n = L0.map.N;
    auto t0 = std::chrono::steady_clock::now();
    hist.clear();
    secs.clear();
    x.assign(n, 0.0);
    const double bnorm = std::sqrt(cdot(L0, b, b));
    if (bnorm == 0.0) return ST_CONVERGED;
    vec r = b, e;
    for (int j = 1; j <= maxit; ++j) {
        vcycle(H, 0, r, e);
        for (int64_t i = 0; i < n; ++i) x[i] = x[i] + e[i];
        residual(L0, x, b, r);
        const double rel = std::sqrt(cdot(L0, r, r)) / bnorm;
        hist.push_back(rel);
        secs.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
        if (rel < tol) return ST_CONVERGED;
    }
    return ST_MAXIT;
}

// ------------------------------------------------------------- forcing ------
// Counter-based SplitMix64 forcing (OD-9): value depends only on (seed,
// component, storage coordinates), never on the decomposition.
static inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static inline uint64_t key5(uint64_t seed, uint64_t c, uint64_t i, uint64_t j, uint64_t k) {
    return mix64(mix64(mix64(mix64(mix64(seed) ^ c) ^ k) ^ j) ^ i);
}
static inline double unit01(uint64_t h) { return static_cast<double>(h >> 11) * 0x1.0p-53; }

// Dirichlet value of a (non-active) face of component c at storage coordinates
// (x,y,z) for the lid-driven cavity: u = 1 on the
// faces of the ring cells above the top (y = ny), 0 elsewhere.
static double lid_value(const Level& L, int c, int x, int y, int z) {
    (void)x;
    (void)z;
    return (c == 0 && y == L.map.n[1]) ? 1.0 : 0.0;
}

// assemble_rhs: b = f - L_{active,Dirichlet} g, i.e. every
// stencil leg of an active row into a Dirichlet face moves to the right-hand
// side with the opposite sign of its matrix entry (momentum: -eta/h^2 legs;
// continuity: +-1/h legs to Dirichlet faces).
template <class GV>
static void dirichlet_rhs_g(const Level& L, vec& b, GV&& value);
static void dirichlet_rhs(const Level& L, vec& b) {
    dirichlet_rhs_g(L, b, [&](int c, int x, int y, int z) { return lid_value(L, c, x, y, z); });
}
// General BoundaryData: value(c, x, y, z) is the Dirichlet velocity of the face of
// component c at storage coordinates (x, y, z) (ring faces included: tangential coordinates -1 and n).
template <class GV>
static void dirichlet_rhs_g(const Level& L, vec& b, GV&& value) {
    const DofMap& m = L.map;
    const int d[6][3] = {{-1, 0, 0}, {1, 0, 0}, {0, -1, 0}, {0, 1, 0}, {0, 0, -1}, {0, 0, 1}};
    for (int64_t q = 0; q < m.off[3]; ++q) {
        const int c = m.comp[q];
        const auto& p = m.pos[q];
        for (int k = 0; k < 6; ++k) {
            const int x = p[0] + d[k][0], y = p[1] + d[k][1], z = p[2] + d[k][2];
            if (m.face(c, x, y, z) != ST_DIRICHLET) continue;
            const double gv = value(c, x, y, z);
            if (gv != 0.0) b[q] = b[q] + L.eta_h2 * gv;  // row entry -eta/h^2 -> rhs +eta/h^2 g
        }
    }
    for (int64_t q = m.off[3]; q < m.N; ++q) {  // continuity legs to Dirichlet faces
        const auto& p = m.pos[q];
        for (int c = 0; c < 3; ++c)
            for (int side = 0; side < 2; ++side) {
                int f3[3] = {p[0], p[1], p[2]};
                f3[c] += side;
                if (m.face(c, f3[0], f3[1], f3[2]) != ST_DIRICHLET) continue;
                const double gv = value(c, f3[0], f3[1], f3[2]);
                // (L~x)_C = -(x_R - x_L)/h: entry -1/h on the right face, +1/h on the left face
                if (gv != 0.0) b[q] = b[q] - (side ? -L.inv_h : L.inv_h) * gv;
            }
    }
}

// kind: 0 = iid U[-1,1] (cfg 0,1,3); 1 = 8 Fourier modes (cfg 2); 2 = channel (cfg 4);
// 3 = lid-driven cavity (zero body force, lid u = 1 at the top y face).
static void forcing(const Level& L, int kind, uint64_t seed, vec& b) {
    const DofMap& m = L.map;
    b.assign(m.N, 0.0);
    if (kind == 3) {
        dirichlet_rhs(L, b);
        return;
    }
    double amp[3][8];
    int kw[3][8][3];
    if (kind == 1)
        for (int c = 0; c < 3; ++c)
            for (int md = 0; md < 8; ++md) {
                for (int a = 0; a < 3; ++a) kw[c][md][a] = 1 + static_cast<int>(key5(seed, 16 + c, md, a, 0) % 8);
                const double u1 = 1.0 - unit01(key5(seed, 32 + c, md, 0, 1));
                const double u2 = unit01(key5(seed, 32 + c, md, 0, 2));
                amp[c][md] = std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
            }
    const double h = L.h;
    for (int64_t q = 0; q < m.off[3]; ++q) {
        const int c = m.comp[q];
        const auto& p = m.pos[q];
        const uint64_t hsh = key5(seed, c, p[0], p[1], p[2]);
        const double u = 2.0 * unit01(hsh) - 1.0;
        if (kind == 0) b[q] = u;
        else if (kind == 2) b[q] = (c == 0 ? 1.0 : 0.0) + 0.1 * u;
        else {
            double xyz[3];
            for (int a = 0; a < 3; ++a) xyz[a] = (a == c) ? p[a] * h : (p[a] + 0.5) * h;
            double s = 0.0;
            for (int md = 0; md < 8; ++md)
                s = s + amp[c][md] * std::sin(3.141592653589793 * kw[c][md][0] * xyz[0]) *
                            std::sin(3.141592653589793 * kw[c][md][1] * xyz[1]) *
                            std::sin(3.141592653589793 * kw[c][md][2] * xyz[2]);
            b[q] = s;
        }
    }
}

// ----------------------------------------------------------- census ---------
// DOF census for the walled cavity (interior box + implicit Dirichlet ring),
// dim 2 or 3 (PAPER Table 1).
static void census_box(int dim, int nx, int ny, int nz, int width, int64_t* out) {
    CellGrid g;
    g.dim = dim;
    g.n[0] = nx;
    g.n[1] = ny;
    g.n[2] = dim == 3 ? nz : 1;
    g.lab.assign(static_cast<size_t>(g.n[0]) * g.n[1] * g.n[2], LAB_I);
    DofMap m = classify(g, width);
    int64_t v1 = 0;
    for (uint8_t f : m.v1) v1 += f;
    out[0] = m.N;
    out[1] = v1;
}

}  // namespace orc

// =========================================================== C ABI (ctypes) ==
using namespace orc;

struct OrcHandle {
    std::unique_ptr<Hierarchy> H;
    std::string err;
};

static thread_local std::string g_last_err;

extern "C" {

const char* orc_last_error() { return g_last_err.c_str(); }

void orc_set_threads(int t) { g_threads = t < 1 ? 1 : t; }

// Walled box with nx*ny*nz interior cells, uniform spacing h.
// tile_min: cell count from which a level's DGS is tile-ordered (0: default 256^3; < 0: never).
void* orc_create(int nx, int ny, int nz, double h, double eta, double gamma, int levels, int nu, int band_width,
                 int64_t tile_min) {
    try {
        CellGrid g;
        g.dim = 3;
        g.n[0] = nx;
        g.n[1] = ny;
        g.n[2] = nz;
        g.h = h;
        g.lab.assign(static_cast<size_t>(nx) * ny * nz, LAB_I);
        auto* o = new OrcHandle();
        o->H = build_hierarchy(g, eta, gamma, levels, nu, band_width,
                               tile_min < 0 ? std::numeric_limits<int64_t>::max() : tile_min);
        return o;
    } catch (const std::exception& e) {
        g_last_err = e.what();
        return nullptr;
    }
}
// General labelled domain: lab[(z * ny + y) * nx + x] in {0 Dirichlet, 1 Interior,
// 2 Exterior} inside an implicit Dirichlet ring; DGS never tile-ordered.
void* orc_create_labeled(int nx, int ny, int nz, double h, const uint8_t* lab, double eta, double gamma, int levels,
                         int nu, int band_width) {
    try {
        CellGrid g;
        g.dim = 3;
        g.n[0] = nx;
        g.n[1] = ny;
        g.n[2] = nz;
        g.h = h;
        g.lab.assign(lab, lab + static_cast<size_t>(nx) * ny * nz);
        for (uint8_t l : g.lab)
            if (l > LAB_E) throw std::runtime_error("labels must be 0 (D), 1 (I) or 2 (E)");
        auto* o = new OrcHandle();
        o->H = build_hierarchy(g, eta, gamma, levels, nu, band_width, std::numeric_limits<int64_t>::max());
        return o;
    } catch (const std::exception& e) {
        g_last_err = e.what();
        return nullptr;
    }
}
void orc_destroy(void* h) { delete static_cast<OrcHandle*>(h); }

static Hierarchy& HH(void* h) { return *static_cast<OrcHandle*>(h)->H; }
static vec V(const double* p, int64_t n) { return vec(p, p + n); }
static void out(const vec& v, double* p) { std::memcpy(p, v.data(), v.size() * sizeof(double)); }

int orc_nlevels(void* h) { return static_cast<int>(HH(h).lv.size()); }
int64_t orc_ndof(void* h, int l) { return HH(h).lv[l]->map.N; }
void orc_counts(void* h, int l, int64_t* c5) {
    const DofMap& m = HH(h).lv[l]->map;
    for (int k = 0; k < 4; ++k) c5[k] = m.cnt[k];
    int64_t v1 = 0;
    for (uint8_t f : m.v1) v1 += f;
    c5[4] = v1;
}
void orc_v1_mask(void* h, int l, uint8_t* mask) {
    const DofMap& m = HH(h).lv[l]->map;
    std::memcpy(mask, m.v1.data(), m.v1.size());
}
void orc_set_skip_reverse(void* h, int s) { HH(h).skip_reverse = s != 0; }
void orc_set_cycle(void* h, int kind) { HH(h).cycle = kind; }
// 0: the GPU's smoother order (OD-1/OD-2); 1: SPEC-literal sequential order (comparison mode)
void orc_set_order(void* h, int order) { HH(h).order = order; }
// DGS tiling of level l: out4 = {ntc, tile_x, tile_y, tile_z}
void orc_dgs_tile(void* h, int l, int* out4) {
    const Level& L = *HH(h).lv[l];
    out4[0] = L.ntc;
    for (int a = 0; a < 3; ++a) out4[1 + a] = L.tile[a];
}
// Vanka flavour: kind 0 symmetric multiplicative, 1 additive with damping omega.
void orc_set_vanka(void* h, int kind, double omega) {
    HH(h).vanka.kind = kind;
    HH(h).vanka.omega = omega;
}
int orc_mg_solve(void* h, const double* b, double* x, double tol, int maxit, double* hist, double* secs, int* iters) {
    Hierarchy& H = HH(h);
    const int64_t n = H.lv[0]->map.N;
    vec xx, hh, ss;
    const int st = mg_solve(H, V(b, n), xx, tol, maxit, hh, ss);
    out(xx, x);
    for (size_t k = 0; k < hh.size(); ++k) { hist[k] = hh[k]; secs[k] = ss[k]; }
    *iters = static_cast<int>(hh.size());
    return st;
}

void orc_apply(void* h, int l, int penalized, const double* x, double* y) {
    const Level& L = *HH(h).lv[l];
    vec yy;
    apply(L, V(x, L.map.N), yy, penalized != 0);
    out(yy, y);
}
void orc_residual(void* h, int l, const double* x, const double* b, double* r) {
    const Level& L = *HH(h).lv[l];
    vec rr;
    residual(L, V(x, L.map.N), V(b, L.map.N), rr);
    out(rr, r);
}
// op: 0 one DGS phase (arg = phase 0..19), 1 symmetric DGS, 2 one Vanka colour
// (arg = colour), 3 symmetric Vanka, 4 smooth (Alg. 3), 5 one additive Vanka, 7 one direct-on-V1 solve.
int orc_smoother(void* h, int l, int op, int arg, double* x, const double* b) {
    try {
        Hierarchy& H = HH(h);
        const Level& L = *H.lv[l];
        vec xx = V(x, L.map.N), bb = V(b, L.map.N);
        DgsScratch scratch;
        if (op == 0) dgs_phase(L, xx, bb, arg & 31, arg >> 5, scratch);
        else if (op == 1) symmetric_dgs(L, xx, bb, H.skip_reverse, H.order);
        else if (op == 2) vanka_colour(L, xx, bb, arg);
        else if (op == 3) vanka_symmetric(L, xx, bb, H.order);
        else if (op == 4) smooth(L, xx, bb, H.nu, H.skip_reverse, H.vanka, H.order);
        else if (op == 5) vanka_additive(L, xx, bb, H.vanka.omega);
        else if (op == 7) vanka_direct(L, xx, bb);
        else throw std::runtime_error("bad smoother op");
        out(xx, x);
        return 0;
    } catch (const std::exception& e) {
        g_last_err = e.what();
        return -1;
    }
}
void orc_restrict(void* h, int lf, const double* rf, double* rc) {
    Hierarchy& H = HH(h);
    vec o;
    restrict_(*H.lv[lf], *H.lv[lf + 1], V(rf, H.lv[lf]->map.N), o);
    out(o, rc);
}
void orc_prolong(void* h, int lf, const double* xc, double* xf) {
    Hierarchy& H = HH(h);
    vec o;
    prolong(*H.lv[lf], *H.lv[lf + 1], V(xc, H.lv[lf + 1]->map.N), o);
    out(o, xf);
}
void orc_coarse_solve(void* h, const double* b, double* x) {
    Hierarchy& H = HH(h);
    vec o;
    coarse_solve(H, V(b, H.lv.back()->map.N), o);
    out(o, x);
}
void orc_vcycle(void* h, const double* b, double* x) {
    Hierarchy& H = HH(h);
    vec o;
    vcycle(H, 0, V(b, H.lv[0]->map.N), o);
    out(o, x);
}
// Dense L (penalized=0) or L̃ (1) of level l into a (N x N row-major, caller-sized).
void orc_assemble_dense(void* h, int l, int penalized, double* a) {
    const Level& L = *HH(h).lv[l];
    auto d = assemble_dense(L, penalized != 0);
    std::memcpy(a, d.data(), d.size() * sizeof(double));
}
void orc_coarse_inverse(void* h, double* k) {
    Hierarchy& H = HH(h);
    std::memcpy(k, H.coarse_inv.data(), H.coarse_inv.size() * sizeof(double));
}
// returns status; hist/secs sized maxit; *iters = number of history entries
int orc_sqmr(void* h, const double* b, double* x, double tol, int maxit, int precond, double* hist,
             double* secs, int* iters) {
    Hierarchy& H = HH(h);
    const int64_t n = H.lv[0]->map.N;
    vec xx, hh, ss;
    const int st = sqmr(H, V(b, n), xx, tol, maxit, precond, hh, ss);
    out(xx, x);
    for (size_t k = 0; k < hh.size(); ++k) { hist[k] = hh[k]; secs[k] = ss[k]; }
    *iters = static_cast<int>(hh.size());
    return st;
}
double orc_cdot(void* h, const double* a, const double* b) {
    const Level& L = *HH(h).lv[0];
    return cdot(L, V(a, L.map.N), V(b, L.map.N));
}
void orc_forcing(void* h, int kind, uint64_t seed, double* b) {
    const Level& L = *HH(h).lv[0];
    vec bb;
    forcing(L, kind, seed, bb);
    out(bb, b);
}
static double g_forcing_eta = 1.0;  // eta used by the lid (Dirichlet) contributions of forcing_box
void orc_set_forcing_eta(double eta) { g_forcing_eta = eta; }
// Forcing on a walled box without building a hierarchy (no coarse factorisation).
void orc_forcing_box(int nx, int ny, int nz, double h, int kind, uint64_t seed, double* b) {
    CellGrid g;
    g.dim = 3;
    g.n[0] = nx;
    g.n[1] = ny;
    g.n[2] = nz;
    g.h = h;
    g.lab.assign(static_cast<size_t>(nx) * ny * nz, LAB_I);
    Level L;
    L.map = classify(g, 1);
    L.h = h;
    L.eta_h2 = g_forcing_eta / (h * h);
    L.inv_h = 1.0 / h;
    vec bb;
    forcing(L, kind, seed, bb);
    out(bb, b);
}
// assemble_rhs on a labelled grid with general Dirichlet data: b += the stencil
// legs into Dirichlet faces.  g[c] holds the face values of component c over the extents
// n_a + 1 along its own axis and n_a + 2 along the others (tangential index shifted by one: the
// ring faces -1 and n_a are included), x fastest.
void orc_dirichlet_rhs(void* h, const double* gu, const double* gv, const double* gw, double* b) {
    Hierarchy& H = HH(h);
    const Level& L = *H.lv[0];
    const double* g[3] = {gu, gv, gw};
    const int n[3] = {L.map.n[0], L.map.n[1], L.map.n[2]};
    vec bb = V(b, L.map.N);
    dirichlet_rhs_g(L, bb, [&](int c, int x, int y, int z) {
        const int p[3] = {x, y, z};
        int e[3], q[3];
        for (int a = 0; a < 3; ++a) {
            e[a] = n[a] + (a == c ? 1 : 2);
            q[a] = p[a] + (a == c ? 0 : 1);
            if (q[a] < 0 || q[a] >= e[a]) return 0.0;
        }
        return g[c][(static_cast<size_t>(q[2]) * e[1] + q[1]) * e[0] + q[0]];
    });
    out(bb, b);
}

void orc_census_box(int dim, int nx, int ny, int nz, int width, int64_t* out2) {
    census_box(dim, nx, ny, nz, width, out2);
}
// Generic coarsening check on an explicit label array.
void orc_coarsen_labels(int dim, int nx, int ny, int nz, const uint8_t* lab, uint8_t* out_lab) {
    CellGrid g;
    g.dim = dim;
    g.n[0] = nx;
    g.n[1] = ny;
    g.n[2] = dim == 3 ? nz : 1;
    g.lab.assign(lab, lab + static_cast<size_t>(g.n[0]) * g.n[1] * g.n[2]);
    CellGrid c = coarsen(g);
    std::memcpy(out_lab, c.lab.data(), c.lab.size());
}
// Census of an explicit label array: out = {N, |V1|, n_u, n_v, n_w, n_p}.
void orc_census_labels(int dim, int nx, int ny, int nz, const uint8_t* lab, int width, int64_t* out6) {
    CellGrid g;
    g.dim = dim;
    g.n[0] = nx;
    g.n[1] = ny;
    g.n[2] = dim == 3 ? nz : 1;
    g.lab.assign(lab, lab + static_cast<size_t>(g.n[0]) * g.n[1] * g.n[2]);
    DofMap m = classify(g, width);
    int64_t v1 = 0;
    for (uint8_t f : m.v1) v1 += f;
    out6[0] = m.N;
    out6[1] = v1;
    for (int k = 0; k < 4; ++k) out6[2 + k] = m.cnt[k];
}

}  // extern "C"
