// smg_internal.h — device layout and kernel launchers of the B200 MG-SQMR path.
//
// HBM layout: every level vector is four padded SoA boxes
// [u | v | w | p], one per field, each with slots [-1, n_a] along every axis a
// (a one-slot ghost ring).  u-face x-index I (I = 0 and I = nx are the wall
// faces) lives at x-slot I, so all four fields share one slot index per cell:
// the faces on the low side of cell (x,y,z) and its pressure all sit at
// slot(x,y,z).  Ghost and wall slots hold 0 forever (kernels never write
// them), which realises the homogeneous Dirichlet ring without branches.
// Rows are padded so that x = 0 is 32-byte aligned: slot x lives at row
// offset x + 4, pitch px = round_up(nx + 5, 8) doubles.
#pragma once

#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

namespace smg {

struct Geom {
    int nx, ny, nz;      // interior cells held (nz = local planes of a z-slab)
    int px, py, pz;      // padded extents (doubles)
    int64_t sy, sz;      // strides of y and z
    int64_t fs;          // stride between fields of one vector (multiple of 32)
    int xo;              // row offset of slot x = 0 (4: 32-byte aligned rows; 1: compact small levels)
    int zg;              // ghost planes on each z side (1 whole level; 2 for z-slabs: radius-2 halos)
    int z0, gnz;         // global z of local plane 0, global number of planes
    __host__ __device__ __forceinline__ int64_t slot(int x, int y, int z) const {
        return static_cast<int64_t>(z + zg) * sz + static_cast<int64_t>(y + 1) * sy + (x + xo);
    }
    __host__ __device__ __forceinline__ int gz(int z) const { return z + z0; }  // local -> global plane
    int64_t vec_len() const { return 4 * fs; }
};

// Levels whose whole vector fits in one SM's shared memory use a compact
// layout (x-offset 1, unaligned pitch) so a CTA can smooth them in smem.
constexpr int64_t kSmemLevelCells = 6144;

// Whole level (z0 = 0, nz = gnz) or a z-slab [z0, z0 + nzl) of a gnz-plane level.
inline Geom make_geom(int nx, int ny, int nz, int z0 = 0, int gnz = -1, int zg = 1) {
    Geom g;
    g.nx = nx;
    g.ny = ny;
    g.nz = nz;
    g.z0 = z0;
    g.gnz = gnz < 0 ? nz : gnz;
    g.zg = zg;
    const bool compact = zg == 1 && gnz < 0 && static_cast<int64_t>(nx + 2) * (ny + 2) * (nz + 2) <= kSmemLevelCells;
    g.xo = compact ? 1 : 4;
    g.px = compact ? nx + 2 : ((nx + 5) + 7) / 8 * 8;
    g.py = ny + 2;
    g.pz = nz + 2 * zg;
    g.sy = g.px;
    g.sz = static_cast<int64_t>(g.px) * g.py;
    const int64_t cells = g.sz * g.pz;
    g.fs = (cells + 31) / 32 * 32;
    return g;
}

// Per-level operator constants (LevelOperator).
struct LevelK {
    Geom g;
    double eta_h2;  // eta / h^2
    double inv_h;   // 1 / h
    double gamma;   // penalty of L~
    double dv;      // DGS diagonal, velocity: 6 eta / h^2
    double dp;      // DGS diagonal, pressure: -6 (1 + gamma eta) / h^2
    int bw;         // band width
    // c_b = m_C^T b per cell (the b part of the reverse DGS pressure update, fixed while b
    // is): launch_dgs_cb fills it before a sweep; prev steps then read L~x only
    double* cb = nullptr;
    // tiled levels: b and c_b in tile-major order (5 x 1024 doubles per tile), filled by launch_dgs_cb
    double* bp = nullptr;
    int tiled = 0;  // DGS sweep in tile order (OD-1 rev. 2, dgs_tiled)
    // General labelled domain: per cell slot (one field long, ghosts 0) the DofMap
    // bits CLS_* of the cell's pressure and its three low faces; nullptr on the walled box,
    // whose statuses are analytic.
    const uint32_t* cls = nullptr;
};

// DofMap bits of a cell slot on a labelled level (classify_dofs SPEC:45-53, partition_band
// SPEC:63-71): active pressure / low u, v, w face; band cell; low faces in V2; and per low face
// its momentum diagonal 6 - (dropped Neumann legs) in 3 bits from bit 8 + 3 comp.
constexpr uint32_t CLS_P = 1, CLS_U = 2, CLS_V = 4, CLS_W = 8, CLS_BAND = 16, CLS_U2 = 32, CLS_V2 = 64, CLS_W2 = 128;
constexpr int CLS_DIAG_SHIFT = 8;

// ---- stencil launchers (kernels.cu) ----
// y = L~x (gamma) or, with b != nullptr, y = b - L~x, on active slots only.
void launch_apply(const LevelK& L, const double* x, const double* b, double* y, double gamma, cudaStream_t s);
void launch_dgs_vel(const LevelK& L, double* x, const double* b, int colour, cudaStream_t s);
void launch_dgs_pdelta(const LevelK& L, const double* x, const double* b, double* delta, int colour,
                       cudaStream_t s);
// colour: the parity colour whose deltas `delta` holds (labelled levels touch only its neighbourhood)
void launch_dgs_papply(const LevelK& L, double* x, const double* delta, cudaStream_t s, int colour = -1);
void launch_dgs_prev(const LevelK& L, double* x, const double* b, int colour, cudaStream_t s);
// L.cb[C] = m_C^T b for every cell (reverse pressure phases need it; call when b changes).
void launch_dgs_cb(const LevelK& L, const double* b, cudaStream_t s);
// Vanka colour order (oracle kVankaOrder = 0,7,1,6,2,5,3,4): the parity colour visited at
// step j (0..7) of a forward sweep; the reverse sweep visits them backwards.
#ifdef __CUDACC__
__host__ __device__
#endif
inline constexpr int vanka_order(int j) { return (j & 1) ? 7 - (j >> 1) : (j >> 1); }
// Merged complementary pairs: bit m of `pairs` set -> list m holds parity m (first first[m]
// entries) then parity 7-m, and list 7-m is empty (one Jacobi phase for both colours).
struct VankaPairs {
    int pairs = 0;
    int first[4] = {0, 0, 0, 0};
};
// kidx (labelled levels): per block the index of its signature class in ktab (nullptr: the face mask)
void launch_vanka_delta(const LevelK& L, const double* x, const double* b, const int32_t* cells,
                        const uint8_t* masks, int ncells, const double* ktab, double* delta, cudaStream_t s,
                        const uint16_t* kidx = nullptr);
// amask (z-slabs, optional): per block, the slots this part owns (bit s = slot s, bit 6 = p).
void launch_vanka_apply(const LevelK& L, double* x, const int32_t* cells, const uint8_t* masks, int ncells,
                        const double* delta, cudaStream_t s, const uint8_t* amask = nullptr);
// Cooperative (persistent, grid-synchronised) symmetric sweeps: nu Vanka sweeps
// over the 8 colour lists; nph DGS phases (20 = full symmetric sweep).
// pr: merged complementary colour pairs (list m = parity m + parity 7-m, one phase
// each; see VankaLists in kernels.cu).
// xb (optional): second level vector for the ping-pong sweep (one barrier per
// phase); refresh[0..nrefresh) lists the slots Vanka reads, copied x -> xb first.
void launch_vanka_sym_coop(const LevelK& L, double* x, const double* b, const int32_t* const* cells,
                           const uint8_t* const* masks, const int* n, const double* ktab, double* delta, int nu,
                           cudaStream_t s, double* xb = nullptr, const int32_t* refresh = nullptr,
                           int64_t nrefresh = 0, const VankaPairs& pr = VankaPairs{});
int vanka_pairs_pay(const int* n);  // mask of the pairs to merge on a level with these list sizes
// One kernel per step (13 steps for the 20 phases); xb, d1 unused.
void launch_dgs_sym_coop(const LevelK& L, double* x, const double* b, double* d0, double* d1, int nph,
                         cudaStream_t s, double* xb = nullptr);
// Restriction of coarse LOCAL planes [zc_lo, zc_lo + nzc) (nzc < 0: all); the
// fine slab must hold the fine planes 2zc-1 .. 2zc+2 (halos included).
void launch_restrict(const LevelK& F, const LevelK& C, const double* rf, double* bc, cudaStream_t s, int zc_lo = 0,
                     int nzc = -1);
void launch_prolong_add(const LevelK& F, const LevelK& C, const double* xc, double* xf, cudaStream_t s);
// x[slots] = K b[slots] (accumulate: x[slots] += K b[slots], the direct-on-V1 correction)
void launch_coarse_gemv(const double* ksym, const int32_t* slots, int n, const double* b, double* x,
                        cudaStream_t s, bool accumulate = false);
void launch_pack(const LevelK& L, const double* padded, double* compact, cudaStream_t s);
void launch_unpack(const LevelK& L, const double* compact, double* padded, cudaStream_t s);
// labelled levels: compact[k] = padded[slots[k]] / padded[slots[k]] = compact[k], k < n
void launch_gather(const int32_t* slots, int64_t n, const double* padded, double* compact, cudaStream_t s);
void launch_scatter(const int32_t* slots, int64_t n, const double* compact, double* padded, cudaStream_t s);

// ---- BLAS-1 (kernels.cu); n = padded vector length (multiple of 32) ----
// Canonical inner products (OD-12 rev. 2): block partials over 32 x 8 cells x
// 4 planes at global block indices, then one fixed-order final.  dot_partials(g): doubles of a
// partial buffer for the fine level (two products).
int64_t dot_partials(const Geom& g);
constexpr int kDotZBlock = 4;  // planes per dot block: fine-level slabs start and end on a z-block
// a.b and, if c != nullptr, c.d -> out[0], out[1] on the device
void launch_cdot2(const Geom& g, const double* a, const double* b, const double* c, const double* d,
                  double* partials, double* out, cudaStream_t s);
// the two halves of launch_cdot2: this part's block partials, and the final over all blocks
void launch_cdot_planes(const Geom& g, const double* a, const double* b, const double* c, const double* d,
                        double* partials, cudaStream_t s);
void launch_cdot_final(const Geom& g, const double* partials, double* out, cudaStream_t s);
// final over the partials into sc[S_D0..1] + the Alg. 4 scalar update `which` (0 first, 1 alpha,
// 2 nu/c/tau/cd/cq, 3 rel/convergence/beta, -1 none)
void launch_final_scalar(const Geom& g, const double* partials, double* sc, int which, cudaStream_t s);
// fused SQMR steps (kernels.cu k_apply_q / k_apply_x): q1 = t + beta q0, tn = L q1 and the
// partials of q1.tn; x1 = x0 + (cd d0 + cq q), d1 = cd d0 + cq q and the partials of
// ||b - L x1||^2.  halo_lo/hi (slab parts): also write the ghost plane below / above.
void launch_apply_q(const LevelK& L, const double* t, const double* q0, double* q1, double* tn, const double* sc,
                    double* partials, int halo_lo, int halo_hi, cudaStream_t s, int second = 0);
void launch_apply_x(const LevelK& L, const double* x0, const double* d0, const double* q, const double* b, double* x1,
                    double* d1, const double* sc, double* partials, int halo_lo, int halo_hi, cudaStream_t s);
// Tile-ordered DGS (OD-1 rev. 2): a level is tiled iff it has >= tile_min cells (0: 256^3,
// < 0: never) and its extents are multiples of the tile (16 x 8 x 8) with >= 2 tiles per axis.
bool dgs_tiled(int nx, int ny, int nz, int64_t tile_min);
int dgs_tile_dim(int axis);
// phases [ph0, ph1) of the 20-phase numbering on the tiles of colour T
void launch_dgs_tile_phases(const LevelK& L, double* x, const double* b, int T, int ph0, int ph1, cudaStream_t s,
                            int zsel = 0, bool packed = false);
// symmetric sweep (nph = 20) or forward half (nph = 10) in tile order; L.cb must hold m^T b
void launch_dgs_tiled(const LevelK& L, double* x, const double* b, int nph, cudaStream_t s, bool packed = false);
// Single colour-compact DGS phases (used by the z-slab path).
void launch_dgs_vel_c(const LevelK& L, double* x, const double* b, int colour, cudaStream_t s);
void launch_dgs_pf_delta_c(const LevelK& L, const double* x, const double* b, double* d, int c, cudaStream_t s);
void launch_dgs_pf_apply_c(const LevelK& L, double* x, const double* d, int c, cudaStream_t s);
void launch_dgs_prev_c(const LevelK& L, double* x, const double* b, int c, cudaStream_t s);
int64_t frame_doubles(const Geom& g, int bw);
void launch_frame_copy(const Geom& g, int bw, double* x, double* buf0, int zs0, double* buf1, int zs1, bool to_buf,
                       cudaStream_t s);
void launch_axpy(double* y, const double* x, double alpha, int64_t n, cudaStream_t s);          // y += alpha x
void launch_xpby(double* y, const double* x, double beta, int64_t n, cudaStream_t s);           // y = x + beta y
void launch_dx_update(double* d, double* x, const double* q, double cd, double cq, int64_t n,
                      cudaStream_t s);  // d = cd d + cq q; x = x + d

// SQMR scalar slots in device memory (Alg. 4 state + dot results).
enum SqmrSlot {
    S_D0 = 0, S_D1 = 1, S_BNORM = 2, S_TAU = 3, S_NUOLD = 4, S_RHO = 5, S_ALPHA = 6, S_NU = 7, S_CD = 8,
    S_CQ = 9, S_RHONEW = 10, S_BETA = 11, S_REL = 12, S_STATUS = 13, S_TOL = 14, S_COUNT = 16
};
// status slot: 0 running, 1 converged, 2 breakdown before the residual (sigma), 3 breakdown after it (rho).
// One additive Vanka application over all n band blocks (any order);
// d7: scratch of 7 fields (g.fs each).  Bit-identical to the oracle's fixed order.
void launch_vanka_additive(const LevelK& L, double* x, const double* b, const int32_t* cells, const uint8_t* masks,
                           int n, const double* ktab, double* d7, double omega, cudaStream_t s,
                           const uint16_t* kidx = nullptr);
void launch_axpy_s(double* s_, const double* t, const double* sc, int64_t n, cudaStream_t s);

// Number of our kernels launched so far (per process), for the bench's gpu_launches.
int64_t launch_count();
// First rejected launch (cudaError_t) since the last call, 0 if none.
int take_launch_error();

}  // namespace smg
