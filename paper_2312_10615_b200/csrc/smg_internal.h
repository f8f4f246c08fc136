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
#include <cuda_runtime.h>

namespace smg {

struct Geom {
    int nx, ny, nz;      // interior cells
    int px, py, pz;      // padded extents (doubles)
    int64_t sy, sz;      // strides of y and z
    int64_t fs;          // stride between fields of one vector (multiple of 32)
    __host__ __device__ __forceinline__ int64_t slot(int x, int y, int z) const {
        return static_cast<int64_t>(z + 1) * sz + static_cast<int64_t>(y + 1) * sy + (x + 4);
    }
    int64_t vec_len() const { return 4 * fs; }
};

inline Geom make_geom(int nx, int ny, int nz) {
    Geom g;
    g.nx = nx;
    g.ny = ny;
    g.nz = nz;
    g.px = ((nx + 5) + 7) / 8 * 8;
    g.py = ny + 2;
    g.pz = nz + 2;
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
};

// ---- stencil launchers (kernels.cu) ----
// y = L~x (gamma) or, with b != nullptr, y = b - L~x, on active slots only.
void launch_apply(const LevelK& L, const double* x, const double* b, double* y, double gamma, cudaStream_t s);
void launch_dgs_vel(const LevelK& L, double* x, const double* b, int colour, cudaStream_t s);
void launch_dgs_pdelta(const LevelK& L, const double* x, const double* b, double* delta, int colour,
                       cudaStream_t s);
void launch_dgs_papply(const LevelK& L, double* x, const double* delta, cudaStream_t s);
void launch_dgs_prev(const LevelK& L, double* x, const double* b, int colour, cudaStream_t s);
void launch_vanka_delta(const LevelK& L, const double* x, const double* b, const int32_t* cells,
                        const uint8_t* masks, int ncells, const double* ktab, double* delta, cudaStream_t s);
void launch_vanka_apply(const LevelK& L, double* x, const int32_t* cells, const uint8_t* masks, int ncells,
                        const double* delta, cudaStream_t s);
void launch_restrict(const LevelK& F, const LevelK& C, const double* rf, double* bc, cudaStream_t s);
void launch_prolong_add(const LevelK& F, const LevelK& C, const double* xc, double* xf, cudaStream_t s);
void launch_coarse_gemv(const double* ksym, const int32_t* slots, int n, const double* b, double* x,
                        cudaStream_t s);
void launch_pack(const LevelK& L, const double* padded, double* compact, cudaStream_t s);
void launch_unpack(const LevelK& L, const double* compact, double* padded, cudaStream_t s);

// ---- BLAS-1 (kernels.cu); n = padded vector length (multiple of 32) ----
constexpr int kPartials = 2 * (4 * 1025 + 4);  // scratch doubles for launch_cdot2
// Canonical (bit-reproducible, oracle-identical) a.b and, if c != nullptr,
// c.d over the level geometry g -> out[0], out[1] on the device.  nz <= 1024.
void launch_cdot2(const Geom& g, const double* a, const double* b, const double* c, const double* d,
                  double* partials, double* out, cudaStream_t s);
void launch_axpy(double* y, const double* x, double alpha, int64_t n, cudaStream_t s);          // y += alpha x
void launch_xpby(double* y, const double* x, double beta, int64_t n, cudaStream_t s);           // y = x + beta y
void launch_dx_update(double* d, double* x, const double* q, double cd, double cq, int64_t n,
                      cudaStream_t s);  // d = cd d + cq q; x = x + d

// Number of our kernels launched so far (per process), for the bench's gpu_launches.
int64_t launch_count();

}  // namespace smg
