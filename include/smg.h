/*
 * smg.h — C-ABI of the B200-native MG-preconditioned SQMR Stokes solver.
 *
 * Drop-in boundary for the hot path of arXiv 2312.10615.  The
 * reference ships only proj/include/stokesmg/util.hpp (kept verbatim in
 * signature as include/stokesmg/util.hpp); its solver exists only as the
 * behavioural spec SPEC.md, so every entry point below cites the SPEC
 * operation it replaces.  The host C++ API (include/stokesmg/solver.hpp) and
 * the Python tests call exactly these symbols; plain pointers and sizes only.
 *
 * Vectors crossing the boundary are the SPEC's compact FieldVector: the active
 * DOFs of one level numbered u-lex, v-lex, w-lex, p-lex, x fastest
 * (SPEC:34-42, 48, 84, 111-114).  The context owns all device memory.
 * Return values: 0 on success, negative smg_err on failure (details in
 * smg_last_error).  Solver status is reported separately.
 * A context is not thread-safe; distinct contexts are independent.
 */
#ifndef SMG_H
#define SMG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct smg_ctx smg_ctx;

enum smg_err {
    SMG_OK = 0,
    SMG_EINVAL = -1,   /* bad argument / length mismatch   */
    SMG_ECUDA = -2,    /* CUDA runtime error                                  */
    SMG_ENCCL = -3,    /* NCCL error                                          */
    SMG_ECAP = -4,     /* coarsest system above the dense cap      */
    SMG_ENOMEM = -5,   /* device allocation failed                            */
    SMG_ESINGULAR = -6 /* singular local/coarse matrix             */
};

enum smg_status {
    SMG_CONVERGED = 0,
    SMG_MAX_ITERATIONS = 1,
    SMG_BREAKDOWN = 2
};

/* Walled box: nx*ny*nz interior cells of spacing h inside an implicit no-slip
 * Dirichlet ring (cube and channel configs of BASELINE.json). */
typedef struct smg_grid_desc {
    int dim; /* must be 3 */
    int nx, ny, nz;
    double h;
} smg_grid_desc;

/* SmootherConfig + CycleConfig + LevelOperator parameters. */
typedef struct smg_params {
    double eta;      /* viscosity eta                                  */
    double gamma;    /* penalty gamma of L~ (preconditioner only)      */
    int levels;      /* V-cycle levels n >= 1                          */
    int nu;          /* symmetric multiplicative Vanka sweeps per side */
    int band_width;  /* V1 band width (Chebyshev)                      */
    int flags;       /* SMG_FLAG_*                                     */
    int cycle;       /* 0 V-cycle, 1 W-cycle       */
    int vanka;       /* 0 symmetric multiplicative, 1 additive, 2 direct solve on V1
                        (dense, |V1| <= 20000, benchmarking mode) */
    double omega;    /* additive damping in (0, 1]; <= 0 means 1.0 (SPEC default) */
    int64_t dgs_tile_min; /* DGS traversal (OD-1 rev. 2): levels with >= this many cells whose
                             extents are multiples of 16 x 8 x 8 (>= 2 tiles per axis) sweep
                             their DGS tile by tile; 0: 256^3 (default), < 0: never */
} smg_params;

#define SMG_FLAG_SKIP_REVERSE_DGS 1 /* fault injection: symmetry negative control */
#define SMG_FLAG_NO_PRECOND 2       /* solve_driver method `sqmr`: smg_sqmr_solve runs
                                      Alg. 4 with the identity preconditioner, t = s */

/* ResidualHistory: caller-owned arrays of `capacity` entries. */
typedef struct smg_history {
    int capacity;
    int count;
    double* rel_residual; /* ||b - L x_j|| / ||b||                 */
    double* seconds;      /* wall seconds since solve start       */
} smg_history;

/* Timing of the last solve, measured with CUDA events on the solver stream. */
typedef struct smg_timing {
    double solve_ms;        /* SQMR loop on device-resident data           */
    double h2d_ms, d2h_ms;  /* host<->device transfers of the last e2e call */
    int iterations;
    int64_t kernel_launches; /* own kernels launched during the solve      */
} smg_timing;

/* build_hierarchy: grids, operators, transfers, Vanka tables,
 * coarse dense inverse; uploads everything.  ngpu > 1 builds a z-slab
 * decomposition over the listed devices (a device may repeat: parts then share
 * it, which emulates the multi-GPU data path on one GPU); see smg_slab_plan.
 * Results are bit-identical for every ngpu. */
int smg_create(const smg_grid_desc* grid, const smg_params* params, int ngpu, const int* dev_ids,
               smg_ctx** out);
/* General labelled domain (PAPER section 5): labels[(z*ny + y)*nx + x] is the CellLabel
 * of cell (x, y, z) -- 0 Dirichlet, 1 Interior, 2 Exterior -- inside the implicit
 * Dirichlet ring.  classify_dofs: a face between two Interior cells is
 * active, a face of a Dirichlet cell carries the value 0, a face touching an Exterior cell is
 * Inactive (homogeneous Neumann: its stencil legs are dropped); pressures are active
 * in Interior cells.  coarsen_grid labels the coarser levels, partition_band
 * gives V1 / V2, Vanka blocks are factorised once per signature class.
 * Extents must be divisible by 2^(levels-1) (pad with Exterior cells).  One GPU; the
 * smoother runs one kernel per phase (no DGS tiling), every params.vanka flavour.  Every other entry
 * point works on the context; vectors are the compact FieldVector of this DofMap. */
int smg_create_labeled(const smg_grid_desc* grid, const uint8_t* labels, const smg_params* params, int device,
                       smg_ctx** out);
/* coarsen_grid, host only: out holds (nx/2)(ny/2)(nz/2) labels; even extents. */
int smg_coarsen_labels(const smg_grid_desc* grid, const uint8_t* labels, uint8_t* out);
/* classify_dofs + partition_band census of a labelled grid (host only):
 * out6 = {N, |V1|, n_u, n_v, n_w, n_p}; returns N. */
int64_t smg_census_labeled(const smg_grid_desc* grid, const uint8_t* labels, int band_width, int64_t* out6);
/* smg_forcing on the active faces of a labelled grid (same generator: a function of the seed,
 * the component and the face's storage coordinates). */
int smg_forcing_labeled(const smg_grid_desc* grid, const uint8_t* labels, int kind, uint64_t seed, double* b);

/* assemble_rhs on a labelled grid with general BoundaryData, host
 * only: b += the stencil legs of the active rows into Dirichlet-valued faces.  g_c holds the
 * Dirichlet velocity of every face of component c over n_a + 1 faces along its own axis and
 * n_a + 2 along the two others (tangential index shifted by one, so the faces of the ring cells,
 * coordinates -1 and n_a, are included), x fastest; entries at non-Dirichlet faces are ignored.
 * b is the compact FieldVector of the grid's DofMap (add the body force before or after). */
int smg_assemble_rhs_labeled(const smg_grid_desc* grid, const uint8_t* labels, double eta, const double* gu,
                             const double* gv, const double* gw, double* b);

/* Multi-process z-slab decomposition: one process per GPU, NCCL over NVLink.
 * Rank 0 calls smg_nccl_unique_id and the caller's launcher (torch.distributed,
 * MPI, ...) broadcasts the 128-byte id; every rank then calls smg_create_rank
 * with its own device.  The context holds the rank's slab of the distributed
 * levels (smg_slab_plan) and a replicated copy of the coarser ones; halo planes
 * travel by ncclSend/ncclRecv with the z neighbours, the canonical plane
 * partials of every inner product by one ncclAllReduce, the restricted residual
 * of the first replicated level by ncclAllGather.  Every later call on the
 * context is collective (same calls, same order on all ranks); host vectors
 * are the full compact FieldVector on every rank.  Results are bit-identical
 * to one GPU.  libnccl.so.2 is loaded at run time (SMG_NCCL_LIB overrides the
 * name), so single-process contexts never need NCCL. */
int smg_nccl_unique_id(unsigned char id[128]);
int smg_create_rank(const smg_grid_desc* grid, const smg_params* params, int rank, int nranks, int device,
                    const unsigned char id[128], smg_ctx** out);
void smg_destroy(smg_ctx* ctx);
/* assemble_rhs, host only: adds the Dirichlet-data contributions
 * of a scenario to b (compact order).  scenario 0: lid-driven cavity (PAPER:368,
 * 434), tangential u = value on the top (y = ny) lid, no-slip elsewhere. */
int smg_assemble_rhs(const smg_grid_desc* grid, double eta, int scenario, double value, double* b);
/* DOF census of the walled box (host only): out2 = {N, |V1|}; returns N
 * (classify_dofs + partition_band counts; PAPER Table 1). */
int64_t smg_census(const smg_grid_desc* grid, int band_width, int64_t* out2);
/* z-slab plan (host only, no device needed): returns the number of leading
 * levels split over nparts (>= 1, or <= 0 if the grid cannot be split), and for
 * `rank` the first global plane z0[l] and plane count nzl[l] of every level
 * (replicated levels: 0 and the whole level).  Either array may be NULL.  A level is
 * split while its slab keeps >= 2 planes, an even count, tile alignment on tiled levels, and
 * (levels >= 1) at least 64^3 cells -- smaller levels are gathered (SMG_SLAB_MIN_CELLS overrides). */
int smg_slab_plan(const smg_grid_desc* grid, int levels, int nparts, int rank, int* z0, int* nzl);
/* DGS tiling of a level (host only): out4 = {tile colours (8 tiled, 1 not), tile x, y, z}
 * under the rule of smg_params.dgs_tile_min (the default when tile_min = 0). */
int smg_dgs_tile(const smg_grid_desc* grid, int level, int64_t tile_min, int* out4);
const char* smg_last_error(const smg_ctx* ctx);
const char* smg_version(void);

int smg_num_levels(const smg_ctx* ctx);
/* Active DOF counts of a level: out5 = {n_u, n_v, n_w, n_p, |V1|}; returns N. */
int64_t smg_level_ndof(const smg_ctx* ctx, int level, int64_t* out5);

/* discretization.apply: y = L x (penalized = 0) or L~ x. */
int smg_apply(smg_ctx* ctx, int level, int penalized, const double* x, double* y);
/* r = b - L~ x on a level (Alg. 1 line 9). */
int smg_residual(smg_ctx* ctx, int level, const double* x, const double* b, double* r);

/* Smoother entry points.  op: 0 one DGS phase (arg = phase
 * 0..19: forward 0,1 velocity red/black, 2..9 pressure parity colours 0..7;
 * reverse 10..17 pressure colours 7..0, 18,19 velocity black/red; on a tiled
 * level arg = phase + 32 T acts on the tiles of colour T only), 1
 * symmetric_dgs, 2 one Vanka colour (arg = colour 0..7), 3 symmetric
 * multiplicative Vanka, 4 smooth (Alg. 3, with the params' Vanka flavour), 5 one
 * additive Vanka application, 7 one direct-on-V1 solve (params.vanka = 2).  x is
 * updated in place. */
int smg_smoother(smg_ctx* ctx, int level, int op, int arg, double* x, const double* b);

/* transfer between level and level+1: rc = R rf, xf = P xc. */
int smg_restrict(smg_ctx* ctx, int level, const double* rf, double* rc);
int smg_prolong(smg_ctx* ctx, int level, const double* xc, double* xf);
/* exact coarsest solve: x = L~_c^{-1} b on the last level. */
int smg_coarse_solve(smg_ctx* ctx, const double* b, double* x);
/* cycle: x = V-cycle(L~, b, 0). */
int smg_vcycle(smg_ctx* ctx, const double* b, double* x);

/* sqmr_solve with the V-cycle preconditioner: host buffers in,
 * host solution out (end-to-end path).  *status gets an smg_status. */
int smg_sqmr_solve(smg_ctx* ctx, const double* b, double* x, double tol, int maxit, smg_history* hist,
                   int* status);

/* mg_solve: pure multigrid on L~, x_j = x_{j-1} + cycle(b - L~ x_{j-1}),
 * history of ||b - L~ x_j|| / ||b||; single-part contexts. */
int smg_mg_solve(smg_ctx* ctx, const double* b, double* x, double tol, int maxit, smg_history* hist, int* status);

/* Device-resident path used for kernel-level timing: upload b once, solve with
 * everything in HBM, read x back separately. */
int smg_set_rhs(smg_ctx* ctx, const double* b);
int smg_solve_resident(smg_ctx* ctx, double tol, int maxit, smg_history* hist, int* status);
int smg_get_solution(smg_ctx* ctx, double* x);
int smg_last_timing(const smg_ctx* ctx, smg_timing* out);
/* Times `reps` back-to-back launches of one component on `level` (CUDA events
 * on the solver stream, average ms per launch).  which: 0 apply L, 1 residual,
 * 2 symmetric DGS sweep (20 phases), 3 V-cycle from this level, 4 symmetric
 * Vanka sweep(s), 5 smooth (Alg. 3), 6 restrict, 7 prolong-add, 8 coarse
 * solve, 9 fused pair of inner products, 10 axpy, 11 one SQMR iteration graph,
 * 12 the once-per-level-visit m^T b pass (on tiled levels also the tile-major copy
 * of b), 13 / 14 the DGS sweep / the smooth as a V-cycle runs them (12 done before). */
int smg_time_kernel(smg_ctx* ctx, int which, int level, int reps, double* avg_ms);

/* Debug aid (compute-sanitizer is not available on every GPU pool): with SMG_GUARD=1 in the
 * environment at smg_create time every device buffer of the context is allocated between two
 * 4 KiB guard bands; this returns the number of guard bytes any kernel has overwritten so far
 * (0: no out-of-bounds store; always 0 when the guards are off), or a negative smg_err. */
int64_t smg_check_guards(smg_ctx* ctx);

/* Brackets a region for ncu --profile-from-start off (cudaProfilerStart/Stop). */
int smg_profiler_range(int on);

/* Pinned host buffers for the end-to-end path. */
void* smg_host_alloc(int64_t bytes);
void smg_host_free(void* p);

/* Synthetic forcing of the BASELINE configs (OD-9), host side, compact order.
 * kind 0: iid U[-1,1]; 1: 8 Fourier modes; 2: channel 1 + U[-0.1,0.1] on u.
 * b must hold smg_level_ndof(ctx, 0) doubles.  threads <= 1: sequential. */
int smg_forcing(const smg_grid_desc* grid, int kind, uint64_t seed, double* b, int threads);

#ifdef __cplusplus
}
#endif
#endif /* SMG_H */
