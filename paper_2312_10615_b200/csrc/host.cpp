// host.cpp — host driver and C-ABI of the B200 MG-SQMR Stokes solver.
//
// Builds the hierarchy for a walled box, precomputes the Vanka
// local inverses and the coarsest dense inverse (
// OD-4), owns all device memory, and drives the V-cycle (PAPER Alg. 1, 3) and
// SQMR (PAPER Alg. 4) on one CUDA stream.  There is no CPU fallback: every
// numeric step of a solve runs in kernels.cu.  Compiled with
// -ffp-contract=off so the host-side tables (local/coarse inverses, forcing)
// follow the arithmetic contract of DESIGN.md §4.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <type_traits>
#include <unordered_map>
#include <vector>

#include <cuda_profiler_api.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges cost nothing unless a tool (nsys / ncu --nvtx) is attached
#include <nccl.h>  // types only: libnccl.so.2 is loaded at run time (single-process contexts never need it)

#include "../../include/smg.h"
#include "smg_internal.h"

using namespace smg;

namespace {

struct SmgError : std::runtime_error {
    int code;
    SmgError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// NVTX range of a host-side region (solve / iteration / V-cycle level / smooth / transfers): the
// tracing hook of SURVEY §5.  Inside a stream capture it marks the capture, not the replay.
struct Nvtx {
    explicit Nvtx(const char* name) { nvtxRangePushA(name); }
    Nvtx(const char* name, int l) {
        char buf[48];
        std::snprintf(buf, sizeof buf, "%s L%d", name, l);
        nvtxRangePushA(buf);
    }
    ~Nvtx() { nvtxRangePop(); }
    Nvtx(const Nvtx&) = delete;
    Nvtx& operator=(const Nvtx&) = delete;
};

#define CK(call)                                                                                  \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess)                                                                    \
            throw SmgError(SMG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));        \
    } while (0)

// ---- NCCL, resolved with dlopen on first use (multi-process z-slab contexts only) ----
struct NcclApi {
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclCommSplit) commSplit = nullptr;  // optional (NCCL >= 2.18): the halo communicator
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclAllReduce) allReduce = nullptr;
    decltype(&ncclAllGather) allGather = nullptr;
    decltype(&ncclBroadcast) broadcast = nullptr;
    decltype(&ncclGetErrorString) errorString = nullptr;
    std::string err;
};

const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        const char* name = std::getenv("SMG_NCCL_LIB");
        void* h = dlopen(name ? name : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.err = std::string("dlopen libnccl.so.2: ") + dlerror();
            return a;
        }
        auto sym = [&](auto& f, const char* n) { f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, n)); };
        sym(a.getUniqueId, "ncclGetUniqueId");
        sym(a.commInitRank, "ncclCommInitRank");
        sym(a.commDestroy, "ncclCommDestroy");
        sym(a.commSplit, "ncclCommSplit");
        sym(a.groupStart, "ncclGroupStart");
        sym(a.groupEnd, "ncclGroupEnd");
        sym(a.send, "ncclSend");
        sym(a.recv, "ncclRecv");
        sym(a.allReduce, "ncclAllReduce");
        sym(a.allGather, "ncclAllGather");
        sym(a.broadcast, "ncclBroadcast");
        sym(a.errorString, "ncclGetErrorString");
        if (!a.getUniqueId || !a.commInitRank || !a.commDestroy || !a.groupStart || !a.groupEnd || !a.send ||
            !a.recv || !a.allReduce || !a.allGather || !a.broadcast || !a.errorString)
            a.err = "libnccl.so.2: missing symbols";
        return a;
    }();
    if (!api.err.empty()) throw SmgError(SMG_ENCCL, api.err);
    return api;
}

#define NK(call)                                                                                  \
    do {                                                                                          \
        ncclResult_t r_ = (call);                                                                 \
        if (r_ != ncclSuccess)                                                                    \
            throw SmgError(SMG_ENCCL, std::string(#call) + ": " + nccl().errorString(r_));        \
    } while (0)

void host_parallel(int64_t n, int threads, const std::function<void(int64_t, int64_t)>& body) {
    threads = std::max<int>(1, std::min<int64_t>(threads, n));
    if (threads == 1) { body(0, n); return; }
    std::vector<std::thread> ts;
    for (int t = 0; t < threads; ++t) {
        const int64_t lo = n * t / threads, hi = n * (t + 1) / threads;
        ts.emplace_back([lo, hi, &body] { body(lo, hi); });
    }
    for (auto& t : ts) t.join();
}

int host_threads() {
    const unsigned hc = std::thread::hardware_concurrency();
    return hc == 0 ? 1 : static_cast<int>(std::min(hc, 32u));
}

// ------------------------------------------------------- dense algebra ------
// LU with partial pivoting (full-row swaps), inverse by per-column forward /
// back substitution, then exact symmetrisation K = (A^-1 + A^-T)/2 (OD-4).
std::vector<double> dense_inverse_sym(std::vector<double> a, int n) {
    std::vector<int> piv(n);
    const int T = host_threads();
    for (int k = 0; k < n; ++k) {
        int p = k;
        double best = std::fabs(a[static_cast<size_t>(k) * n + k]);
        for (int i = k + 1; i < n; ++i) {
            const double v = std::fabs(a[static_cast<size_t>(i) * n + k]);
            if (v > best) { best = v; p = i; }
        }
        if (best == 0.0) throw SmgError(SMG_ESINGULAR, "coarse LU: singular matrix");
        piv[k] = p;
        if (p != k)
            for (int j = 0; j < n; ++j) std::swap(a[static_cast<size_t>(k) * n + j], a[static_cast<size_t>(p) * n + j]);
        const double d = a[static_cast<size_t>(k) * n + k];
        const int rows = n - k - 1;
        auto elim = [&](int64_t lo, int64_t hi) {
            const double* rk = &a[static_cast<size_t>(k) * n];
            for (int64_t t = lo; t < hi; ++t) {
                double* ri = &a[static_cast<size_t>(k + 1 + t) * n];
                const double m = ri[k] / d;
                ri[k] = m;
                if (m != 0.0)
                    for (int j = k + 1; j < n; ++j) ri[j] = ri[j] - m * rk[j];
            }
        };
        if (static_cast<int64_t>(rows) * (n - k) > 200000) host_parallel(rows, T, elim);
        else elim(0, rows);
    }
    std::vector<double> inv(static_cast<size_t>(n) * n, 0.0);  // inv[col*n + i] = (A^-1)_{i,col}
    host_parallel(n, T, [&](int64_t lo, int64_t hi) {
        std::vector<double> y(n);
        for (int64_t col = lo; col < hi; ++col) {
            std::fill(y.begin(), y.end(), 0.0);
            y[col] = 1.0;
            for (int k = 0; k < n; ++k)
                if (piv[k] != k) std::swap(y[k], y[piv[k]]);
            for (int i = 0; i < n; ++i) {
                double s = y[i];
                const double* ri = &a[static_cast<size_t>(i) * n];
                for (int j = 0; j < i; ++j) s = s - ri[j] * y[j];
                y[i] = s;
            }
            for (int i = n - 1; i >= 0; --i) {
                double s = y[i];
                const double* ri = &a[static_cast<size_t>(i) * n];
                for (int j = i + 1; j < n; ++j) s = s - ri[j] * y[j];
                y[i] = s / ri[i];
            }
            for (int i = 0; i < n; ++i) inv[static_cast<size_t>(col) * n + i] = y[i];
        }
    });
    std::vector<double> k(static_cast<size_t>(n) * n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            k[static_cast<size_t>(i) * n + j] =
                0.5 * (inv[static_cast<size_t>(j) * n + i] + inv[static_cast<size_t>(i) * n + j]);
    return k;
}

// Gauss-Jordan with partial pivoting for the <= 7x7 Vanka blocks.
void small_inverse(const double* m, int n, double* out /* n x n */) {
    double a[49], e[49];
    for (int i = 0; i < n * n; ++i) { a[i] = m[i]; e[i] = 0.0; }
    for (int i = 0; i < n; ++i) e[i * n + i] = 1.0;
    for (int k = 0; k < n; ++k) {
        int p = k;
        double best = std::fabs(a[k * n + k]);
        for (int i = k + 1; i < n; ++i)
            if (std::fabs(a[i * n + k]) > best) { best = std::fabs(a[i * n + k]); p = i; }
        if (best == 0.0) throw SmgError(SMG_ESINGULAR, "vanka: singular local matrix (SPEC:288)");
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
    for (int i = 0; i < n * n; ++i) out[i] = e[i];
}

// ----------------------------------------------------------- forcing --------
inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
inline uint64_t key5(uint64_t seed, uint64_t c, uint64_t i, uint64_t j, uint64_t k) {
    return mix64(mix64(mix64(mix64(mix64(seed) ^ c) ^ k) ^ j) ^ i);
}
inline double unit01(uint64_t h) { return static_cast<double>(h >> 11) * 0x1.0p-53; }

// ------------------------------------------------------------ context -------
struct DevLevel {
    LevelK k{};
    int64_t counts[5] = {0, 0, 0, 0, 0};  // nu, nv, nw, np, |V1|
    int64_t N = 0;
    double *x = nullptr, *b = nullptr, *r = nullptr, *pd = nullptr;  // pd: DGS delta (one field)
    double *pd0 = nullptr, *pd1 = nullptr;  // alternating delta buffers of the cooperative DGS sweep
    int32_t* vk_cells[8] = {};
    uint8_t* vk_mask[8] = {};
    uint8_t* vk_amask[8] = {};  // z-slab levels: owned slots per block (nullptr: all)
    double* xb = nullptr;         // ping-pong partner of x for the Vanka sweep
    double *wb = nullptr, *wx = nullptr;  // W-cycle: rhs / correction of the second recursive call
    int32_t* vk_refresh = nullptr;  // slots every Vanka residual reads (refreshed x -> xb per sweep)
    int64_t vk_nrefresh = 0;
    int vk_n[8] = {};
    // lists of the symmetric sweeps: as vk_* with merged complementary pairs (list m = parity m,
    // then parity 7-m; see VankaPairs)
    int32_t* sw_cells[8] = {};
    uint8_t* sw_mask[8] = {};
    uint8_t* sw_amask[8] = {};  // z-slab levels: owned slots per block of the (merged) sweep lists
    int sw_n[8] = {};
    VankaPairs sw_pairs;
    // additive Vanka (params.vanka == 1): every block in one list + the 7-field correction scratch
    int32_t* va_cells = nullptr;
    uint8_t* va_mask = nullptr;
    int va_n = 0;
    double* va_d7 = nullptr;
    double* ktab = nullptr;  // [64][49]
    // direct-on-V1 (params.vanka == 2): symmetric dense inverse of the V1 x V1
    // principal sub-block of L~ and the padded slots of the V1 DOFs (ascending compact order)
    double* v1_k = nullptr;
    int32_t* v1_slots = nullptr;
    int v1_n = 0;
    // general labelled domain: DofMap bits per cell slot (LevelK::cls points here),
    // padded slot of every active DOF in compact order, signature class of every Vanka block
    uint32_t* cls = nullptr;
    int32_t* pack_slots = nullptr;
    uint16_t* vk_kidx[8] = {};
    uint16_t* sw_kidx[4] = {};  // merged complementary pairs (list m = parity m, then parity 7 - m)
    uint16_t* va_kidx = nullptr;  // additive Vanka: classes of the one list of all blocks
    std::shared_ptr<struct HostMap> hm;
};

// classify_dofs + partition_band on a labelled CellGrid: the host-side DofMap of one
// level.  Cells outside the labelled box are the implicit Dirichlet ring.  A face is
// stored with the cell on its high side (the u face between cells x-1 and x at cell x), so faces
// and pressures share one index; ids follow the SPEC numbering (u-lex, v-lex, w-lex, p-lex, x
// fastest).
enum : uint8_t { LAB_D = 0, LAB_I = 1, LAB_E = 2 };
constexpr int32_t ST_DIRICHLET = -1, ST_INACTIVE = -2;
struct HostMap {
    int nx = 0, ny = 0, nz = 0;
    std::vector<uint8_t> lab, band;
    std::vector<int32_t> id[4];   // per cell: compact id of the low u, v, w face / the pressure, or a status
    std::vector<uint8_t> drop[3];  // per cell and low face: stencil legs into Inactive faces
    int64_t cnt[4] = {0, 0, 0, 0}, N = 0, v1 = 0;
    size_t ci(int x, int y, int z) const { return (static_cast<size_t>(z) * ny + y) * nx + x; }
    bool inside(int x, int y, int z) const { return x >= 0 && y >= 0 && z >= 0 && x < nx && y < ny && z < nz; }
    uint8_t at(int x, int y, int z) const { return inside(x, y, z) ? lab[ci(x, y, z)] : static_cast<uint8_t>(LAB_D); }
    // low face of component c of cell (x, y, z); faces beyond the box belong to ring cells: Dirichlet
    int32_t face(int c, int x, int y, int z) const { return inside(x, y, z) ? id[c][ci(x, y, z)] : ST_DIRICHLET; }
    int32_t cell(int x, int y, int z) const { return inside(x, y, z) ? id[3][ci(x, y, z)] : ST_INACTIVE; }
    bool is_band(int x, int y, int z) const { return inside(x, y, z) && band[ci(x, y, z)]; }
};

}  // namespace

struct smg_ctx {
    int device = 0;
    cudaStream_t st = nullptr;
    smg_params prm{};
    smg_grid_desc grid{};
    std::vector<DevLevel> lv;
    double* coarse_k = nullptr;
    int32_t* coarse_slots = nullptr;
    int nc = 0;
    double* vk_delta = nullptr;
    // SQMR vectors on the fine level (s = lv[0].b, t = lv[0].x, scratch = lv[0].r)
    // q, d and x_sqmr ping-pong between iterations (the fused kernels read the old and write the
    // new vector): buffer [j & 1] holds the values after iteration j
    double *q = nullptr, *d = nullptr, *xs = nullptr, *rhs = nullptr;
    double *q2 = nullptr, *d2 = nullptr, *xs2 = nullptr;
    int xcur = 0;  // buffer holding the current solution (0: xs, 1: xs2)
    double* compact = nullptr;
    double* partials = nullptr;
    double* dscal = nullptr;
    double* hscal = nullptr;  // pinned
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaGraphExec_t graph = nullptr, graph2 = nullptr;  // one SQMR iteration (even / odd parity)
    int64_t graph_kernels = 0;
    bool graph_captured_now = false;
    cudaGraphExec_t init_graph = nullptr;  // SQMR lines 1-4 (initial V-cycle), opt-in
    int64_t init_kernels = 0;
    std::string err;
    smg_timing timing{};
    std::vector<void*> allocs;
    bool rhs_set = false;
    // z-slab decomposition: this context is part `rank` of `nparts`;
    // levels < ndist are slabs of their level, the others are replicated whole.
    int rank = 0, nparts = 1, ndist = 0;
    std::vector<smg_ctx*> parts;                    // parts[0] == the owning (master) context
    std::vector<std::unique_ptr<smg_ctx>> owned;   // parts 1..P-1 (owned by the master)
    double* shared_partials = nullptr;             // plane partials all parts write (master's device)
    bool own_stream = true;
    // multi-process mode (smg_create_rank): this process holds part `rank` only; halos,
    // plane partials and gathers travel through NCCL on the part's stream
    bool mp = false;
    ncclComm_t comm = nullptr;
    // Comm stream (overlap): the halo transfers of a tiled DGS phase run here while the
    // interior tile layers run on `st`.  evb: boundary tiles done (st -> cst); evc: transfer done
    // (cst -> st).  Parts sharing the master's stream share its comm stream.  hcomm: a split of
    // `comm` for the transfers on the comm stream (the same communicator when ncclCommSplit is missing).
    cudaStream_t cst = nullptr;
    bool own_cst = false;
    cudaEvent_t evb = nullptr, evc = nullptr;
    ncclComm_t hcomm = nullptr;
    bool on_cst = false;  // master only: transports are being enqueued on the comm streams
    // halo frames (exchange_frame): send up / send down / received from above / received from below
    double* fbuf[4] = {nullptr, nullptr, nullptr, nullptr};
    // general labelled domain (smg_create_labeled): fine-level cell labels, x fastest; empty: walled box
    std::vector<uint8_t> labels;

    // SMG_GUARD=1 (debug; compute-sanitizer is closed on the GPU pool): every device buffer sits
    // between two 4 KiB guard bands filled with 0xA5; smg_check_guards reports any band a kernel
    // wrote into (an out-of-bounds store of a stencil, list or tile kernel).
    static constexpr size_t kGuard = 4096;
    struct GuardRec {
        unsigned char* base;
        size_t bytes;
    };
    std::vector<GuardRec> guards;
    bool guard_on = std::getenv("SMG_GUARD") && std::atoi(std::getenv("SMG_GUARD")) != 0;
    template <class T>
    T* dalloc(int64_t count) {
        void* p = nullptr;
        size_t bytes = static_cast<size_t>(count) * sizeof(T);
        if (!bytes) bytes = 8;
        const size_t pad = guard_on ? kGuard : 0;
        const size_t body = (bytes + 255) / 256 * 256;
        cudaError_t e = cudaMalloc(&p, body + 2 * pad);
        if (e != cudaSuccess) throw SmgError(SMG_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
        allocs.push_back(p);
        unsigned char* base = static_cast<unsigned char*>(p);
        if (guard_on) {
            CK(cudaMemsetAsync(base, 0xA5, body + 2 * pad, st));
            guards.push_back({base, body});
        }
        CK(cudaMemsetAsync(base + pad, 0, bytes, st));
        return reinterpret_cast<T*>(base + pad);
    }
    // number of guard bytes overwritten since creation (0 when the guards are off)
    int64_t check_guards() {
        if (!guard_on) return 0;
        CK(cudaStreamSynchronize(st));
        std::vector<unsigned char> h(2 * kGuard);
        int64_t bad = 0;
        for (const GuardRec& g : guards) {
            CK(cudaMemcpy(h.data(), g.base, kGuard, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(h.data() + kGuard, g.base + kGuard + g.bytes, kGuard, cudaMemcpyDeviceToHost));
            for (unsigned char c : h) bad += c != 0xA5;
        }
        return bad;
    }
    ~smg_ctx() {
        if (st) cudaStreamSynchronize(st);
        owned.clear();  // parts may share this context's stream: destroy them first
        for (void* p : allocs) cudaFree(p);
        if (hscal) cudaFreeHost(hscal);
        if (graph) cudaGraphExecDestroy(graph);
        if (graph2) cudaGraphExecDestroy(graph2);
        if (init_graph) cudaGraphExecDestroy(init_graph);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        if (evb) cudaEventDestroy(evb);
        if (evc) cudaEventDestroy(evc);
        if (cst && own_cst) {
            cudaStreamSynchronize(cst);
            cudaStreamDestroy(cst);
        }
        if (hcomm && hcomm != comm) nccl().commDestroy(hcomm);
        if (comm) nccl().commDestroy(comm);
        if (st && own_stream) cudaStreamDestroy(st);
    }
};

namespace {

int64_t vlen(const DevLevel& L) { return L.k.g.vec_len(); }


// Dense rows of L~ on a box level in compact numbering, restricted to the DOFs with
// sel[id] >= 0 (sel = nullptr: every DOF): A[sel[r] * nsel + sel[c]], and the padded slot of every
// selected DOF.  Entries accumulate in the oracle's ltilde_row order (diagonal, six neighbours,
// p_left, p_right; continuity: the six faces, then -gamma), so A is bit-identical to the oracle's.
void assemble_box_dense(const DevLevel& C, double gamma, const int32_t* sel, int nsel, std::vector<double>& A,
                        std::vector<int32_t>& slots) {
    const int nx = C.k.g.nx, ny = C.k.g.ny, nz = C.k.g.nz;
    const int64_t nu = C.counts[0], nv = C.counts[1], nw = C.counts[2];
    auto uid = [&](int x, int y, int z) -> int {
        if (x < 1 || x > nx - 1 || y < 0 || y >= ny || z < 0 || z >= nz) return -1;
        return static_cast<int>((static_cast<int64_t>(z) * ny + y) * (nx - 1) + (x - 1));
    };
    auto vid = [&](int x, int y, int z) -> int {
        if (x < 0 || x >= nx || y < 1 || y > ny - 1 || z < 0 || z >= nz) return -1;
        return static_cast<int>(nu + (static_cast<int64_t>(z) * (ny - 1) + (y - 1)) * nx + x);
    };
    auto wid = [&](int x, int y, int z) -> int {
        if (x < 0 || x >= nx || y < 0 || y >= ny || z < 1 || z > nz - 1) return -1;
        return static_cast<int>(nu + nv + (static_cast<int64_t>(z - 1) * ny + y) * nx + x);
    };
    auto pid = [&](int x, int y, int z) -> int {
        if (x < 0 || x >= nx || y < 0 || y >= ny || z < 0 || z >= nz) return -1;
        return static_cast<int>(nu + nv + nw + (static_cast<int64_t>(z) * ny + y) * nx + x);
    };
    auto loc = [&](int id) { return id < 0 ? -1 : (sel ? sel[id] : id); };
    A.assign(static_cast<size_t>(nsel) * nsel, 0.0);
    slots.assign(nsel, 0);
    const double e2 = C.k.eta_h2, ih = C.k.inv_h;
    auto put = [&](int r, int col, double v) {
        const int c = loc(col);
        if (c >= 0) A[static_cast<size_t>(r) * nsel + c] += v;
    };
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x) {
                const int64_t sl = C.k.g.slot(x, y, z);
                for (int comp = 0; comp < 3; ++comp) {
                    auto fid = [&](int a, int b2, int c3) {
                        return comp == 0 ? uid(a, b2, c3) : comp == 1 ? vid(a, b2, c3) : wid(a, b2, c3);
                    };
                    const int r = loc(fid(x, y, z));
                    if (r < 0) continue;
                    slots[r] = static_cast<int32_t>(comp * C.k.g.fs + sl);
                    put(r, fid(x, y, z), 6.0 * e2);
                    const int d[6][3] = {{-1, 0, 0}, {1, 0, 0}, {0, -1, 0}, {0, 1, 0}, {0, 0, -1}, {0, 0, 1}};
                    for (int k = 0; k < 6; ++k) put(r, fid(x + d[k][0], y + d[k][1], z + d[k][2]), -e2);
                    const int lx = x - (comp == 0), ly = y - (comp == 1), lz = z - (comp == 2);
                    put(r, pid(lx, ly, lz), -ih);
                    put(r, pid(x, y, z), ih);
                }
                const int r = loc(pid(x, y, z));
                if (r < 0) continue;
                slots[r] = static_cast<int32_t>(3 * C.k.g.fs + sl);
                put(r, uid(x, y, z), ih);
                put(r, uid(x + 1, y, z), -ih);
                put(r, vid(x, y, z), ih);
                put(r, vid(x, y + 1, z), -ih);
                put(r, wid(x, y, z), ih);
                put(r, wid(x, y, z + 1), -ih);
                put(r, pid(x, y, z), -gamma);
            }
}

// compact id -> index among the V1 DOFs (ascending), -1 for V2 (partition_band)
int v1_selection(const DevLevel& L, int bw, std::vector<int32_t>& sel) {
    const int nx = L.k.g.nx, ny = L.k.g.ny, nz = L.k.g.nz;
    auto band = [&](int x, int y, int z) {
        return x < bw || y < bw || z < bw || x >= nx - bw || y >= ny - bw || z >= nz - bw;
    };
    sel.assign(static_cast<size_t>(L.N), -1);
    int n = 0;
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (int x = 1; x < nx; ++x)
                if (band(x, y, z) || band(x - 1, y, z)) sel[(static_cast<int64_t>(z) * ny + y) * (nx - 1) + (x - 1)] = 0;
    for (int z = 0; z < nz; ++z)
        for (int y = 1; y < ny; ++y)
            for (int x = 0; x < nx; ++x)
                if (band(x, y, z) || band(x, y - 1, z))
                    sel[L.counts[0] + (static_cast<int64_t>(z) * (ny - 1) + (y - 1)) * nx + x] = 0;
    for (int z = 1; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x)
                if (band(x, y, z) || band(x, y, z - 1))
                    sel[L.counts[0] + L.counts[1] + (static_cast<int64_t>(z - 1) * ny + y) * nx + x] = 0;
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x)
                if (band(x, y, z))
                    sel[L.counts[0] + L.counts[1] + L.counts[2] + (static_cast<int64_t>(z) * ny + y) * nx + x] = 0;
    for (auto& v : sel)
        if (v == 0) v = n++;
    return n;
}

// ---- general labelled domains ----
// coarsen_grid: a coarse cell is Dirichlet if any child is, else Interior if any child
// is, else Exterior.
std::vector<uint8_t> coarsen_labels(const std::vector<uint8_t>& f, int nx, int ny, int nz) {
    const int cx = nx / 2, cy = ny / 2, cz = nz / 2;
    std::vector<uint8_t> c(static_cast<size_t>(cx) * cy * cz, LAB_E);
    for (int z = 0; z < cz; ++z)
        for (int y = 0; y < cy; ++y)
            for (int x = 0; x < cx; ++x) {
                bool anyD = false, anyI = false;
                for (int k = 0; k < 2; ++k)
                    for (int j = 0; j < 2; ++j)
                        for (int i = 0; i < 2; ++i) {
                            const uint8_t l = f[(static_cast<size_t>(2 * z + k) * ny + (2 * y + j)) * nx + (2 * x + i)];
                            anyD |= l == LAB_D;
                            anyI |= l == LAB_I;
                        }
                c[(static_cast<size_t>(z) * cy + y) * cx + x] = anyD ? LAB_D : (anyI ? LAB_I : LAB_E);
            }
    return c;
}

// classify_dofs + partition_band of one labelled level.
std::shared_ptr<HostMap> classify_labeled(std::vector<uint8_t> lab, int nx, int ny, int nz, int bw) {
    auto hm = std::make_shared<HostMap>();
    HostMap& m = *hm;
    m.nx = nx;
    m.ny = ny;
    m.nz = nz;
    m.lab = std::move(lab);
    const size_t nc = static_cast<size_t>(nx) * ny * nz;
    int64_t next = 0;
    for (int c = 0; c < 3; ++c) {
        m.id[c].assign(nc, ST_DIRICHLET);
        const int64_t first = next;
        for (int z = 0; z < nz; ++z)
            for (int y = 0; y < ny; ++y)
                for (int x = 0; x < nx; ++x) {
                    const uint8_t a = m.at(x - (c == 0), y - (c == 1), z - (c == 2)), b = m.at(x, y, z);
                    int32_t st;
                    if (a == LAB_D || b == LAB_D) st = ST_DIRICHLET;
                    else if (a == LAB_I && b == LAB_I) st = static_cast<int32_t>(next++);
                    else st = ST_INACTIVE;
                    m.id[c][m.ci(x, y, z)] = st;
                }
        m.cnt[c] = next - first;
    }
    m.id[3].assign(nc, ST_INACTIVE);
    for (size_t q = 0; q < nc; ++q)
        if (m.lab[q] == LAB_I) m.id[3][q] = static_cast<int32_t>(next++);
    m.cnt[3] = next - (m.cnt[0] + m.cnt[1] + m.cnt[2]);
    m.N = next;
    m.band.assign(nc, 0);
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x) {
                bool band = false;
                for (int k = -bw; k <= bw && !band; ++k)
                    for (int j = -bw; j <= bw && !band; ++j)
                        for (int i = -bw; i <= bw && !band; ++i)
                            if (m.at(x + i, y + j, z + k) != LAB_I) band = true;
                m.band[m.ci(x, y, z)] = band;
            }
    const int d[6][3] = {{-1, 0, 0}, {1, 0, 0}, {0, -1, 0}, {0, 1, 0}, {0, 0, -1}, {0, 0, 1}};
    for (int c = 0; c < 3; ++c) {
        m.drop[c].assign(nc, 0);
        for (int z = 0; z < nz; ++z)
            for (int y = 0; y < ny; ++y)
                for (int x = 0; x < nx; ++x) {
                    if (m.id[c][m.ci(x, y, z)] < 0) continue;
                    int dr = 0;
                    for (auto& k : d)
                        if (m.face(c, x + k[0], y + k[1], z + k[2]) == ST_INACTIVE) ++dr;  // dropped Neumann leg
                    m.drop[c][m.ci(x, y, z)] = static_cast<uint8_t>(dr);
                    if (m.is_band(x, y, z) || m.is_band(x - (c == 0), y - (c == 1), z - (c == 2))) ++m.v1;
                }
    }
    for (size_t q = 0; q < nc; ++q)
        if (m.id[3][q] >= 0 && m.band[q]) ++m.v1;
    return hm;
}

// Sparse row r of L~ in the oracle's ltilde_row order (diagonal, six same-component neighbours,
// p_left, p_right; continuity: the six faces, then -gamma), handed to put(col, value).
template <class Put>
void labeled_row(const HostMap& m, double e2, double ih, double gamma, int comp, int x, int y, int z, Put&& put) {
    if (comp < 3) {
        put(m.face(comp, x, y, z), (6.0 - m.drop[comp][m.ci(x, y, z)]) * e2);
        const int d[6][3] = {{-1, 0, 0}, {1, 0, 0}, {0, -1, 0}, {0, 1, 0}, {0, 0, -1}, {0, 0, 1}};
        for (auto& k : d) put(m.face(comp, x + k[0], y + k[1], z + k[2]), -e2);
        put(m.cell(x - (comp == 0), y - (comp == 1), z - (comp == 2)), -ih);
        put(m.cell(x, y, z), ih);
    } else {
        put(m.face(0, x, y, z), ih);
        put(m.face(0, x + 1, y, z), -ih);
        put(m.face(1, x, y, z), ih);
        put(m.face(1, x, y + 1, z), -ih);
        put(m.face(2, x, y, z), ih);
        put(m.face(2, x, y, z + 1), -ih);
        put(m.cell(x, y, z), -gamma);
    }
}

// Dense L~ of a labelled level restricted to the DOFs with sel[id] >= 0 (nullptr: all), and their
// padded slots -- assemble_box_dense for a general DofMap.
void assemble_labeled_dense(const DevLevel& C, double gamma, const int32_t* sel, int nsel, std::vector<double>& A,
                            std::vector<int32_t>& slots) {
    const HostMap& m = *C.hm;
    A.assign(static_cast<size_t>(nsel) * nsel, 0.0);
    slots.assign(nsel, 0);
    auto loc = [&](int32_t id) { return id < 0 ? -1 : (sel ? sel[id] : id); };
    for (int z = 0; z < m.nz; ++z)
        for (int y = 0; y < m.ny; ++y)
            for (int x = 0; x < m.nx; ++x)
                for (int comp = 0; comp < 4; ++comp) {
                    const int r = loc(m.id[comp][m.ci(x, y, z)]);
                    if (r < 0) continue;
                    slots[r] = static_cast<int32_t>(comp * C.k.g.fs + C.k.g.slot(x, y, z));
                    labeled_row(m, C.k.eta_h2, C.k.inv_h, gamma, comp, x, y, z, [&](int32_t col, double v) {
                        const int cc = loc(col);
                        if (cc >= 0) A[static_cast<size_t>(r) * nsel + cc] += v;
                    });
                }
}

// Device tables of one labelled level: DofMap bits, pack list, Vanka blocks by parity colour with
// their signature classes (the local matrix depends on which faces are active and on
// each active face's dropped legs) and the class inverses.
void build_level_labeled(smg_ctx* c, int l, std::vector<uint8_t> lab, int& max_vk) {
    DevLevel& L = c->lv[l];
    const smg_params& p = c->prm;
    const Geom& G = L.k.g;
    const int nx = G.nx, ny = G.ny, nz = G.nz;
    L.hm = classify_labeled(std::move(lab), nx, ny, nz, p.band_width);
    const HostMap& m = *L.hm;
    for (int k = 0; k < 4; ++k) L.counts[k] = m.cnt[k];
    L.counts[4] = m.v1;
    L.N = m.N;
    std::vector<uint32_t> cls(static_cast<size_t>(G.fs), 0u);
    std::vector<int32_t> pack(static_cast<size_t>(m.N), 0);
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x) {
                const size_t q = m.ci(x, y, z);
                const int64_t sl = G.slot(x, y, z);
                uint32_t b = 0;
                const bool bc = m.band[q] != 0;
                if (bc) b |= CLS_BAND;
                if (m.id[3][q] >= 0) {
                    b |= CLS_P;
                    pack[m.id[3][q]] = static_cast<int32_t>(3 * G.fs + sl);
                }
                for (int comp = 0; comp < 3; ++comp) {
                    if (m.id[comp][q] < 0) continue;
                    b |= CLS_U << comp;
                    if (!bc && !m.is_band(x - (comp == 0), y - (comp == 1), z - (comp == 2))) b |= CLS_U2 << comp;
                    b |= static_cast<uint32_t>(6 - m.drop[comp][q]) << (CLS_DIAG_SHIFT + 3 * comp);
                    pack[m.id[comp][q]] = static_cast<int32_t>(comp * G.fs + sl);
                }
                cls[sl] = b;
            }
    L.cls = c->dalloc<uint32_t>(G.fs);
    L.k.cls = L.cls;
    L.pack_slots = c->dalloc<int32_t>(m.N);
    CK(cudaMemcpyAsync(L.cls, cls.data(), cls.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(L.pack_slots, pack.data(), pack.size() * sizeof(int32_t), cudaMemcpyHostToDevice, c->st));
    CK(cudaStreamSynchronize(c->st));
    // Vanka blocks: band cells with an active pressure; slots [uL, uR, vL, vR, wL, wR, p]
    std::vector<int32_t> cells[8];
    std::vector<uint8_t> masks[8];
    std::vector<uint16_t> kidx[8];
    std::unordered_map<int, int> keys;  // signature key -> class index
    std::vector<double> ktab;
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x) {
                const size_t q = m.ci(x, y, z);
                if (m.id[3][q] < 0 || !m.band[q]) continue;
                const int fx[6][4] = {{0, x, y, z}, {0, x + 1, y, z}, {1, x, y, z}, {1, x, y + 1, z}, {2, x, y, z}, {2, x, y, z + 1}};
                int mask = 0, key = 0, dr[6] = {};
                for (int s2 = 0; s2 < 6; ++s2) {
                    if (m.face(fx[s2][0], fx[s2][1], fx[s2][2], fx[s2][3]) < 0) continue;
                    mask |= 1 << s2;
                    dr[s2] = m.drop[fx[s2][0]][m.ci(fx[s2][1], fx[s2][2], fx[s2][3])];
                    key |= dr[s2] << (6 + 3 * s2);
                }
                key |= mask;
                const auto hit = keys.find(key);
                int ki = hit == keys.end() ? -1 : hit->second;
                if (ki < 0) {  // new class: invert C_i L~ C_i^T over the active slots, scatter to the 7-slot layout
                    if (keys.size() >= 65535) throw SmgError(SMG_ECAP, "more than 65535 Vanka signature classes");
                    ki = static_cast<int>(keys.size());
                    keys.emplace(key, ki);
                    int slot[7], nb = 0;
                    for (int s2 = 0; s2 < 6; ++s2)
                        if (mask & (1 << s2)) slot[nb++] = s2;
                    slot[nb++] = 6;
                    double lm[49] = {}, inv[49];
                    for (int a = 0; a < nb; ++a)
                        for (int b2 = 0; b2 < nb; ++b2) {
                            const int sa = slot[a], sb = slot[b2];
                            double v = 0.0;
                            if (sa < 6 && sb < 6) {
                                if (sa == sb) v = (6.0 - dr[sa]) * L.k.eta_h2;
                                else if ((sa >> 1) == (sb >> 1)) v = -L.k.eta_h2;  // the cell's two faces of one axis
                            } else if (sa < 6 && sb == 6) {
                                v = (sa & 1) ? -L.k.inv_h : L.k.inv_h;  // low face: the cell is its p_right
                            } else if (sa == 6 && sb < 6) {
                                v = (sb & 1) ? -L.k.inv_h : L.k.inv_h;
                            } else {
                                v = -p.gamma;
                            }
                            lm[a * nb + b2] = v;
                        }
                    small_inverse(lm, nb, inv);
                    ktab.resize(ktab.size() + 49, 0.0);
                    for (int a = 0; a < nb; ++a)
                        for (int b2 = 0; b2 < nb; ++b2) ktab[static_cast<size_t>(ki) * 49 + slot[a] * 7 + slot[b2]] = inv[a * nb + b2];
                }
                const int col = (x & 1) + 2 * (y & 1) + 4 * (z & 1);
                cells[col].push_back(static_cast<int32_t>(G.slot(x, y, z)));
                masks[col].push_back(static_cast<uint8_t>(mask));
                kidx[col].push_back(static_cast<uint16_t>(ki));
            }
    for (int col = 0; col < 8; ++col) {
        const size_t n = cells[col].size();
        L.vk_n[col] = L.sw_n[col] = static_cast<int>(n);
        max_vk = std::max(max_vk, L.vk_n[col]);
        L.vk_cells[col] = L.sw_cells[col] = c->dalloc<int32_t>(n);
        L.vk_mask[col] = L.sw_mask[col] = c->dalloc<uint8_t>(n);
        L.vk_kidx[col] = c->dalloc<uint16_t>(n);
        CK(cudaMemcpyAsync(L.vk_cells[col], cells[col].data(), n * sizeof(int32_t), cudaMemcpyHostToDevice, c->st));
        CK(cudaMemcpyAsync(L.vk_mask[col], masks[col].data(), n, cudaMemcpyHostToDevice, c->st));
        CK(cudaMemcpyAsync(L.vk_kidx[col], kidx[col].data(), n * sizeof(uint16_t), cudaMemcpyHostToDevice, c->st));
        CK(cudaStreamSynchronize(c->st));
    }
    // sweep lists: complementary parities (m, 7 - m) never touch each other's DOFs on any labelling
    // (a residual stencil reaches along one axis), so each pair is one Jacobi phase (8 per sweep)
    for (int pq = 0; pq < 4; ++pq) {
        std::vector<int32_t> mc(cells[pq]);
        mc.insert(mc.end(), cells[7 - pq].begin(), cells[7 - pq].end());
        std::vector<uint8_t> mm(masks[pq]);
        mm.insert(mm.end(), masks[7 - pq].begin(), masks[7 - pq].end());
        std::vector<uint16_t> mk(kidx[pq]);
        mk.insert(mk.end(), kidx[7 - pq].begin(), kidx[7 - pq].end());
        const size_t n = mc.size();
        L.sw_n[pq] = static_cast<int>(n);
        L.sw_n[7 - pq] = 0;
        max_vk = std::max(max_vk, L.sw_n[pq]);
        L.sw_cells[pq] = c->dalloc<int32_t>(n);
        L.sw_mask[pq] = c->dalloc<uint8_t>(n);
        L.sw_kidx[pq] = c->dalloc<uint16_t>(n);
        CK(cudaMemcpyAsync(L.sw_cells[pq], mc.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice, c->st));
        CK(cudaMemcpyAsync(L.sw_mask[pq], mm.data(), n, cudaMemcpyHostToDevice, c->st));
        CK(cudaMemcpyAsync(L.sw_kidx[pq], mk.data(), n * sizeof(uint16_t), cudaMemcpyHostToDevice, c->st));
        CK(cudaStreamSynchronize(c->st));
    }
    L.ktab = c->dalloc<double>(std::max<size_t>(ktab.size(), 49));
    CK(cudaMemcpyAsync(L.ktab, ktab.data(), ktab.size() * sizeof(double), cudaMemcpyHostToDevice, c->st));
    CK(cudaStreamSynchronize(c->st));
    if (p.vanka == 1) {  // additive Vanka: every block in one list + the 7-field correction scratch
        std::vector<int32_t> ac;
        std::vector<uint8_t> am;
        std::vector<uint16_t> ak;
        for (int col = 0; col < 8; ++col) {
            ac.insert(ac.end(), cells[col].begin(), cells[col].end());
            am.insert(am.end(), masks[col].begin(), masks[col].end());
            ak.insert(ak.end(), kidx[col].begin(), kidx[col].end());
        }
        L.va_n = static_cast<int>(ac.size());
        L.va_cells = c->dalloc<int32_t>(L.va_n);
        L.va_mask = c->dalloc<uint8_t>(L.va_n);
        L.va_kidx = c->dalloc<uint16_t>(L.va_n);
        L.va_d7 = c->dalloc<double>(7 * G.fs);
        CK(cudaMemcpyAsync(L.va_cells, ac.data(), ac.size() * sizeof(int32_t), cudaMemcpyHostToDevice, c->st));
        CK(cudaMemcpyAsync(L.va_mask, am.data(), am.size(), cudaMemcpyHostToDevice, c->st));
        CK(cudaMemcpyAsync(L.va_kidx, ak.data(), ak.size() * sizeof(uint16_t), cudaMemcpyHostToDevice, c->st));
        CK(cudaStreamSynchronize(c->st));
    }
    if (p.vanka == 2 && l + 1 < p.levels) {  // direct-on-V1: dense symmetric inverse of the V1 x V1 sub-block
        std::vector<int32_t> sel(static_cast<size_t>(m.N), -1), vslots;
        int n1 = 0;
        // V1 DOFs ascending in compact order
        std::vector<uint8_t> isv1(static_cast<size_t>(m.N), 0);
        for (int z = 0; z < nz; ++z)
            for (int y = 0; y < ny; ++y)
                for (int x = 0; x < nx; ++x) {
                    const size_t q = m.ci(x, y, z);
                    for (int comp = 0; comp < 3; ++comp)
                        if (m.id[comp][q] >= 0 &&
                            (m.band[q] || m.is_band(x - (comp == 0), y - (comp == 1), z - (comp == 2))))
                            isv1[m.id[comp][q]] = 1;
                    if (m.id[3][q] >= 0 && m.band[q]) isv1[m.id[3][q]] = 1;
                }
        for (int64_t k = 0; k < m.N; ++k)
            if (isv1[k]) sel[k] = n1++;
        if (n1 > 20000) throw SmgError(SMG_ECAP, "direct-on-V1: |V1| above the dense cap 20000 (SPEC:365)");
        std::vector<double> A11;
        assemble_labeled_dense(L, p.gamma, sel.data(), n1, A11, vslots);
        const std::vector<double> K1 = n1 ? dense_inverse_sym(std::move(A11), n1) : std::vector<double>();
        L.v1_n = n1;
        L.v1_k = c->dalloc<double>(static_cast<int64_t>(n1) * n1);
        L.v1_slots = c->dalloc<int32_t>(n1);
        CK(cudaMemcpyAsync(L.v1_k, K1.data(), K1.size() * sizeof(double), cudaMemcpyHostToDevice, c->st));
        CK(cudaMemcpyAsync(L.v1_slots, vslots.data(), vslots.size() * sizeof(int32_t), cudaMemcpyHostToDevice, c->st));
        CK(cudaStreamSynchronize(c->st));
    }
}

// ---- setup ----
void build(smg_ctx* c, const std::vector<double>* shared_coarse = nullptr, std::vector<double>* coarse_out = nullptr,
           cudaStream_t shared_stream = nullptr) {
    const smg_grid_desc& g = c->grid;
    if (!(c->prm.omega > 0.0)) c->prm.omega = 1.0;  // SPEC default inside the preconditioner
    const smg_params& p = c->prm;
    if (g.dim != 3) throw SmgError(SMG_EINVAL, "dim must be 3");
    if (p.levels < 1) throw SmgError(SMG_EINVAL, "levels < 1");
    if (p.nu < 1 || p.band_width < 1) throw SmgError(SMG_EINVAL, "nu and band_width must be >= 1");
    if (p.cycle != 0 && p.cycle != 1) throw SmgError(SMG_EINVAL, "cycle must be 0 (V) or 1 (W)");
    if (p.vanka < 0 || p.vanka > 2)
        throw SmgError(SMG_EINVAL, "vanka must be 0 (multiplicative), 1 (additive) or 2 (direct solve on V1)");
    if (p.omega > 1.0) throw SmgError(SMG_EINVAL, "omega must lie in (0, 1] (<= 0: default 1)");
    if (p.vanka != 0 && c->ndist > 0)
        throw SmgError(SMG_EINVAL, "additive Vanka / direct-on-V1: single-part contexts only");
    if (!(g.h > 0)) throw SmgError(SMG_EINVAL, "h must be > 0");
    const bool labeled = !c->labels.empty();
    if (labeled && (c->nparts > 1 || c->ndist > 0))
        throw SmgError(SMG_EINVAL, "labelled domains: single-part contexts only");
    std::vector<uint8_t> lab = c->labels;  // labels of the level being built
    const int div = 1 << (p.levels - 1);
    if (g.nx % div || g.ny % div || g.nz % div)
        throw SmgError(SMG_EINVAL, "extents must be divisible by 2^(levels-1)");
    if (g.nx > 1024 || g.ny > 1024 || g.nz > 1024) throw SmgError(SMG_EINVAL, "extents above 1024 per GPU");
    if (g.nx / div < 2 || g.ny / div < 2 || g.nz / div < 2)
        throw SmgError(SMG_EINVAL, "coarsened extent below 2 (SPEC:82)");
    CK(cudaSetDevice(c->device));
    if (shared_stream) {
        c->st = shared_stream;
        c->own_stream = false;
    } else {
        CK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
    }
    CK(cudaEventCreate(&c->ev0));
    CK(cudaEventCreate(&c->ev1));
    c->lv.resize(p.levels);
    int max_vk = 1;
    for (int l = 0; l < p.levels; ++l) {
        DevLevel& L = c->lv[l];
        const int nx = g.nx >> l, ny = g.ny >> l, nz = g.nz >> l;
        const double h = g.h * static_cast<double>(1 << l);
        const bool dist = l < c->ndist;
        const int nzl = dist ? nz / c->nparts : nz, z0 = dist ? c->rank * nzl : 0;
        L.k.g = dist ? make_geom(nx, ny, nzl, z0, nz, 2) : make_geom(nx, ny, nz);
        L.k.eta_h2 = p.eta / (h * h);
        L.k.inv_h = 1.0 / h;
        L.k.gamma = p.gamma;
        L.k.dv = 6.0 * L.k.eta_h2;
        L.k.dp = -6.0 * (1.0 + p.gamma * p.eta) / (h * h);
        L.k.bw = p.band_width;
        L.k.tiled = (!labeled && dgs_tiled(nx, ny, nz, p.dgs_tile_min)) ? 1 : 0;
        L.counts[0] = static_cast<int64_t>(nx - 1) * ny * nz;
        L.counts[1] = static_cast<int64_t>(nx) * (ny - 1) * nz;
        L.counts[2] = static_cast<int64_t>(nx) * ny * (nz - 1);
        L.counts[3] = static_cast<int64_t>(nx) * ny * nz;
        L.N = L.counts[0] + L.counts[1] + L.counts[2] + L.counts[3];
        const int64_t vl = vlen(L);
        L.x = c->dalloc<double>(vl);
        L.b = c->dalloc<double>(vl);
        L.r = c->dalloc<double>(vl);
        L.pd = c->dalloc<double>(L.k.g.fs);
        if (p.cycle == 1 && l >= 2 && l + 1 < p.levels) {
            L.wb = c->dalloc<double>(vl);
            L.wx = c->dalloc<double>(vl);
        }
        L.pd0 = c->dalloc<double>(L.k.g.fs);
        L.pd1 = c->dalloc<double>(L.k.g.fs);
        L.k.cb = c->dalloc<double>(L.k.g.fs);
        if (L.k.tiled) L.k.bp = c->dalloc<double>(static_cast<int64_t>(5) * L.k.g.nx * L.k.g.ny * L.k.g.nz);
        if (labeled) {
            if (l > 0) lab = coarsen_labels(lab, nx * 2, ny * 2, nz * 2);
            build_level_labeled(c, l, lab, max_vk);
            continue;
        }
        // Vanka blocks: band cells, slot + active-face mask, by colour
        const int bw = p.band_width;
        auto band = [&](int x, int y, int z) {
            return x < bw || y < bw || z < bw || x >= nx - bw || y >= ny - bw || z >= nz - bw;
        };
        std::vector<int32_t> cells[8];
        std::vector<uint8_t> masks[8], amasks[8];
        bool used[64] = {};
        int64_t v1 = 0;
        for (int z = 0; z < nz; ++z)
            for (int y = 0; y < ny; ++y)
                for (int x = 0; x < nx; ++x) {
                    const bool bc = band(x, y, z);
                    // V1 census: faces on the low side of this cell + its pressure
                    if (x >= 1 && (bc || band(x - 1, y, z))) ++v1;
                    if (y >= 1 && (bc || band(x, y - 1, z))) ++v1;
                    if (z >= 1 && (bc || band(x, y, z - 1))) ++v1;
                    if (!bc) continue;
                    ++v1;
                    // Vanka blocks of the owned planes, plus (z-slabs) the band blocks of the halo plane
                    // below, recomputed here only to apply their top w face, which lives in plane z0
                    const bool owned = z >= z0 && z < z0 + nzl;
                    const bool halo_below = dist && c->rank > 0 && z == z0 - 1;
                    if (!owned && !halo_below) continue;
                    int am = 127;
                    if (halo_below) am = 32;
                    else if (dist && z == z0 + nzl - 1 && z + 1 < nz) am = 127 & ~32;
                    int m = 0;
                    if (x >= 1) m |= 1;
                    if (x + 1 <= nx - 1) m |= 2;
                    if (y >= 1) m |= 4;
                    if (y + 1 <= ny - 1) m |= 8;
                    if (z >= 1) m |= 16;
                    if (z + 1 <= nz - 1) m |= 32;
                    const int col = (x & 1) + 2 * (y & 1) + 4 * (z & 1);
                    cells[col].push_back(static_cast<int32_t>(L.k.g.slot(x, y, z - z0)));
                    masks[col].push_back(static_cast<uint8_t>(m));
                    amasks[col].push_back(static_cast<uint8_t>(am));
                    used[m] = true;
                }
        L.counts[4] = v1;
        if (!dist) {  // read set of the band blocks: their 7 DOFs and every stencil input of their residuals
            const Geom& G = L.k.g;
            std::vector<uint8_t> need(static_cast<size_t>(G.vec_len()), 0);
            auto mark_mom = [&](int64_t f, int64_t sn, int64_t pfield) {
                const int64_t o[7] = {0, -1, 1, -G.sy, G.sy, -G.sz, G.sz};
                for (int64_t d : o) need[f + d] = 1;
                need[pfield] = 1;
                need[pfield - sn] = 1;
            };
            for (int col = 0; col < 8; ++col)
                for (size_t t = 0; t < cells[col].size(); ++t) {
                    const int64_t i = cells[col][t];
                    const int m = masks[col][t];
                    const int64_t fs = G.fs;
                    const int64_t P = 3 * fs + i;
                    if (m & 1) mark_mom(i, 1, P);
                    if (m & 2) mark_mom(i + 1, 1, P + 1);
                    if (m & 4) mark_mom(fs + i, G.sy, P);
                    if (m & 8) mark_mom(fs + i + G.sy, G.sy, P + G.sy);
                    if (m & 16) mark_mom(2 * fs + i, G.sz, P);
                    if (m & 32) mark_mom(2 * fs + i + G.sz, G.sz, P + G.sz);
                    need[i] = need[i + 1] = need[fs + i] = need[fs + i + G.sy] = need[2 * fs + i] =
                        need[2 * fs + i + G.sz] = need[P] = 1;
                }
            // minus the DOFs the sweep's first phase writes (list vanka_order(0) = parity 0, with
            // parity 7 when that pair is merged): the refresh then runs concurrently with the
            // first phase (no conflicting writes; the first phase reads only x)
            int nsz[8];
            for (int col = 0; col < 8; ++col) nsz[col] = static_cast<int>(cells[col].size());
            const int pm0 = vanka_pairs_pay(nsz);
            for (int col : {0, 7}) {
                if (col == 7 && !(pm0 & 1)) continue;
                for (size_t t = 0; t < cells[col].size(); ++t) {
                    const int64_t i = cells[col][t];
                    const int m = masks[col][t];
                    const int64_t fs = G.fs;
                    const int64_t dof[7] = {i, i + 1, fs + i, fs + i + G.sy, 2 * fs + i, 2 * fs + i + G.sz, 3 * fs + i};
                    for (int q = 0; q < 7; ++q)
                        if (q == 6 || (m & (1 << q))) need[dof[q]] = 0;
                }
            }
            std::vector<int32_t> lst;
            for (int64_t k = 0; k < static_cast<int64_t>(need.size()); ++k)
                if (need[k]) lst.push_back(static_cast<int32_t>(k));
            L.vk_nrefresh = static_cast<int64_t>(lst.size());
            L.vk_refresh = c->dalloc<int32_t>(L.vk_nrefresh);
            CK(cudaMemcpyAsync(L.vk_refresh, lst.data(), lst.size() * sizeof(int32_t), cudaMemcpyHostToDevice, c->st));
            L.xb = c->dalloc<double>(G.vec_len());
            CK(cudaStreamSynchronize(c->st));
        }
        for (int col = 0; col < 8; ++col) {
            L.vk_n[col] = static_cast<int>(cells[col].size());
            max_vk = std::max(max_vk, L.vk_n[col]);
            L.vk_cells[col] = c->dalloc<int32_t>(L.vk_n[col]);
            L.vk_mask[col] = c->dalloc<uint8_t>(L.vk_n[col]);
            CK(cudaMemcpyAsync(L.vk_cells[col], cells[col].data(), cells[col].size() * sizeof(int32_t),
                               cudaMemcpyHostToDevice, c->st));
            CK(cudaMemcpyAsync(L.vk_mask[col], masks[col].data(), masks[col].size(), cudaMemcpyHostToDevice, c->st));
            if (dist) {
                L.vk_amask[col] = c->dalloc<uint8_t>(L.vk_n[col]);
                CK(cudaMemcpyAsync(L.vk_amask[col], amasks[col].data(), amasks[col].size(), cudaMemcpyHostToDevice,
                                   c->st));
            }
            CK(cudaStreamSynchronize(c->st));
        }
        // sweep lists: complementary pairs (m, 7-m) folded into list m (one phase each; see
        // VankaLists in kernels.cu)
        for (int col = 0; col < 8; ++col) {
            L.sw_cells[col] = L.vk_cells[col];
            L.sw_mask[col] = L.vk_mask[col];
            L.sw_amask[col] = L.vk_amask[col];
            L.sw_n[col] = L.vk_n[col];
        }
        L.sw_pairs = VankaPairs{};
        // slab levels run per-phase kernels (no persistent-sweep capacity to respect): always merge,
        // so every part of a level takes the same 8 phases
        const int pm = dist ? 0xf : vanka_pairs_pay(L.vk_n);
        for (int pq = 0; pq < 4; ++pq) {
            if (!((pm >> pq) & 1)) continue;
            std::vector<int32_t> mc(cells[pq]);
            mc.insert(mc.end(), cells[7 - pq].begin(), cells[7 - pq].end());
            std::vector<uint8_t> mm(masks[pq]);
            mm.insert(mm.end(), masks[7 - pq].begin(), masks[7 - pq].end());
            L.sw_n[pq] = static_cast<int>(mc.size());
            L.sw_n[7 - pq] = 0;
            max_vk = std::max(max_vk, L.sw_n[pq]);
            L.sw_cells[pq] = c->dalloc<int32_t>(L.sw_n[pq]);
            L.sw_mask[pq] = c->dalloc<uint8_t>(L.sw_n[pq]);
            CK(cudaMemcpyAsync(L.sw_cells[pq], mc.data(), mc.size() * sizeof(int32_t), cudaMemcpyHostToDevice, c->st));
            CK(cudaMemcpyAsync(L.sw_mask[pq], mm.data(), mm.size(), cudaMemcpyHostToDevice, c->st));
            if (dist) {
                std::vector<uint8_t> ma(amasks[pq]);
                ma.insert(ma.end(), amasks[7 - pq].begin(), amasks[7 - pq].end());
                L.sw_amask[pq] = c->dalloc<uint8_t>(L.sw_n[pq]);
                CK(cudaMemcpyAsync(L.sw_amask[pq], ma.data(), ma.size(), cudaMemcpyHostToDevice, c->st));
            }
            CK(cudaStreamSynchronize(c->st));
            L.sw_pairs.pairs |= 1 << pq;
            L.sw_pairs.first[pq] = static_cast<int>(cells[pq].size());
        }
        if (p.vanka == 1 && !dist) {
            std::vector<int32_t> ac;
            std::vector<uint8_t> am;
            for (int col = 0; col < 8; ++col) {
                ac.insert(ac.end(), cells[col].begin(), cells[col].end());
                am.insert(am.end(), masks[col].begin(), masks[col].end());
            }
            L.va_n = static_cast<int>(ac.size());
            L.va_cells = c->dalloc<int32_t>(L.va_n);
            L.va_mask = c->dalloc<uint8_t>(L.va_n);
            L.va_d7 = c->dalloc<double>(7 * L.k.g.fs);
            CK(cudaMemcpyAsync(L.va_cells, ac.data(), ac.size() * sizeof(int32_t), cudaMemcpyHostToDevice, c->st));
            CK(cudaMemcpyAsync(L.va_mask, am.data(), am.size(), cudaMemcpyHostToDevice, c->st));
            CK(cudaStreamSynchronize(c->st));
        }
        if (p.vanka == 2 && !dist && l + 1 < p.levels) {  // direct-on-V1: A11^{-1}, dense (capped like the coarsest)
            std::vector<int32_t> sel, vslots;
            const int n1 = v1_selection(L, bw, sel);
            if (n1 > 20000) throw SmgError(SMG_ECAP, "direct-on-V1: |V1| above the dense cap 20000 (SPEC:365)");
            std::vector<double> A11;
            assemble_box_dense(L, p.gamma, sel.data(), n1, A11, vslots);
            const std::vector<double> K1 = dense_inverse_sym(std::move(A11), n1);
            L.v1_n = n1;
            L.v1_k = c->dalloc<double>(static_cast<int64_t>(n1) * n1);
            L.v1_slots = c->dalloc<int32_t>(n1);
            CK(cudaMemcpyAsync(L.v1_k, K1.data(), K1.size() * sizeof(double), cudaMemcpyHostToDevice, c->st));
            CK(cudaMemcpyAsync(L.v1_slots, vslots.data(), vslots.size() * sizeof(int32_t), cudaMemcpyHostToDevice, c->st));
            CK(cudaStreamSynchronize(c->st));
        }
        // local inverses C_i L~ C_i^T per face mask, scattered to the 7-slot layout
        std::vector<double> ktab(64 * 49, 0.0);
        for (int m = 0; m < 64; ++m) {
            if (!used[m]) continue;
            int slot[7], nb = 0;
            for (int s = 0; s < 6; ++s)
                if (m & (1 << s)) slot[nb++] = s;
            slot[nb++] = 6;
            double lm[49] = {}, inv[49];
            for (int a = 0; a < nb; ++a)
                for (int b2 = 0; b2 < nb; ++b2) {
                    const int sa = slot[a], sb = slot[b2];
                    double v = 0.0;
                    if (sa < 6 && sb < 6) {
                        if (sa == sb) v = 6.0 * L.k.eta_h2;
                        else if ((sa >> 1) == (sb >> 1)) v = -L.k.eta_h2;  // uL-uR of one cell
                    } else if (sa < 6 && sb == 6) {
                        v = (sa & 1) ? -L.k.inv_h : L.k.inv_h;  // left face: cell is p_right
                    } else if (sa == 6 && sb < 6) {
                        v = (sb & 1) ? -L.k.inv_h : L.k.inv_h;
                    } else {
                        v = -p.gamma;
                    }
                    lm[a * nb + b2] = v;
                }
            small_inverse(lm, nb, inv);
            for (int a = 0; a < nb; ++a)
                for (int b2 = 0; b2 < nb; ++b2) ktab[m * 49 + slot[a] * 7 + slot[b2]] = inv[a * nb + b2];
        }
        L.ktab = c->dalloc<double>(64 * 49);
        CK(cudaMemcpyAsync(L.ktab, ktab.data(), ktab.size() * sizeof(double), cudaMemcpyHostToDevice, c->st));
        CK(cudaStreamSynchronize(c->st));
    }
    c->vk_delta = c->dalloc<double>(static_cast<int64_t>(max_vk) * 8);

    // coarsest level: dense L~ in compact order, symmetric inverse (OD-4)
    DevLevel& C = c->lv.back();
    if (C.N > 20000) throw SmgError(SMG_ECAP, "coarsest system above dense cap 20000 (SPEC:365): add levels");
    const int n = static_cast<int>(C.N);
    c->nc = n;
    std::vector<double> A;
    std::vector<int32_t> slots;
    if (labeled) assemble_labeled_dense(C, p.gamma, nullptr, n, A, slots);
    else assemble_box_dense(C, p.gamma, nullptr, n, A, slots);
    std::vector<double> K;
    if (shared_coarse) K = *shared_coarse;  // same matrix on every part: factorise once
    else if (n > 0) K = dense_inverse_sym(std::move(A), n);
    if (coarse_out) *coarse_out = K;
    c->coarse_k = c->dalloc<double>(static_cast<int64_t>(n) * n);
    c->coarse_slots = c->dalloc<int32_t>(n);
    CK(cudaMemcpyAsync(c->coarse_k, K.data(), K.size() * sizeof(double), cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(c->coarse_slots, slots.data(), slots.size() * sizeof(int32_t), cudaMemcpyHostToDevice, c->st));

    // SQMR vectors and reduction scratch
    const int64_t vl0 = vlen(c->lv[0]);
    c->q = c->dalloc<double>(vl0);
    c->d = c->dalloc<double>(vl0);
    c->xs = c->dalloc<double>(vl0);
    c->q2 = c->dalloc<double>(vl0);
    c->d2 = c->dalloc<double>(vl0);
    c->xs2 = c->dalloc<double>(vl0);
    c->rhs = c->dalloc<double>(vl0);
    int64_t maxN = 0;
    for (auto& L : c->lv) maxN = std::max(maxN, L.N);
    c->compact = c->dalloc<double>(maxN);
    c->partials = c->dalloc<double>(dot_partials(c->lv[0].k.g));  // zero outside this part's blocks
    c->dscal = c->dalloc<double>(S_COUNT);
    CK(cudaMallocHost(&c->hscal, 8 * sizeof(double)));
    CK(cudaStreamSynchronize(c->st));
}

// ---- V-cycle orchestration (Alg. 1 + Alg. 3) ----
void vanka_sym(smg_ctx* c, int l, double* x, const double* b) {
    DevLevel& L = c->lv[l];
    for (int pass = 0; pass < 2; ++pass)
        for (int k = 0; k < 8; ++k) {
            const int col = vanka_order(pass == 0 ? k : 7 - k);
            launch_vanka_delta(L.k, x, b, L.vk_cells[col], L.vk_mask[col], L.vk_n[col], L.ktab, c->vk_delta, c->st,
                               L.vk_kidx[col]);
            launch_vanka_apply(L.k, x, L.vk_cells[col], L.vk_mask[col], L.vk_n[col], c->vk_delta, c->st);
        }
}

// DGS phases (OD-1): forward 0,1 velocity red/black; 2..9 pressure parity
// colours 0..7; reverse 10..17 pressure colours 7..0; 18,19 velocity black/red.
constexpr int kDgsPhases = 20;
void dgs_phase(smg_ctx* c, int l, double* x, const double* b, int ph) {
    DevLevel& L = c->lv[l];
    if (L.k.tiled) {  // arg = phase + 32 T: one phase on the tiles of colour T
        const int T = ph >> 5;
        ph &= 31;
        if (T > 7 || ph >= kDgsPhases) throw SmgError(SMG_EINVAL, "bad DGS phase / tile colour");
        if (ph >= 10 && ph <= 17) launch_dgs_cb(L.k, b, c->st);
        launch_dgs_tile_phases(L.k, x, b, T, ph, ph + 1, c->st);
        return;
    }
    if (ph == 0 || ph == 1) {
        launch_dgs_vel(L.k, x, b, ph, c->st);
    } else if (ph >= 2 && ph <= 9) {
        launch_dgs_pdelta(L.k, x, b, L.pd, ph - 2, c->st);
        launch_dgs_papply(L.k, x, L.pd, c->st, ph - 2);
    } else if (ph >= 10 && ph <= 17) {
        launch_dgs_cb(L.k, b, c->st);
        launch_dgs_prev(L.k, x, b, 17 - ph, c->st);
    } else if (ph == 18 || ph == 19) {
        launch_dgs_vel(L.k, x, b, 19 - ph, c->st);
    } else {
        throw SmgError(SMG_EINVAL, "bad DGS phase");
    }
}

// cb_ready: L.k.cb already holds m_C^T b for this b (the V-cycle fills it once for
// the pre- and post-smooth of a level visit)
void symmetric_dgs(smg_ctx* c, int l, double* x, const double* b, bool cb_ready = false) {
    const int nph = (c->prm.flags & SMG_FLAG_SKIP_REVERSE_DGS) ? kDgsPhases / 2 : kDgsPhases;
    DevLevel& L = c->lv[l];
    if (nph > kDgsPhases / 2 && !cb_ready) launch_dgs_cb(L.k, b, c->st);  // m_C^T b for the reverse steps
    if (L.k.cls) {  // labelled level: one masked kernel per phase
        for (int ph = 0; ph < nph; ++ph) {
            if (ph <= 1 || ph >= 18) {
                launch_dgs_vel(L.k, x, b, ph <= 1 ? ph : 19 - ph, c->st);
            } else if (ph <= 9) {
                launch_dgs_pdelta(L.k, x, b, L.pd, ph - 2, c->st);
                launch_dgs_papply(L.k, x, L.pd, c->st, ph - 2);
            } else {
                launch_dgs_prev(L.k, x, b, 17 - ph, c->st);
            }
        }
        return;
    }
    if (L.k.tiled) {
        launch_dgs_tiled(L.k, x, b, nph, c->st, /*packed=*/cb_ready || nph > kDgsPhases / 2);
        return;
    }
    launch_dgs_sym_coop(L.k, x, b, L.pd0, L.pd1, nph, c->st, L.xb);
}

void vanka_sym_coop(smg_ctx* c, int l, double* x, const double* b) {
    DevLevel& L = c->lv[l];
    if (L.k.cls) {  // labelled level: merged colour pairs 0..3, then 3..0, a delta / apply launch each
        for (int k = 0; k < c->prm.nu; ++k)
            for (int ph = 0; ph < 8; ++ph) {
                const int pq = ph < 4 ? ph : 7 - ph;
                launch_vanka_delta(L.k, x, b, L.sw_cells[pq], L.sw_mask[pq], L.sw_n[pq], L.ktab, c->vk_delta, c->st,
                                   L.sw_kidx[pq]);
                launch_vanka_apply(L.k, x, L.sw_cells[pq], L.sw_mask[pq], L.sw_n[pq], c->vk_delta, c->st);
            }
        return;
    }
    launch_vanka_sym_coop(L.k, x, b, L.sw_cells, L.sw_mask, L.sw_n, L.ktab, c->vk_delta, c->prm.nu, c->st, L.xb,
                          L.vk_refresh, L.vk_nrefresh, L.sw_pairs);
}

void vanka_additive(smg_ctx* c, int l, double* x, const double* b) {
    DevLevel& L = c->lv[l];
    if (!L.va_d7) throw SmgError(SMG_EINVAL, "additive Vanka needs params.vanka = 1 (single-part contexts)");
    launch_vanka_additive(L.k, x, b, L.va_cells, L.va_mask, L.va_n, L.ktab, L.va_d7, c->prm.omega, c->st, L.va_kidx);
}

// direct-on-V1: x_V1 += A11^{-1} (b - L~x)_V1 -- the residual into the level's r
// scratch, then the dense symmetric inverse applied in the coarse GEMV's summation order
void vanka_direct(smg_ctx* c, int l, double* x, const double* b) {
    DevLevel& L = c->lv[l];
    if (!L.v1_k) throw SmgError(SMG_EINVAL, "direct-on-V1 needs params.vanka = 2 (single-part contexts)");
    launch_apply(L.k, x, b, L.r, L.k.gamma, c->st);
    launch_coarse_gemv(L.v1_k, L.v1_slots, L.v1_n, L.r, x, c->st, /*accumulate=*/true);
}

void smooth(smg_ctx* c, int l, double* x, const double* b, bool cb_ready = false) {
    Nvtx r("smooth", l);
    if (c->prm.vanka == 2) {  // Alg. 3 with the exact V1 solve (idempotent: once per side)
        vanka_direct(c, l, x, b);
        symmetric_dgs(c, l, x, b, cb_ready);
        vanka_direct(c, l, x, b);
        return;
    }
    if (c->prm.vanka == 1) {  // Alg. 3 with additive Vanka on V1
        for (int k = 0; k < c->prm.nu; ++k) vanka_additive(c, l, x, b);
        symmetric_dgs(c, l, x, b, cb_ready);
        for (int k = 0; k < c->prm.nu; ++k) vanka_additive(c, l, x, b);
        return;
    }
    vanka_sym_coop(c, l, x, b);
    symmetric_dgs(c, l, x, b, cb_ready);
    vanka_sym_coop(c, l, x, b);
}

void coarse_solve(smg_ctx* c, const double* b, double* x) {
    launch_coarse_gemv(c->coarse_k, c->coarse_slots, c->nc, b, x, c->st);
}

void vcycle(smg_ctx* c, int l, const double* b, double* x) {
    Nvtx r("vcycle", l);
    DevLevel& L = c->lv[l];
    if (l == static_cast<int>(c->lv.size()) - 1) { coarse_solve(c, b, x); return; }
    CK(cudaMemsetAsync(x, 0, vlen(L) * sizeof(double), c->st));
    const bool cb = !(c->prm.flags & SMG_FLAG_SKIP_REVERSE_DGS);
    if (cb) launch_dgs_cb(L.k, b, c->st);  // m_C^T b once for both smooths of this visit
    smooth(c, l, x, b, cb);
    DevLevel& C = c->lv[l + 1];
    launch_apply(L.k, x, b, L.r, L.k.gamma, c->st);
    launch_restrict(L.k, C.k, L.r, C.b, c->st);
    vcycle(c, l + 1, C.b, C.x);
    // W-cycle: second recursive call below the finest level, on the residual of
    // the first (skipped when the child is the exact coarsest solve)
    if (c->prm.cycle == 1 && l >= 1 && l + 2 < static_cast<int>(c->lv.size())) {
        launch_apply(C.k, C.x, C.b, C.wb, C.k.gamma, c->st);
        vcycle(c, l + 1, C.wb, C.wx);
        launch_axpy(C.x, C.wx, 1.0, vlen(C), c->st);
    }
    launch_prolong_add(L.k, C.k, C.x, x, c->st);
    smooth(c, l, x, b, cb);
}

// ---- host <-> device compact vectors ----
void upload(smg_ctx* c, int l, const double* host, double* dev_padded) {
    DevLevel& L = c->lv[l];
    CK(cudaMemcpyAsync(c->compact, host, L.N * sizeof(double), cudaMemcpyHostToDevice, c->st));
    if (L.pack_slots) launch_scatter(L.pack_slots, L.N, c->compact, dev_padded, c->st);
    else launch_unpack(L.k, c->compact, dev_padded, c->st);
}
void download(smg_ctx* c, int l, const double* dev_padded, double* host) {
    DevLevel& L = c->lv[l];
    if (L.pack_slots) launch_gather(L.pack_slots, L.N, dev_padded, c->compact, c->st);
    else launch_pack(L.k, dev_padded, c->compact, c->st);
    CK(cudaMemcpyAsync(host, c->compact, L.N * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
}

// =================================================== z-slab decomposition ====
// P parts each own a z-slab of every level l < ndist (2 halo
// planes per side) and a replicated copy of the coarser levels.  Every smoother
// phase on a slab level is followed by a halo exchange, so each part applies
// exactly the single-GPU per-point updates to its planes: results are
// bit-identical to one part.  Parts may share one device (emulation, used by
// the tests) or sit on separate devices (peer copies, cudaMemcpyDefault).
using Sel = double* (*)(DevLevel&);
double* sel_x(DevLevel& L) { return L.x; }
double* sel_b(DevLevel& L) { return L.b; }
double* sel_r(DevLevel& L) { return L.r; }
double* sel_d0(DevLevel& L) { return L.pd0; }
double* sel_d1(DevLevel& L) { return L.pd1; }

bool shared_stream(smg_ctx* m) {
    for (smg_ctx* p : m->parts)
        if (p->st != m->st) return false;
    return true;
}

// stream a transport of part p is enqueued on: the part's compute stream, or its comm stream
// while the master context is in an overlapped phase (on_cst)
cudaStream_t tstream(smg_ctx* m, smg_ctx* p) { return m->on_cst ? p->cst : p->st; }
ncclComm_t tcomm(smg_ctx* m) { return m->on_cst ? m->hcomm : m->comm; }

// stream-order barrier across parts (no-op when all parts share one stream), on the transport streams
void part_barrier(smg_ctx* m) {
    if (shared_stream(m)) return;
    std::vector<cudaEvent_t> ev(m->parts.size());
    for (size_t k = 0; k < m->parts.size(); ++k) {
        CK(cudaSetDevice(m->parts[k]->device));
        CK(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming));
        CK(cudaEventRecord(ev[k], tstream(m, m->parts[k])));
    }
    for (size_t k = 0; k < m->parts.size(); ++k) {
        CK(cudaSetDevice(m->parts[k]->device));
        for (size_t j = 0; j < ev.size(); ++j)
            if (j != k) CK(cudaStreamWaitEvent(tstream(m, m->parts[k]), ev[j], 0));
    }
    for (auto e : ev) cudaEventDestroy(e);
    CK(cudaSetDevice(m->device));
}

// Comm streams and fork / join events of every part, and (one process per GPU) the halo
// communicator: created at the first overlapped phase.
void ensure_comm_streams(smg_ctx* m) {
    if (m->cst) return;
    for (smg_ctx* p : m->parts) {
        CK(cudaSetDevice(p->device));
        if (p != m && p->st == m->st) {
            p->cst = m->cst;
        } else {
            CK(cudaStreamCreateWithFlags(&p->cst, cudaStreamNonBlocking));
            p->own_cst = true;
        }
        CK(cudaEventCreateWithFlags(&p->evb, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&p->evc, cudaEventDisableTiming));
    }
    CK(cudaSetDevice(m->device));
    if (m->mp && !m->hcomm) {
        const NcclApi& N = nccl();
        m->hcomm = m->comm;
        if (N.commSplit) {
            ncclComm_t h = nullptr;
            if (N.commSplit(m->comm, 0, m->rank, &h, nullptr) == ncclSuccess && h) m->hcomm = h;
        }
    }
}

// multi-process halo exchange of this rank's slab vector `v` (geometry g, nf fields):
// the same 2-plane transfers as the in-process copies below, as NCCL send/recv
// pairs with the z neighbours (rank -+ 1), grouped into one launch on the transport stream
void halo_nccl(smg_ctx* m, double* v, const Geom& g, int nf, int f0 = 0) {
    const NcclApi& N = nccl();
    const size_t n2 = static_cast<size_t>(2 * g.sz);
    cudaStream_t ts = tstream(m, m);
    ncclComm_t cm = tcomm(m);
    NK(N.groupStart());
    for (int f = f0; f < f0 + nf; ++f) {
        double* a = v + f * g.fs;
        if (m->rank + 1 < m->nparts) {  // top halo (planes nz, nz+1) <-> upper part's planes 0, 1
            NK(N.send(a + (g.zg + g.nz - 2) * g.sz, n2, ncclDouble, m->rank + 1, cm, ts));
            NK(N.recv(a + (g.zg + g.nz) * g.sz, n2, ncclDouble, m->rank + 1, cm, ts));
        }
        if (m->rank > 0) {  // bottom halo (planes -2, -1) <-> lower part's planes nz-2, nz-1
            NK(N.send(a + g.zg * g.sz, n2, ncclDouble, m->rank - 1, cm, ts));
            NK(N.recv(a, n2, ncclDouble, m->rank - 1, cm, ts));
        }
    }
    NK(N.groupEnd());
}

// halo exchange of a slab level: 2 planes each way between neighbours; the nf fields from f0
// (a phase that changed only some fields refreshes only those: the other halos are still current)
void exchange(smg_ctx* m, int l, Sel sel, int nf, int f0 = 0) {
    Nvtx r("halo_exchange", l);
    if (m->mp) {
        halo_nccl(m, sel(m->lv[l]), m->lv[l].k.g, nf, f0);
        return;
    }
    part_barrier(m);
    for (size_t p = 0; p + 1 < m->parts.size(); ++p) {
        DevLevel &lo = m->parts[p]->lv[l], &hi = m->parts[p + 1]->lv[l];
        const Geom& g = lo.k.g;
        const size_t pitch = g.fs * sizeof(double), width = 2 * g.sz * sizeof(double);
        double *vlo = sel(lo) + f0 * g.fs, *vhi = sel(hi) + f0 * g.fs;
        // lo top halo (planes nz, nz+1) <- hi owned planes 0, 1
        CK(cudaMemcpy2DAsync(vlo + (g.nz + g.zg) * g.sz, pitch, vhi + g.zg * g.sz, pitch, width, nf,
                             cudaMemcpyDefault, tstream(m, m->parts[p])));
        // hi bottom halo (planes -2, -1) <- lo owned planes nz-2, nz-1
        CK(cudaMemcpy2DAsync(vhi, pitch, vlo + g.nz * g.sz, pitch, width, nf, cudaMemcpyDefault,
                             tstream(m, m->parts[p + 1])));
    }
    part_barrier(m);
}

// every part's owned coarse planes [z0c, z0c + nzc) of a replicated level -> all parts
void allgather_planes(smg_ctx* m, int l, Sel sel, int nzc) {
    const Geom& g = m->lv[l].k.g;
    if (m->mp) {  // per field, the parts' plane ranges are contiguous and rank-ordered: in-place all-gather
        const NcclApi& N = nccl();
        const size_t cnt = static_cast<size_t>(nzc) * g.sz;
        NK(N.groupStart());
        for (int f = 0; f < 4; ++f) {
            double* base = sel(m->lv[l]) + f * g.fs + g.zg * g.sz;
            NK(N.allGather(base + m->rank * cnt, base, cnt, ncclDouble, m->comm, m->st));
        }
        NK(N.groupEnd());
        return;
    }
    part_barrier(m);
    const size_t pitch = g.fs * sizeof(double), width = nzc * g.sz * sizeof(double);
    for (size_t p = 0; p < m->parts.size(); ++p)
        for (size_t q = 0; q < m->parts.size(); ++q) {
            if (p == q) continue;
            const int64_t off = (static_cast<int64_t>(p) * nzc + g.zg) * g.sz;
            CK(cudaMemcpy2DAsync(sel(m->parts[q]->lv[l]) + off, pitch, sel(m->parts[p]->lv[l]) + off, pitch, width, 4,
                                 cudaMemcpyDefault, m->parts[q]->st));
        }
    part_barrier(m);
}

template <class F>
void each(smg_ctx* m, F&& f) {
    for (smg_ctx* p : m->parts) {
        CK(cudaSetDevice(p->device));
        f(p);
    }
    CK(cudaSetDevice(m->device));
}

// Halo refresh after a Vanka phase on a slab level: the phase changed band DOFs only, which on the
// exchanged planes is a frame along the x and y walls (kernels.cu k_frame_copy) unless the planes
// are within reach of a z wall (thin slabs: the whole planes go).  Pack the frames of the 2 planes x
// 4 fields, move them (NCCL send/recv or a peer copy), unpack into the ghost planes: ~1.5% of the
// plane bytes at 512^2.
void exchange_frame(smg_ctx* m, int l) {
    const Geom& g0 = m->lv[l].k.g;
    const int bw = m->lv[l].k.bw;
    // SMG_DIST_FRAMES: 0 = never, 2 = wherever the geometry allows (tests), default: where the planes
    // are large enough for the saved transfer to pay for the pack and unpack launches (>= 2 MiB per
    // direction, i.e. planes from about 180^2 slots: ~2 us at NVLink speed against ~3 us of launches
    // plus the ~10 us either message costs)
    const int mode = std::getenv("SMG_DIST_FRAMES") ? std::atoi(std::getenv("SMG_DIST_FRAMES")) : 1;
    const bool large = 8 * g0.sz * static_cast<int64_t>(sizeof(double)) >= (int64_t{2} << 20);
    if (mode == 0 || (mode == 1 && !large) || g0.nz < bw + 4 || g0.nx < 4 * (bw + 2) || g0.ny < 4 * (bw + 2)) {
        exchange(m, l, sel_x, 4);
        return;
    }
    Nvtx r("halo_frames", l);
    if (!m->fbuf[0]) {  // sized for the finest level (the largest planes)
        each(m, [&](smg_ctx* p) {
            const int64_t n = frame_doubles(p->lv[0].k.g, p->lv[0].k.bw);
            for (double*& b : p->fbuf) b = p->dalloc<double>(n);
        });
    }
    const int64_t n = frame_doubles(g0, bw);
    const int P = m->nparts;
    auto pack = [&](smg_ctx* p) {  // top planes nz-2, nz-1 -> fbuf[0]; bottom planes 0, 1 -> fbuf[1]
        const Geom& g = p->lv[l].k.g;
        launch_frame_copy(g, bw, p->lv[l].x, p->rank + 1 < P ? p->fbuf[0] : nullptr, g.zg + g.nz - 2,
                          p->rank > 0 ? p->fbuf[1] : nullptr, g.zg, true, p->st);
    };
    auto unpack = [&](smg_ctx* p) {  // fbuf[2] -> ghost planes nz, nz+1; fbuf[3] -> ghost planes -2, -1
        const Geom& g = p->lv[l].k.g;
        launch_frame_copy(g, bw, p->lv[l].x, p->rank + 1 < P ? p->fbuf[2] : nullptr, g.zg + g.nz,
                          p->rank > 0 ? p->fbuf[3] : nullptr, 0, false, p->st);
    };
    if (m->mp) {
        const NcclApi& N = nccl();
        pack(m);
        NK(N.groupStart());
        if (m->rank + 1 < P) {
            NK(N.send(m->fbuf[0], static_cast<size_t>(n), ncclDouble, m->rank + 1, m->comm, m->st));
            NK(N.recv(m->fbuf[2], static_cast<size_t>(n), ncclDouble, m->rank + 1, m->comm, m->st));
        }
        if (m->rank > 0) {
            NK(N.send(m->fbuf[1], static_cast<size_t>(n), ncclDouble, m->rank - 1, m->comm, m->st));
            NK(N.recv(m->fbuf[3], static_cast<size_t>(n), ncclDouble, m->rank - 1, m->comm, m->st));
        }
        NK(N.groupEnd());
        unpack(m);
        return;
    }
    each(m, pack);
    part_barrier(m);
    for (size_t q = 0; q + 1 < m->parts.size(); ++q) {
        smg_ctx *lo = m->parts[q], *hi = m->parts[q + 1];
        CK(cudaMemcpyAsync(hi->fbuf[3], lo->fbuf[0], n * sizeof(double), cudaMemcpyDefault, hi->st));
        CK(cudaMemcpyAsync(lo->fbuf[2], hi->fbuf[1], n * sizeof(double), cudaMemcpyDefault, lo->st));
    }
    each(m, unpack);
    part_barrier(m);  // the next pack must not overwrite a frame a neighbour is still copying
}

// Symmetric multiplicative Vanka on a slab level: the merged complementary colour pairs of the
// single-part sweep (8 Jacobi phases instead of 16 when all four pairs pay, bit-identical), one halo
// exchange per phase.  The pair decision depends on the level's global list sizes only through
// vanka_pairs_pay of this part's lists; parts of one level hold the same colours, so every part
// takes the same phases.
void dist_vanka_sym(smg_ctx* m, int l) {
    const int pairs = m->lv[l].sw_pairs.pairs;
    for (smg_ctx* p : m->parts)
        if (p->lv[l].sw_pairs.pairs != pairs) throw SmgError(SMG_EINVAL, "slab parts disagree on the merged Vanka pairs");
    for (int sweep = 0; sweep < m->prm.nu; ++sweep)
        for (int k = 0; k < 16; ++k) {
            const int j = k < 8 ? k : 15 - k;
            const int col = vanka_order(j);
            if ((j & 1) && ((pairs >> (7 - col)) & 1)) continue;  // folded into its partner's phase
            each(m, [&](smg_ctx* p) {
                DevLevel& L = p->lv[l];
                launch_vanka_delta(L.k, L.x, L.b, L.sw_cells[col], L.sw_mask[col], L.sw_n[col], L.ktab, p->vk_delta, p->st);
                launch_vanka_apply(L.k, L.x, L.sw_cells[col], L.sw_mask[col], L.sw_n[col], p->vk_delta, p->st,
                                   L.sw_amask[col]);
            });
            exchange_frame(m, l);
        }
}

// Tiled slab level, after a forward tile phase of colour T: a part's boundary tiles of that
// colour have updated the pressures (and, at the top, the w faces) of the neighbour's first
// plane, which the part holds as a ghost plane.  Exactly one side of every slab boundary ran
// (the two boundary tile layers differ in z parity), and its ghost plane was current before
// the phase, so that side pushes the whole plane to the owner: up (P and W of ghost plane nz
// -> the upper part's plane 0) when the lower part's top tile layer has T's z parity, else
// down (P of ghost plane -1 -> the lower part's plane nz - 1).
void push_ghosts(smg_ctx* m, int l, int T) {
    const Geom& g0 = m->lv[l].k.g;
    const int tz = dgs_tile_dim(2);
    // z parity of the top tile layer of part r: ((z0 + nzl) / tz - 1) & 1, z0 = r nzl
    auto top_ran = [&](int r) { return ((((r + 1) * g0.nz) / tz - 1) & 1) == ((T >> 2) & 1); };
    if (m->mp) {
        const NcclApi& N = nccl();
        const Geom& g = g0;
        cudaStream_t ts = tstream(m, m);
        ncclComm_t cm = tcomm(m);
        double* X = m->lv[l].x;
        const size_t n1 = static_cast<size_t>(g.sz);
        NK(N.groupStart());
        const int r = m->rank;
        if (r + 1 < m->nparts) {  // boundary with the upper part
            if (top_ran(r)) {
                for (int f : {2, 3}) NK(N.send(X + f * g.fs + (g.zg + g.nz) * g.sz, n1, ncclDouble, r + 1, cm, ts));
            } else {
                NK(N.recv(X + 3 * g.fs + (g.zg + g.nz - 1) * g.sz, n1, ncclDouble, r + 1, cm, ts));
            }
        }
        if (r > 0) {  // boundary with the lower part
            if (top_ran(r - 1)) {
                for (int f : {2, 3}) NK(N.recv(X + f * g.fs + g.zg * g.sz, n1, ncclDouble, r - 1, cm, ts));
            } else {
                NK(N.send(X + 3 * g.fs + (g.zg - 1) * g.sz, n1, ncclDouble, r - 1, cm, ts));
            }
        }
        NK(N.groupEnd());
        return;
    }
    part_barrier(m);
    for (size_t p = 0; p + 1 < m->parts.size(); ++p) {
        DevLevel &lo = m->parts[p]->lv[l], &hi = m->parts[p + 1]->lv[l];
        const Geom& g = lo.k.g;
        const size_t pitch = g.fs * sizeof(double), width = g.sz * sizeof(double);
        if (top_ran(static_cast<int>(p))) {  // W, P of lo's ghost plane nz -> hi's plane 0
            CK(cudaMemcpy2DAsync(hi.x + 2 * g.fs + g.zg * g.sz, pitch, lo.x + 2 * g.fs + (g.zg + g.nz) * g.sz, pitch,
                                 width, 2, cudaMemcpyDefault, tstream(m, m->parts[p + 1])));
        } else {  // P of hi's ghost plane -1 -> lo's plane nz - 1
            CK(cudaMemcpyAsync(lo.x + 3 * g.fs + (g.zg + g.nz - 1) * g.sz, hi.x + 3 * g.fs + (g.zg - 1) * g.sz,
                               width, cudaMemcpyDefault, tstream(m, m->parts[p])));
        }
    }
    part_barrier(m);
}

void dist_dgs_sym(smg_ctx* m, int l) {
    const int nph = (m->prm.flags & SMG_FLAG_SKIP_REVERSE_DGS) ? 10 : 20;
    each(m, [&](smg_ctx* p) { launch_dgs_cb(p->lv[l].k, p->lv[l].b, p->st); });  // b halos are valid here
    if (m->lv[l].k.tiled) {  // tile order (OD-1 rev. 2): one launch + one exchange per tile colour
        // Overlap (SMG_DIST_OVERLAP, default on): the part's bottom and top tile layers first; their
        // updates are all a halo transfer reads (owned planes 0, 1, nz - 2, nz - 1 and, for the push,
        // the adjacent ghost plane), and what it writes (ghost planes, the pushed plane 0 / nz - 1) is
        // out of reach of the layers in between (a tile reads at most 2 planes beyond its own 8).  So
        // the transfer runs on the comm stream while the interior layers run on the compute stream;
        // the next phase waits for both.  Same tiles, same arithmetic: bit-identical.
        const bool overlap = !(std::getenv("SMG_DIST_OVERLAP") && std::atoi(std::getenv("SMG_DIST_OVERLAP")) == 0);  // read per sweep (tests)
        const bool ov = overlap && m->lv[l].k.g.nz / dgs_tile_dim(2) >= 3;
        if (ov) ensure_comm_streams(m);
        auto phase = [&](int T, int ph0, int ph1) {
            if (!ov) {
                each(m, [&](smg_ctx* p) { launch_dgs_tile_phases(p->lv[l].k, p->lv[l].x, p->lv[l].b, T, ph0, ph1, p->st, 0, true); });
                if (ph0 < 10) push_ghosts(m, l, T);
                exchange(m, l, sel_x, 4);
                return;
            }
            each(m, [&](smg_ctx* p) {
                launch_dgs_tile_phases(p->lv[l].k, p->lv[l].x, p->lv[l].b, T, ph0, ph1, p->st, 1, true);
                CK(cudaEventRecord(p->evb, p->st));
                CK(cudaStreamWaitEvent(p->cst, p->evb, 0));
            });
            m->on_cst = true;
            try {
                if (ph0 < 10) push_ghosts(m, l, T);
                exchange(m, l, sel_x, 4);
            } catch (...) {
                m->on_cst = false;
                throw;
            }
            m->on_cst = false;
            each(m, [&](smg_ctx* p) {
                CK(cudaEventRecord(p->evc, p->cst));
                launch_dgs_tile_phases(p->lv[l].k, p->lv[l].x, p->lv[l].b, T, ph0, ph1, p->st, 2, true);
                CK(cudaStreamWaitEvent(p->st, p->evc, 0));
            });
        };
        for (int T = 0; T < 8; ++T) phase(T, 0, (T == 7 && nph > 10) ? 20 : 10);
        if (nph > 10)
            for (int T = 6; T >= 0; --T) phase(T, 10, 20);
        return;
    }
    for (int ph = 0; ph < nph; ++ph) {
        int f0 = 0, nf = 4;  // fields the phase changed: velocity phases u, v, w; reverse pressure phases p
        if (ph == 0 || ph == 1 || ph == 18 || ph == 19) {
            const int col = ph < 2 ? ph : 19 - ph;
            each(m, [&](smg_ctx* p) { launch_dgs_vel_c(p->lv[l].k, p->lv[l].x, p->lv[l].b, col, p->st); });
            nf = 3;
        } else if (ph <= 9) {
            const int c = ph - 2;
            Sel sd = (c & 1) ? sel_d1 : sel_d0;
            each(m, [&](smg_ctx* p) {
                DevLevel& L = p->lv[l];
                launch_dgs_pf_delta_c(L.k, L.x, L.b, sd(L), c, p->st);
            });
            exchange(m, l, sd, 1);
            each(m, [&](smg_ctx* p) { launch_dgs_pf_apply_c(p->lv[l].k, p->lv[l].x, sd(p->lv[l]), c, p->st); });
        } else {
            each(m, [&](smg_ctx* p) { launch_dgs_prev_c(p->lv[l].k, p->lv[l].x, p->lv[l].b, 17 - ph, p->st); });
            f0 = 3;
            nf = 1;
        }
        exchange(m, l, sel_x, nf, f0);
    }
}

void dist_smooth(smg_ctx* m, int l) {
    Nvtx r("dist_smooth", l);
    dist_vanka_sym(m, l);
    dist_dgs_sym(m, l);
    dist_vanka_sym(m, l);
}

// V-cycle on the parts; level-l b must hold valid halos
void dist_vcycle(smg_ctx* m, int l) {
    Nvtx r("dist_vcycle", l);
    if (l >= m->ndist) {  // replicated: every part runs the identical single-part cycle
        each(m, [&](smg_ctx* p) { vcycle(p, l, p->lv[l].b, p->lv[l].x); });
        return;
    }
    each(m, [&](smg_ctx* p) { CK(cudaMemsetAsync(p->lv[l].x, 0, vlen(p->lv[l]) * sizeof(double), p->st)); });
    dist_smooth(m, l);
    each(m, [&](smg_ctx* p) {
        DevLevel& L = p->lv[l];
        launch_apply(L.k, L.x, L.b, L.r, L.k.gamma, p->st);
    });
    exchange(m, l, sel_r, 4);
    const bool cdist = l + 1 < m->ndist;
    each(m, [&](smg_ctx* p) {
        DevLevel &L = p->lv[l], &C = p->lv[l + 1];
        if (cdist) launch_restrict(L.k, C.k, L.r, C.b, p->st);
        else launch_restrict(L.k, C.k, L.r, C.b, p->st, L.k.g.z0 / 2, L.k.g.nz / 2);
    });
    if (cdist) exchange(m, l + 1, sel_b, 4);
    else allgather_planes(m, l + 1, sel_b, m->lv[l].k.g.nz / 2);
    dist_vcycle(m, l + 1);
    if (cdist) exchange(m, l + 1, sel_x, 4);
    // W-cycle: second recursive call below the finest level on the residual of the
    // first, as in the single-part vcycle (skipped when the child is the exact coarsest solve)
    if (m->prm.cycle == 1 && l >= 1 && l + 2 < static_cast<int>(m->lv.size())) {
        each(m, [&](smg_ctx* p) {
            DevLevel& C = p->lv[l + 1];
            launch_apply(C.k, C.x, C.b, C.wb, C.k.gamma, p->st);
            std::swap(C.b, C.wb);  // the recursion reads lv[l+1].b and writes lv[l+1].x
            std::swap(C.x, C.wx);
        });
        if (cdist) exchange(m, l + 1, sel_b, 4);
        dist_vcycle(m, l + 1);
        if (cdist) exchange(m, l + 1, sel_x, 4);
        each(m, [&](smg_ctx* p) {
            DevLevel& C = p->lv[l + 1];
            std::swap(C.b, C.wb);
            std::swap(C.x, C.wx);
            launch_axpy(C.x, C.wx, 1.0, vlen(C), p->st);
        });
    }
    each(m, [&](smg_ctx* p) { launch_prolong_add(p->lv[l].k, p->lv[l + 1].k, p->lv[l + 1].x, p->lv[l].x, p->st); });
    exchange(m, l, sel_x, 4);
    dist_smooth(m, l);
}

double* v_q(smg_ctx* p) { return p->q; }
double* v_xs(smg_ctx* p) { return p->xcur ? p->xs2 : p->xs; }
double* v_rhs(smg_ctx* p) { return p->rhs; }
double* v_s(smg_ctx* p) { return p->lv[0].b; }
double* v_t(smg_ctx* p) { return p->lv[0].x; }
double* v_r(smg_ctx* p) { return p->lv[0].r; }

// exchange of a fine-level SQMR vector (not a DevLevel member)
void exchange_vec(smg_ctx* m, double* (*v)(smg_ctx*)) {
    if (m->mp) {
        halo_nccl(m, v(m), m->lv[0].k.g, 4);
        return;
    }
    part_barrier(m);
    for (size_t p = 0; p + 1 < m->parts.size(); ++p) {
        smg_ctx *lo = m->parts[p], *hi = m->parts[p + 1];
        const Geom& g = lo->lv[0].k.g;
        const size_t pitch = g.fs * sizeof(double), width = 2 * g.sz * sizeof(double);
        CK(cudaMemcpy2DAsync(v(lo) + (g.nz + g.zg) * g.sz, pitch, v(hi) + g.zg * g.sz, pitch, width, 4,
                             cudaMemcpyDefault, lo->st));
        CK(cudaMemcpy2DAsync(v(hi), pitch, v(lo) + g.nz * g.sz, pitch, width, 4, cudaMemcpyDefault, hi->st));
    }
    part_barrier(m);
}

void dist_upload(smg_ctx* m, const double* host, double* (*v)(smg_ctx*)) {
    const int64_t n = m->lv[0].N;
    each(m, [&](smg_ctx* p) {
        CK(cudaMemcpyAsync(p->compact, host, n * sizeof(double), cudaMemcpyHostToDevice, p->st));
        launch_unpack(p->lv[0].k, p->compact, v(p), p->st);
    });
    exchange_vec(m, v);
}

void dist_download(smg_ctx* m, double* (*v)(smg_ctx*), double* host) {
    const DevLevel& L0 = m->lv[0];
    const int nx = m->grid.nx, ny = m->grid.ny, gnz = m->grid.nz;
    const int64_t nu = L0.counts[0], nv = L0.counts[1], nw = L0.counts[2];
    // compact ranges of the planes [z0, z1): u, v, w (faces z >= 1), p
    auto ranges = [&](int z0, int z1, int64_t r[4][2]) {
        const int64_t q[4][2] = {
            {static_cast<int64_t>(z0) * ny * (nx - 1), static_cast<int64_t>(z1) * ny * (nx - 1)},
            {nu + static_cast<int64_t>(z0) * (ny - 1) * nx, nu + static_cast<int64_t>(z1) * (ny - 1) * nx},
            {nu + nv + static_cast<int64_t>(std::max(z0, 1) - 1) * ny * nx,
             nu + nv + static_cast<int64_t>(std::min(z1, gnz) - 1) * ny * nx},
            {nu + nv + nw + static_cast<int64_t>(z0) * ny * nx, nu + nv + nw + static_cast<int64_t>(z1) * ny * nx}};
        std::memcpy(r, q, sizeof(q));
    };
    if (m->mp) {  // every rank's ranges broadcast from their owner, then the whole vector to the host
        launch_pack(m->lv[0].k, v(m), m->compact, m->st);
        const NcclApi& N = nccl();
        const int nzl = m->lv[0].k.g.nz;
        NK(N.groupStart());
        for (int r = 0; r < m->nparts; ++r) {
            int64_t rg[4][2];
            ranges(r * nzl, (r + 1) * nzl, rg);
            for (auto& q : rg)
                if (q[1] > q[0])
                    NK(N.broadcast(m->compact + q[0], m->compact + q[0], static_cast<size_t>(q[1] - q[0]), ncclDouble,
                                   r, m->comm, m->st));
        }
        NK(N.groupEnd());
        CK(cudaMemcpyAsync(host, m->compact, L0.N * sizeof(double), cudaMemcpyDeviceToHost, m->st));
        CK(cudaStreamSynchronize(m->st));
        return;
    }
    each(m, [&](smg_ctx* p) {
        launch_pack(p->lv[0].k, v(p), p->compact, p->st);
        const int z0 = p->lv[0].k.g.z0, z1 = z0 + p->lv[0].k.g.nz;
        int64_t r[4][2];
        ranges(z0, z1, r);
        for (auto& rg : r)
            if (rg[1] > rg[0])
                CK(cudaMemcpyAsync(host + rg[0], p->compact + rg[0], (rg[1] - rg[0]) * sizeof(double),
                                   cudaMemcpyDeviceToHost, p->st));
    });
    each(m, [&](smg_ctx* p) { CK(cudaStreamSynchronize(p->st)); });
}

// ======================================================= SQMR, Alg. 4 ====
// One code path for a single part and for the z-slab parts (m = the master context).  Per
// iteration (lines 5-10), with the north_star's fusion of the AXPYs into the inner products:
//   k_axpy_s    s = s - alpha t'
//   V-cycle     t = V(s)
//   k_cdot      partials of ||t||^2 and rho = s.t                      -> final: nu, c, tau, beta
//   k_apply_x   d = cd d + cq q, x = x + d, partials of ||b - L x||^2   (first slot)
//   k_apply_q   q = t + beta q, t' = L q, partials of sigma = q.t'      (second slot; iteration j + 1's)
//                                                                       -> final: rel, rho commit, alpha
// i.e. two reductions per iteration (SURVEY OD-11; slab contexts); the setup runs the first q step on
// its own.  A single part runs k_apply_q first with its own final (three finals, no wasted q step).
// Every scalar lives on the device; a single part replays the iteration as a CUDA graph (one
// per parity of the q / d / x ping-pong) and reads back (rel, status) once per iteration.
// Slab parts: block partials at global block indices are combined by a shared buffer (parts of
// one process) or one NCCL all-reduce (one process per GPU); every part runs the same final,
// so all parts hold identical scalars.  The fused kernels also write q, d and x on the ghost
// planes, so only s needs a halo exchange.

// where a part's block partials go
double* part_out(smg_ctx* m, smg_ctx* p) { return (m->ndist > 0 && !m->mp) ? m->shared_partials : p->partials; }

// combine the block partials of all parts, then the final + scalar update `which` on every part
void finalize(smg_ctx* m, int which) {
    const Geom& g = m->lv[0].k.g;
    if (m->ndist == 0) {
        launch_final_scalar(g, m->partials, m->dscal, which, m->st);
        return;
    }
    if (m->mp) {  // own blocks' partials (zeros elsewhere) summed over ranks: x + 0 = x exactly
        NK(nccl().allReduce(m->partials, m->shared_partials, dot_partials(g), ncclDouble, ncclSum, m->comm, m->st));
        launch_final_scalar(g, m->shared_partials, m->dscal, which, m->st);
        return;
    }
    part_barrier(m);
    each(m, [&](smg_ctx* p) { launch_final_scalar(p->lv[0].k.g, m->shared_partials, p->dscal, which, p->st); });
}

// block partials of a.b (and c.d) on every part
void dots(smg_ctx* m, double* (*a)(smg_ctx*), double* (*b)(smg_ctx*), double* (*c2)(smg_ctx*),
          double* (*d)(smg_ctx*)) {
    each(m, [&](smg_ctx* p) {
        launch_cdot_planes(p->lv[0].k.g, a(p), b(p), c2 ? c2(p) : nullptr, d ? d(p) : nullptr, part_out(m, p), p->st);
    });
}

void pc_vcycle(smg_ctx* m) {  // t = V(s) on the fine level
    if (m->prm.flags & SMG_FLAG_NO_PRECOND) {  // method `sqmr`: identity preconditioner
        each(m, [&](smg_ctx* p) {
            CK(cudaMemcpyAsync(v_t(p), v_s(p), vlen(p->lv[0]) * sizeof(double), cudaMemcpyDeviceToDevice, p->st));
        });
        return;
    }
    if (m->ndist > 0) dist_vcycle(m, 0);
    else vcycle(m, 0, m->lv[0].b, m->lv[0].x);
}

// lines 9 + 5 of iteration `par`: q = t + beta q, t' = L q (into lv[0].r), partials of sigma = q.t' --
// in the first slot (second = 0: the setup's own reduction) or in the second slot next to the
// residual partials of the iteration that just ended
void sqmr_q_step(smg_ctx* m, int par, int second) {
    each(m, [&](smg_ctx* p) {
        DevLevel& F = p->lv[0];
        const int lo = m->ndist > 0 && p->rank > 0, hi = m->ndist > 0 && p->rank + 1 < p->nparts;
        launch_apply_q(F.k, F.x, par ? p->q2 : p->q, par ? p->q : p->q2, F.r, p->dscal, part_out(m, p), lo, hi, p->st,
                       second);
    });
}

// Iteration j (par = (j - 1) & 1) from "alpha_j known, t' = L q_j in lv[0].r": the update of s, the
// V-cycle, {||t||^2, rho} (reduction 1), the d / x update with the true residual, and already the q
// step of iteration j + 1, whose sigma shares reduction 2 with ||r_j||^2 (SURVEY OD-11: the exact
// Alg. 4 with two reductions per iteration; same arithmetic as the three-reduction order, only the
// kernel that forms L q_{j+1} runs before the convergence test of iteration j instead of after it).
// A single part has no all-reduce to save and would only pay the q step wasted after the converged
// iteration (0.5% of a cfg-2 solve), so it keeps the order of Alg. 4 with three finals; slab
// contexts take the two-reduction order.  Both give the same bits.
bool two_reductions(const smg_ctx* m) { return m->ndist > 0; }

void sqmr_iteration(smg_ctx* m, int par) {
    Nvtx r("sqmr_iteration");
    if (!two_reductions(m)) {
        sqmr_q_step(m, par, /*second=*/0);  // lines 9 + 5: q, t' = L q, sigma
        finalize(m, 1);                     // alpha
    }
    each(m, [&](smg_ctx* p) { launch_axpy_s(p->lv[0].b, p->lv[0].r, p->dscal, vlen(p->lv[0]), p->st); });
    if (m->ndist > 0) exchange_vec(m, v_s);
    pc_vcycle(m);                   // line 6: t = V(s)
    dots(m, v_t, v_t, v_s, v_t);    // ||t||^2, rho_j
    finalize(m, 2);                 // nu, c, tau, cd, cq, beta_j
    each(m, [&](smg_ctx* p) {       // lines 7 + 8: d, x and the true residual
        DevLevel& F = p->lv[0];
        const int lo = m->ndist > 0 && p->rank > 0, hi = m->ndist > 0 && p->rank + 1 < p->nparts;
        launch_apply_x(F.k, par ? p->xs2 : p->xs, par ? p->d2 : p->d, par ? p->q : p->q2, p->rhs, par ? p->xs : p->xs2,
                       par ? p->d : p->d2, p->dscal, part_out(m, p), lo, hi, p->st);
    });
    if (!two_reductions(m)) {
        finalize(m, 3);             // rel, convergence, beta
        return;
    }
    sqmr_q_step(m, par ^ 1, /*second=*/1);
    finalize(m, 4);                 // rel_j, convergence, rho commit; alpha_{j+1} (sigma breakdown: status 2)
}

int sqmr(smg_ctx* m, double tol, int maxit, smg_history* hist, int* status) {
    Nvtx r("sqmr_solve");
    auto t0 = std::chrono::steady_clock::now();
    const int64_t l0 = launch_count();
    int64_t graph_launches = 0;
    // The iteration replays as a CUDA graph for a single part and for one-process-per-GPU slab
    // ranks (NCCL send/recv, all-reduce and all-gather are captured with the kernels on the rank's
    // one stream: no host launch latency between the ~10^3 phase kernels and halo groups of a
    // V-cycle; SMG_DIST_GRAPH=0 keeps eager launches).  In-process parts on several streams stay eager.
    static const bool dist_graph = !(std::getenv("SMG_DIST_GRAPH") && std::atoi(std::getenv("SMG_DIST_GRAPH")) == 0);
    // SMG_EMU_GRAPH=1 (measurement aid, tools/time_slabs.py): in-process parts that share ONE stream (all
    // parts emulated on one device) also replay the iteration as a graph -- kernels of every part and the
    // device-local halo copies as nodes -- which takes the host launch cost out of the emulation and leaves
    // what the slab decomposition itself costs on the GPU (smaller kernels, halo copies, extra phases).
    static const bool emu_graph = std::getenv("SMG_EMU_GRAPH") && std::atoi(std::getenv("SMG_EMU_GRAPH")) != 0;
    const bool single = m->ndist == 0 || (m->mp && dist_graph) || (!m->mp && emu_graph && shared_stream(m));
    CK(cudaEventRecord(m->ev0, m->st));
    if (hist) hist->count = 0;
    each(m, [&](smg_ctx* p) {
        const int64_t n = vlen(p->lv[0]);
        CK(cudaMemsetAsync(p->xs, 0, n * sizeof(double), p->st));
        CK(cudaMemsetAsync(p->d, 0, n * sizeof(double), p->st));
        CK(cudaMemsetAsync(p->dscal, 0, S_COUNT * sizeof(double), p->st));
        p->xcur = 0;
    });
    dots(m, v_rhs, v_rhs, nullptr, nullptr);
    finalize(m, -1);
    CK(cudaMemcpyAsync(m->hscal, m->dscal + S_D0, sizeof(double), cudaMemcpyDeviceToHost, m->st));
    each(m, [&](smg_ctx* p) { CK(cudaStreamSynchronize(p->st)); });
    const double bnorm = std::sqrt(m->hscal[0]);
    int st = SMG_MAX_ITERATIONS, iters = 0;
    if (bnorm == 0.0) {
        st = SMG_CONVERGED;
    } else {
        m->hscal[2] = bnorm;
        m->hscal[3] = tol;
        each(m, [&](smg_ctx* p) {  // lines 1-4: s = b, t = V(s), q = t, tau, rho
            CK(cudaMemcpyAsync(p->dscal + S_BNORM, &m->hscal[2], sizeof(double), cudaMemcpyHostToDevice, p->st));
            CK(cudaMemcpyAsync(p->dscal + S_TOL, &m->hscal[3], sizeof(double), cudaMemcpyHostToDevice, p->st));
            CK(cudaMemcpyAsync(v_s(p), p->rhs, vlen(p->lv[0]) * sizeof(double), cudaMemcpyDeviceToDevice, p->st));
        });
        if (m->ndist > 0) exchange_vec(m, v_s);
        pc_vcycle(m);
        each(m, [&](smg_ctx* p) {
            CK(cudaMemcpyAsync(p->q, v_t(p), vlen(p->lv[0]) * sizeof(double), cudaMemcpyDeviceToDevice, p->st));
        });
        dots(m, v_t, v_t, v_s, v_q);
        finalize(m, 0);
        if (two_reductions(m)) {
            sqmr_q_step(m, 0, /*second=*/0);  // iteration 1's q step (beta = 0: q_1 = t), sigma_1 -> alpha_1
            finalize(m, 1);
        }
        CK(cudaMemcpyAsync(m->hscal, m->dscal + S_STATUS, sizeof(double), cudaMemcpyDeviceToHost, m->st));
        each(m, [&](smg_ctx* p) { CK(cudaStreamSynchronize(p->st)); });
        if (m->hscal[0] != 0.0) st = SMG_BREAKDOWN;
        if (single && st == SMG_MAX_ITERATIONS && maxit > 0 && !m->graph) {
            for (int par = 0; par < 2; ++par) {
                const int64_t before = launch_count();
                CK(cudaStreamBeginCapture(m->st, cudaStreamCaptureModeRelaxed));
                sqmr_iteration(m, par);
                cudaGraph_t gr = nullptr;
                CK(cudaStreamEndCapture(m->st, &gr));
                CK(cudaGraphInstantiate(par ? &m->graph2 : &m->graph, gr, 0));
                CK(cudaGraphDestroy(gr));
                m->graph_kernels = launch_count() - before;
                graph_launches -= m->graph_kernels;  // capture-time launches are not executions
            }
        }
        for (int j = 1; j <= maxit && st == SMG_MAX_ITERATIONS; ++j) {
            const int par = (j - 1) & 1;
            Nvtx rj("sqmr_iter", j);
            if (single) {
                CK(cudaGraphLaunch(par ? m->graph2 : m->graph, m->st));
                graph_launches += m->graph_kernels;
            } else {
                sqmr_iteration(m, par);
            }
            if (const int e = take_launch_error())
                throw SmgError(SMG_ECUDA, std::string("kernel launch rejected: ") +
                                              cudaGetErrorString(static_cast<cudaError_t>(e)));
            CK(cudaMemcpyAsync(m->hscal, m->dscal + S_REL, 2 * sizeof(double), cudaMemcpyDeviceToHost, m->st));
            each(m, [&](smg_ctx* p) { CK(cudaStreamSynchronize(p->st)); });
            const double rel = m->hscal[0];
            const int code = static_cast<int>(m->hscal[1]);
            // three-final order: the sigma breakdown belongs to this iteration, which has no residual
            if (code == 2 && !two_reductions(m)) { st = SMG_BREAKDOWN; break; }
            iters = j;
            if (hist && hist->count < hist->capacity) {
                hist->rel_residual[hist->count] = rel;
                hist->seconds[hist->count] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                hist->count++;
            }
            if (code == 1) st = SMG_CONVERGED;
            else if (code == 3) st = SMG_BREAKDOWN;
            else if (code == 2 && j < maxit) st = SMG_BREAKDOWN;  // sigma of iteration j + 1 (which maxit allows) broke down
        }
    }
    each(m, [&](smg_ctx* p) { p->xcur = iters & 1; });  // iteration j wrote buffer [j & 1]
    CK(cudaEventRecord(m->ev1, m->st));
    CK(cudaEventSynchronize(m->ev1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, m->ev0, m->ev1));
    m->timing.solve_ms = ms;
    m->timing.iterations = iters;
    m->timing.kernel_launches = (launch_count() - l0) + graph_launches;
    *status = st;
    return 0;
}

template <class F>
int guard(smg_ctx* c, F&& f) {
    try {
        f();
        if (const int e = take_launch_error())
            throw SmgError(SMG_ECUDA, std::string("kernel launch rejected: ") +
                                          cudaGetErrorString(static_cast<cudaError_t>(e)));
        return 0;
    } catch (const SmgError& e) {
        if (c) c->err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        if (c) c->err = e.what();
        return SMG_EINVAL;
    }
}

void check_level(smg_ctx* c, int l) {
    if (l < 0 || l >= static_cast<int>(c->lv.size())) throw SmgError(SMG_EINVAL, "level out of range");
}

}  // namespace

// ================================================================ C ABI =====
extern "C" {

const char* smg_version(void) { return "smg-b200 0.1 (sm_100a, fp64)"; }

int smg_assemble_rhs(const smg_grid_desc* grid, double eta, int scenario, double value, double* b) {
    // Dirichlet data folded into the right-hand side: scenario 0 = lid-driven
    // cavity, u = value on the ring faces above the top (y = ny): each u-face of the top
    // interior row gets +eta/h^2 * value (its stencil leg to the lid).  Continuity rows see
    // only the no-penetration (zero) normal velocity.
    if (!grid || !b || grid->dim != 3 || scenario != 0 || !(grid->h > 0)) return SMG_EINVAL;
    const int nx = grid->nx, ny = grid->ny, nz = grid->nz;
    const double eta_h2 = eta / (grid->h * grid->h);
    if (value == 0.0) return 0;
    for (int z = 0; z < nz; ++z)
        for (int x = 1; x <= nx - 1; ++x) {
            const int64_t id = (static_cast<int64_t>(z) * ny + (ny - 1)) * (nx - 1) + (x - 1);
            b[id] = b[id] + eta_h2 * value;
        }
    return 0;
}

int64_t smg_census(const smg_grid_desc* grid, int band_width, int64_t* out2) {
    if (!grid || grid->dim != 3 || band_width < 1 || grid->nx < 1 || grid->ny < 1 || grid->nz < 1) return SMG_EINVAL;
    const int nx = grid->nx, ny = grid->ny, nz = grid->nz, bw = band_width;
    auto band = [&](int x, int y, int z) {
        return x < bw || y < bw || z < bw || x >= nx - bw || y >= ny - bw || z >= nz - bw;
    };
    int64_t n = 0, v1 = 0;
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x) {
                const bool bc = band(x, y, z);
                const int nf = (x >= 1) + (y >= 1) + (z >= 1);
                n += nf + 1;
                if (x >= 1 && (bc || band(x - 1, y, z))) ++v1;
                if (y >= 1 && (bc || band(x, y - 1, z))) ++v1;
                if (z >= 1 && (bc || band(x, y, z - 1))) ++v1;
                if (bc) ++v1;
            }
    if (out2) {
        out2[0] = n;
        out2[1] = v1;
    }
    return n;
}

// leading levels that split into nparts z-slabs (slab >= 2 planes, aligned with the finer level;
// on DGS-tiled levels a whole number of tiles, so every tile lies in one part)
static int slab_levels(const smg_grid_desc* grid, int levels, int nparts, int64_t tile_min) {
    int nd = 0;
    // Levels below 64^3 cells are gathered (BASELINE cfg 3 "coarse levels gathered below 64^3"):
    // a distributed level visit costs ~90 halo messages whatever its size, a replicated 32^3 sub-cycle
    // ~0.45 ms of redundant compute.  SMG_SLAB_MIN_CELLS overrides the bound (0: split whatever can be
    // split -- the tests, which exercise the machinery on small grids); level 0 is always split.
    const char* mc = std::getenv("SMG_SLAB_MIN_CELLS");
    const int64_t min_cells = mc ? std::atoll(mc) : int64_t{64} * 64 * 64;
    for (int l = 0; l + 1 < levels; ++l) {
        const int nz = grid->nz >> l;
        if (l >= 1 && static_cast<int64_t>(grid->nx >> l) * (grid->ny >> l) * nz < min_cells) break;
        if (dgs_tiled(grid->nx >> l, grid->ny >> l, nz, tile_min) && (nz % nparts || (nz / nparts) % dgs_tile_dim(2)))
            break;
        // slab of >= 2 planes (halo depth), and even: the child level's planes 2k, 2k+1 then
        // always sit in one slab, so restriction into a slab (or into the replicated first
        // level, coarse planes z0/2 .. (z0 + nzl)/2) covers every coarse plane
        if (nz % nparts || nz / nparts < 2 || (nz / nparts) % 2) break;
        if (l == 0 && (nz / nparts) % kDotZBlock) break;  // inner-product blocks never straddle parts
        nd = l + 1;
    }
    return nd;
}

static int slab_plan_t(const smg_grid_desc* grid, int levels, int nparts, int rank, int* z0, int* nzl,
                       int64_t tile_min) {
    if (!grid || levels < 1 || nparts < 1 || rank < 0 || rank >= nparts) return SMG_EINVAL;
    const int nd = nparts > 1 ? slab_levels(grid, levels, nparts, tile_min) : 0;
    for (int l = 0; l < levels; ++l) {
        const int nz = grid->nz >> l;
        const bool d = l < nd;
        if (z0) z0[l] = d ? rank * (nz / nparts) : 0;
        if (nzl) nzl[l] = d ? nz / nparts : nz;
    }
    return nd;
}
int smg_slab_plan(const smg_grid_desc* grid, int levels, int nparts, int rank, int* z0, int* nzl) {
    return slab_plan_t(grid, levels, nparts, rank, z0, nzl, 0);
}
int smg_dgs_tile(const smg_grid_desc* grid, int level, int64_t tile_min, int* out4) {
    if (!grid || !out4 || level < 0 || level > 20) return SMG_EINVAL;
    const bool t = dgs_tiled(grid->nx >> level, grid->ny >> level, grid->nz >> level, tile_min);
    out4[0] = t ? 8 : 1;
    for (int a = 0; a < 3; ++a) out4[1 + a] = t ? dgs_tile_dim(a) : 0;
    return 0;
}

int smg_create(const smg_grid_desc* grid, const smg_params* params, int ngpu, const int* dev_ids, smg_ctx** out) {
    if (!grid || !params || !out) return SMG_EINVAL;
    *out = nullptr;
    if (ngpu < 1 || ngpu > 64) return SMG_EINVAL;
    auto c = std::make_unique<smg_ctx>();
    c->grid = *grid;
    c->prm = *params;
    c->device = dev_ids ? dev_ids[0] : 0;
    c->nparts = ngpu;
    c->parts.push_back(c.get());
    const int rc = guard(c.get(), [&] {
        if (ngpu > 1) {
            // levels split into z-slabs: slab >= 2 planes, aligned with the next level
            const int nd = slab_plan_t(grid, params->levels, ngpu, 0, nullptr, nullptr, params->dgs_tile_min);
            if (nd <= 0) throw SmgError(SMG_EINVAL, "grid too small for a z-slab split over ngpu parts");
            c->ndist = nd;
        }
        std::vector<double> coarse;
        build(c.get(), nullptr, &coarse);
        for (int r = 1; r < ngpu; ++r) {
            auto q = std::make_unique<smg_ctx>();
            q->grid = *grid;
            q->prm = *params;
            q->device = dev_ids ? dev_ids[r] : c->device;
            q->rank = r;
            q->nparts = ngpu;
            q->ndist = c->ndist;
            build(q.get(), &coarse, nullptr, q->device == c->device ? c->st : nullptr);
            if (q->device != c->device) {
                int ok = 0;
                CK(cudaDeviceCanAccessPeer(&ok, q->device, c->device));
                if (ok) {
                    CK(cudaSetDevice(q->device));
                    cudaDeviceEnablePeerAccess(c->device, 0);
                    CK(cudaSetDevice(c->device));
                    cudaDeviceEnablePeerAccess(q->device, 0);
                    cudaGetLastError();  // tolerate "already enabled"
                }
            }
            c->parts.push_back(q.get());
            c->owned.push_back(std::move(q));
        }
        CK(cudaSetDevice(c->device));
        if (ngpu > 1) c->shared_partials = c->dalloc<double>(dot_partials(c->lv[0].k.g));
    });
    if (rc != 0) {
        std::fprintf(stderr, "smg_create: %s\n", c->err.c_str());
        return rc;
    }
    *out = c.release();
    return 0;
}

int smg_create_labeled(const smg_grid_desc* grid, const uint8_t* labels, const smg_params* params, int device,
                       smg_ctx** out) {
    if (!grid || !labels || !params || !out) return SMG_EINVAL;
    *out = nullptr;
    if (grid->dim != 3 || grid->nx < 1 || grid->ny < 1 || grid->nz < 1) return SMG_EINVAL;
    auto c = std::make_unique<smg_ctx>();
    c->grid = *grid;
    c->prm = *params;
    c->device = device;
    c->parts.push_back(c.get());
    const size_t nc = static_cast<size_t>(grid->nx) * grid->ny * grid->nz;
    c->labels.assign(labels, labels + nc);
    const int rc = guard(c.get(), [&] {
        bool any = false;
        for (uint8_t l : c->labels) {
            if (l > LAB_E) throw SmgError(SMG_EINVAL, "labels must be 0 (Dirichlet), 1 (Interior) or 2 (Exterior)");
            any |= l == LAB_I;
        }
        if (!any) throw SmgError(SMG_EINVAL, "no Interior cell: the grid has no active DOF (SPEC:52)");
        build(c.get());
        if (c->lv.back().N == 0) throw SmgError(SMG_EINVAL, "the coarsest level has no active DOF: use fewer levels");
    });
    if (rc != 0) {
        std::fprintf(stderr, "smg_create_labeled: %s\n", c->err.c_str());
        return rc;
    }
    *out = c.release();
    return 0;
}

int smg_coarsen_labels(const smg_grid_desc* grid, const uint8_t* labels, uint8_t* out) {
    if (!grid || !labels || !out || grid->dim != 3) return SMG_EINVAL;
    if (grid->nx < 2 || grid->ny < 2 || grid->nz < 2 || (grid->nx | grid->ny | grid->nz) & 1) return SMG_EINVAL;
    const size_t nc = static_cast<size_t>(grid->nx) * grid->ny * grid->nz;
    const std::vector<uint8_t> c = coarsen_labels(std::vector<uint8_t>(labels, labels + nc), grid->nx, grid->ny, grid->nz);
    std::memcpy(out, c.data(), c.size());
    return 0;
}

int64_t smg_census_labeled(const smg_grid_desc* grid, const uint8_t* labels, int band_width, int64_t* out6) {
    if (!grid || !labels || grid->dim != 3 || band_width < 1) return SMG_EINVAL;
    const size_t nc = static_cast<size_t>(grid->nx) * grid->ny * grid->nz;
    try {
        const auto m = classify_labeled(std::vector<uint8_t>(labels, labels + nc), grid->nx, grid->ny, grid->nz, band_width);
        if (out6) {
            out6[0] = m->N;
            out6[1] = m->v1;
            for (int k = 0; k < 4; ++k) out6[2 + k] = m->cnt[k];
        }
        return m->N;
    } catch (...) {
        return SMG_EINVAL;
    }
}

int smg_nccl_unique_id(unsigned char id[128]) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    if (!id) return SMG_EINVAL;
    try {
        ncclUniqueId u;
        NK(nccl().getUniqueId(&u));
        std::memcpy(id, &u, sizeof(u));
        return 0;
    } catch (const SmgError& e) {
        std::fprintf(stderr, "smg_nccl_unique_id: %s\n", e.what());
        return e.code;
    }
}

int smg_create_rank(const smg_grid_desc* grid, const smg_params* params, int rank, int nranks, int device,
                    const unsigned char id[128], smg_ctx** out) {
    if (!grid || !params || !out || !id || nranks < 1 || nranks > 1024 || rank < 0 || rank >= nranks)
        return SMG_EINVAL;
    *out = nullptr;
    auto c = std::make_unique<smg_ctx>();
    c->grid = *grid;
    c->prm = *params;
    c->device = device;
    c->rank = rank;
    c->nparts = nranks;
    c->mp = true;
    c->parts.push_back(c.get());
    const int rc = guard(c.get(), [&] {
        // SMG_FORCE_SLABS=1 with one rank: the slab path on one part (exercises the NCCL transport on one GPU)
        const bool force = nranks == 1 && std::getenv("SMG_FORCE_SLABS") && std::atoi(std::getenv("SMG_FORCE_SLABS"));
        if (nranks > 1 || force) {
            const int nd = slab_levels(grid, params->levels, nranks, params->dgs_tile_min);
            if (nd <= 0) throw SmgError(SMG_EINVAL, "grid too small for a z-slab split over nranks parts");
            c->ndist = nd;
        } else {
            c->nparts = 1;
            c->mp = false;  // one rank, no slabs: the single-part path
        }
        CK(cudaSetDevice(device));
        build(c.get());
        if (c->mp) {
            ncclUniqueId u;
            std::memcpy(&u, id, sizeof(u));
            NK(nccl().commInitRank(&c->comm, nranks, u, rank));
            c->shared_partials = c->dalloc<double>(dot_partials(c->lv[0].k.g));
            ensure_comm_streams(c.get());  // comm stream + halo communicator now, never inside a graph capture
        }
    });
    if (rc != 0) {
        std::fprintf(stderr, "smg_create_rank: %s\n", c->err.c_str());
        return rc;
    }
    *out = c.release();
    return 0;
}

void smg_destroy(smg_ctx* ctx) { delete ctx; }

const char* smg_last_error(const smg_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int smg_num_levels(const smg_ctx* ctx) { return ctx ? static_cast<int>(ctx->lv.size()) : 0; }

int64_t smg_level_ndof(const smg_ctx* ctx, int level, int64_t* out5) {
    if (!ctx || level < 0 || level >= static_cast<int>(ctx->lv.size())) return SMG_EINVAL;
    const DevLevel& L = ctx->lv[level];
    if (out5)
        for (int k = 0; k < 5; ++k) out5[k] = L.counts[k];
    return L.N;
}

int smg_apply(smg_ctx* c, int level, int penalized, const double* x, double* y) {
    return guard(c, [&] {
        check_level(c, level);
        if (c->ndist > 0) {
            if (level != 0) throw SmgError(SMG_EINVAL, "z-slab contexts: apply on level 0 only");
            dist_upload(c, x, v_t);
            each(c, [&](smg_ctx* p) {
                launch_apply(p->lv[0].k, v_t(p), nullptr, v_r(p), penalized ? p->lv[0].k.gamma : 0.0, p->st);
            });
            dist_download(c, v_r, y);
            return;
        }
        DevLevel& L = c->lv[level];
        upload(c, level, x, L.x);
        launch_apply(L.k, L.x, nullptr, L.r, penalized ? L.k.gamma : 0.0, c->st);
        download(c, level, L.r, y);
    });
}

int smg_residual(smg_ctx* c, int level, const double* x, const double* b, double* r) {
    return guard(c, [&] {
        if (c->ndist > 0) throw SmgError(SMG_EINVAL, "single-part entry point (use ngpu = 1)");
        check_level(c, level);
        DevLevel& L = c->lv[level];
        upload(c, level, x, L.x);
        upload(c, level, b, L.b);
        launch_apply(L.k, L.x, L.b, L.r, L.k.gamma, c->st);
        download(c, level, L.r, r);
    });
}

int smg_smoother(smg_ctx* c, int level, int op, int arg, double* x, const double* b) {
    return guard(c, [&] {
        if (c->ndist > 0) throw SmgError(SMG_EINVAL, "single-part entry point (use ngpu = 1)");
        check_level(c, level);
        DevLevel& L = c->lv[level];
        upload(c, level, x, L.x);
        upload(c, level, b, L.b);
        if (op == 0) dgs_phase(c, level, L.x, L.b, arg);
        else if (op == 1) symmetric_dgs(c, level, L.x, L.b);
        else if (op == 2) {
            if (arg < 0 || arg > 7) throw SmgError(SMG_EINVAL, "colour out of range");
            launch_vanka_delta(L.k, L.x, L.b, L.vk_cells[arg], L.vk_mask[arg], L.vk_n[arg], L.ktab, c->vk_delta, c->st,
                               L.vk_kidx[arg]);
            launch_vanka_apply(L.k, L.x, L.vk_cells[arg], L.vk_mask[arg], L.vk_n[arg], c->vk_delta, c->st);
        } else if (op == 3 && L.k.cls) {
            vanka_sym(c, level, L.x, L.b);
        } else if (op == 3) {
            launch_vanka_sym_coop(L.k, L.x, L.b, L.sw_cells, L.sw_mask, L.sw_n, L.ktab, c->vk_delta, 1, c->st,
                                  L.xb, L.vk_refresh, L.vk_nrefresh, L.sw_pairs);
        } else if (op == 5) {  // one additive Vanka application
            vanka_additive(c, level, L.x, L.b);
        } else if (op == 7) {  // one direct-on-V1 solve
            vanka_direct(c, level, L.x, L.b);
        } else if (op == 6) {  // per-phase reference path of the symmetric sweeps (test only)
            if (L.k.tiled) {
                for (int T = 0; T < 8; ++T)
                    for (int ph = 0; ph < kDgsPhases / 2; ++ph) dgs_phase(c, level, L.x, L.b, ph + 32 * T);
                for (int T = 7; T >= 0; --T)
                    for (int ph = kDgsPhases / 2; ph < kDgsPhases; ++ph) dgs_phase(c, level, L.x, L.b, ph + 32 * T);
            } else {
                for (int ph = 0; ph < kDgsPhases; ++ph) dgs_phase(c, level, L.x, L.b, ph);
            }
            vanka_sym(c, level, L.x, L.b);
        }
        else if (op == 4) smooth(c, level, L.x, L.b);
        else throw SmgError(SMG_EINVAL, "bad smoother op");
        download(c, level, L.x, x);
    });
}

int smg_restrict(smg_ctx* c, int level, const double* rf, double* rc) {
    return guard(c, [&] {
        if (c->ndist > 0) throw SmgError(SMG_EINVAL, "single-part entry point (use ngpu = 1)");
        check_level(c, level);
        check_level(c, level + 1);
        DevLevel &F = c->lv[level], &C = c->lv[level + 1];
        upload(c, level, rf, F.r);
        launch_restrict(F.k, C.k, F.r, C.b, c->st);
        download(c, level + 1, C.b, rc);
    });
}

int smg_prolong(smg_ctx* c, int level, const double* xc, double* xf) {
    return guard(c, [&] {
        if (c->ndist > 0) throw SmgError(SMG_EINVAL, "single-part entry point (use ngpu = 1)");
        check_level(c, level);
        check_level(c, level + 1);
        DevLevel &F = c->lv[level], &C = c->lv[level + 1];
        upload(c, level + 1, xc, C.x);
        CK(cudaMemsetAsync(F.x, 0, vlen(F) * sizeof(double), c->st));
        launch_prolong_add(F.k, C.k, C.x, F.x, c->st);
        download(c, level, F.x, xf);
    });
}

int smg_coarse_solve(smg_ctx* c, const double* b, double* x) {
    return guard(c, [&] {
        if (c->ndist > 0) throw SmgError(SMG_EINVAL, "single-part entry point (use ngpu = 1)");
        const int l = static_cast<int>(c->lv.size()) - 1;
        DevLevel& C = c->lv[l];
        upload(c, l, b, C.b);
        coarse_solve(c, C.b, C.x);
        download(c, l, C.x, x);
    });
}

int smg_vcycle(smg_ctx* c, const double* b, double* x) {
    return guard(c, [&] {
        if (c->ndist > 0) {
            dist_upload(c, b, v_s);
            dist_vcycle(c, 0);
            dist_download(c, v_t, x);
            return;
        }
        DevLevel& F = c->lv[0];
        upload(c, 0, b, F.b);
        vcycle(c, 0, F.b, F.x);
        download(c, 0, F.x, x);
    });
}

int smg_mg_solve(smg_ctx* c, const double* b, double* x, double tol, int maxit, smg_history* hist, int* status) {
    return guard(c, [&] {
        if (!b || !x || !status) throw SmgError(SMG_EINVAL, "null argument");
        if (c->ndist > 0) throw SmgError(SMG_EINVAL, "single-part entry point (use ngpu = 1)");
        DevLevel& F = c->lv[0];
        const int64_t n = vlen(F);
        double* sc = c->dscal;
        auto t0 = std::chrono::steady_clock::now();
        const int64_t l0 = launch_count();
        upload(c, 0, b, c->rhs);
        CK(cudaEventRecord(c->ev0, c->st));
        if (hist) hist->count = 0;
        CK(cudaMemsetAsync(c->xs, 0, n * sizeof(double), c->st));
        launch_cdot2(F.k.g, c->rhs, c->rhs, nullptr, nullptr, c->partials, sc + S_D0, c->st);
        CK(cudaMemcpyAsync(c->hscal, sc, sizeof(double), cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        const double bnorm = std::sqrt(c->hscal[0]);
        int st = SMG_MAX_ITERATIONS, iters = 0;
        if (bnorm == 0.0) {
            st = SMG_CONVERGED;
        } else {
            CK(cudaMemcpyAsync(F.b, c->rhs, n * sizeof(double), cudaMemcpyDeviceToDevice, c->st));  // r_0 = b
            for (int j = 1; j <= maxit; ++j) {
                vcycle(c, 0, F.b, F.x);                                 // e = cycle(r)
                launch_axpy(c->xs, F.x, 1.0, n, c->st);                 // x += e
                launch_apply(F.k, c->xs, c->rhs, F.b, F.k.gamma, c->st);  // r = b - L~ x
                launch_cdot2(F.k.g, F.b, F.b, nullptr, nullptr, c->partials, sc + S_D0, c->st);
                CK(cudaMemcpyAsync(c->hscal, sc, sizeof(double), cudaMemcpyDeviceToHost, c->st));
                CK(cudaStreamSynchronize(c->st));
                const double rel = std::sqrt(c->hscal[0]) / bnorm;
                iters = j;
                if (hist && hist->count < hist->capacity) {
                    hist->rel_residual[hist->count] = rel;
                    hist->seconds[hist->count] =
                        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                    hist->count++;
                }
                if (rel < tol) { st = SMG_CONVERGED; break; }
            }
        }
        CK(cudaEventRecord(c->ev1, c->st));
        CK(cudaEventSynchronize(c->ev1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
        c->timing.solve_ms = ms;
        c->timing.iterations = iters;
        c->timing.kernel_launches = launch_count() - l0;
        download(c, 0, c->xs, x);
        *status = st;
    });
}

int smg_set_rhs(smg_ctx* c, const double* b) {
    return guard(c, [&] {
        if (c->ndist > 0) {
            dist_upload(c, b, v_rhs);
            c->rhs_set = true;
            return;
        }
        upload(c, 0, b, c->rhs);
        CK(cudaStreamSynchronize(c->st));
        c->rhs_set = true;
    });
}

int smg_solve_resident(smg_ctx* c, double tol, int maxit, smg_history* hist, int* status) {
    return guard(c, [&] {
        if (!c->rhs_set) throw SmgError(SMG_EINVAL, "smg_set_rhs not called");
        if (!status) throw SmgError(SMG_EINVAL, "status is null");
        sqmr(c, tol, maxit, hist, status);
    });
}

int smg_get_solution(smg_ctx* c, double* x) {
    return guard(c, [&] {
        if (c->ndist > 0) dist_download(c, v_xs, x);
        else download(c, 0, v_xs(c), x);
    });
}

int smg_sqmr_solve(smg_ctx* c, const double* b, double* x, double tol, int maxit, smg_history* hist, int* status) {
    return guard(c, [&] {
        if (!b || !x || !status) throw SmgError(SMG_EINVAL, "null argument");
        if (c->ndist > 0) {
            dist_upload(c, b, v_rhs);
            c->rhs_set = true;
            sqmr(c, tol, maxit, hist, status);
            dist_download(c, v_xs, x);
            return;
        }
        CK(cudaEventRecord(c->ev0, c->st));
        upload(c, 0, b, c->rhs);
        CK(cudaEventRecord(c->ev1, c->st));
        CK(cudaEventSynchronize(c->ev1));
        float h2d = 0.f;
        CK(cudaEventElapsedTime(&h2d, c->ev0, c->ev1));
        c->rhs_set = true;
        sqmr(c, tol, maxit, hist, status);
        CK(cudaEventRecord(c->ev0, c->st));
        download(c, 0, v_xs(c), x);
        CK(cudaEventRecord(c->ev1, c->st));
        CK(cudaEventSynchronize(c->ev1));
        float d2h = 0.f;
        CK(cudaEventElapsedTime(&d2h, c->ev0, c->ev1));
        c->timing.h2d_ms = h2d;
        c->timing.d2h_ms = d2h;
    });
}

int smg_last_timing(const smg_ctx* c, smg_timing* out) {
    if (!c || !out) return SMG_EINVAL;
    *out = c->timing;
    return 0;
}

int smg_time_kernel(smg_ctx* c, int which, int level, int reps, double* avg_ms) {
    return guard(c, [&] {
        if (reps < 1 || !avg_ms) throw SmgError(SMG_EINVAL, "bad reps");
        check_level(c, level);
        DevLevel& L = c->lv[level];
        const bool coarse = level == static_cast<int>(c->lv.size()) - 1;
        auto one = [&] {
            switch (which) {
                case 0: launch_apply(L.k, L.x, nullptr, L.r, 0.0, c->st); break;
                case 1: launch_apply(L.k, L.x, L.b, L.r, L.k.gamma, c->st); break;
                case 2: symmetric_dgs(c, level, L.x, L.b); break;
                case 3: vcycle(c, level, L.b, L.x); break;
                case 4: vanka_sym_coop(c, level, L.x, L.b); break;
                case 5: smooth(c, level, L.x, L.b); break;
                case 6:
                    if (!coarse) launch_restrict(L.k, c->lv[level + 1].k, L.r, c->lv[level + 1].b, c->st);
                    break;
                case 7:
                    if (!coarse) launch_prolong_add(L.k, c->lv[level + 1].k, c->lv[level + 1].x, L.x, c->st);
                    break;
                case 8: coarse_solve(c, c->lv.back().b, c->lv.back().x); break;
                case 9: launch_cdot2(L.k.g, L.x, L.x, L.b, L.b, c->partials, c->dscal, c->st); break;
                case 10: launch_axpy_s(L.b, L.x, c->dscal, vlen(L), c->st); break;
                case 11:
                    if (!c->graph) throw SmgError(SMG_EINVAL, "no SQMR graph captured yet");
                    CK(cudaGraphLaunch(c->graph, c->st));
                    break;
                case 12: launch_dgs_cb(L.k, L.b, c->st); break;  // m^T b (+ the tile-major copy of b) of a level visit
                case 13: symmetric_dgs(c, level, L.x, L.b, /*cb_ready=*/true); break;  // the sweep as the V-cycle runs it
                case 14: smooth(c, level, L.x, L.b, /*cb_ready=*/true); break;
                default: throw SmgError(SMG_EINVAL, "bad kernel id");
            }
        };
        if (which == 13 || which == 14) launch_dgs_cb(L.k, L.b, c->st);
        one();
        CK(cudaEventRecord(c->ev0, c->st));
        for (int k = 0; k < reps; ++k) one();
        CK(cudaEventRecord(c->ev1, c->st));
        CK(cudaEventSynchronize(c->ev1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
        *avg_ms = ms / reps;
    });
}

int64_t smg_check_guards(smg_ctx* c) {
    if (!c) return SMG_EINVAL;
    int64_t bad = 0;
    const int rc = guard(c, [&] {
        bad = c->check_guards();
        for (auto& q : c->owned) bad += q->check_guards();
    });
    return rc != 0 ? rc : bad;
}

int smg_profiler_range(int on) {
    const cudaError_t e = on ? cudaProfilerStart() : cudaProfilerStop();
    return e == cudaSuccess ? 0 : SMG_ECUDA;
}

void* smg_host_alloc(int64_t bytes) {
    void* p = nullptr;
    if (cudaMallocHost(&p, static_cast<size_t>(bytes)) != cudaSuccess) return nullptr;
    return p;
}
void smg_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

namespace {
// Synthetic forcing of the BASELINE configs (OD-9) at a face: a pure function of (seed, component,
// storage coordinates), so it is independent of the numbering and of any decomposition.
struct Forcing {
    int kind;
    uint64_t seed;
    double h;
    double amp[3][8];
    int kw[3][8][3];
    Forcing(int kind_, uint64_t seed_, double h_) : kind(kind_), seed(seed_), h(h_) {
        if (kind == 1)
            for (int c = 0; c < 3; ++c)
                for (int md = 0; md < 8; ++md) {
                    for (int a = 0; a < 3; ++a) kw[c][md][a] = 1 + static_cast<int>(key5(seed, 16 + c, md, a, 0) % 8);
                    const double u1 = 1.0 - unit01(key5(seed, 32 + c, md, 0, 1));
                    const double u2 = unit01(key5(seed, 32 + c, md, 0, 2));
                    amp[c][md] = std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
                }
    }
    double operator()(int c, int x, int y, int z) const {
        const double u = 2.0 * unit01(key5(seed, c, x, y, z)) - 1.0;
        if (kind == 0) return u;
        if (kind == 2) return (c == 0 ? 1.0 : 0.0) + 0.1 * u;
        const int p[3] = {x, y, z};
        double xyz[3];
        for (int a = 0; a < 3; ++a) xyz[a] = (a == c) ? p[a] * h : (p[a] + 0.5) * h;
        double s = 0.0;
        for (int md = 0; md < 8; ++md)
            s = s + amp[c][md] * std::sin(3.141592653589793 * kw[c][md][0] * xyz[0]) *
                        std::sin(3.141592653589793 * kw[c][md][1] * xyz[1]) *
                        std::sin(3.141592653589793 * kw[c][md][2] * xyz[2]);
        return s;
    }
};
}  // namespace

int smg_forcing(const smg_grid_desc* grid, int kind, uint64_t seed, double* b, int threads) {
    if (!grid || !b || kind < 0 || kind > 2 || grid->dim != 3) return SMG_EINVAL;
    const int nx = grid->nx, ny = grid->ny, nz = grid->nz;
    const Forcing f(kind, seed, grid->h);
    const int64_t nu = static_cast<int64_t>(nx - 1) * ny * nz, nv = static_cast<int64_t>(nx) * (ny - 1) * nz;
    const int64_t nw = static_cast<int64_t>(nx) * ny * (nz - 1), np = static_cast<int64_t>(nx) * ny * nz;
    // one task per (component, z-plane)
    const int64_t tasks = 3 * static_cast<int64_t>(nz);
    host_parallel(tasks, threads < 1 ? 1 : threads, [&](int64_t lo, int64_t hi) {
        for (int64_t t = lo; t < hi; ++t) {
            const int c = static_cast<int>(t / nz), z = static_cast<int>(t % nz);
            const int ex = nx + (c == 0 ? 1 : 0), ey = ny + (c == 1 ? 1 : 0), ez = nz + (c == 2 ? 1 : 0);
            if (z >= ez) continue;
            for (int y = 0; y < ey; ++y)
                for (int x = 0; x < ex; ++x) {
                    int64_t id;
                    if (c == 0) {
                        if (x < 1 || x > nx - 1) continue;
                        id = (static_cast<int64_t>(z) * ny + y) * (nx - 1) + (x - 1);
                    } else if (c == 1) {
                        if (y < 1 || y > ny - 1) continue;
                        id = nu + (static_cast<int64_t>(z) * (ny - 1) + (y - 1)) * nx + x;
                    } else {
                        if (z < 1 || z > nz - 1) continue;
                        id = nu + nv + (static_cast<int64_t>(z - 1) * ny + y) * nx + x;
                    }
                    b[id] = f(c, x, y, z);
                }
        }
    });
    // pressure rows: b_p = 0 (zero divergence RHS)
    for (int64_t k = 0; k < np; ++k) b[nu + nv + nw + k] = 0.0;
    return 0;
}

int smg_assemble_rhs_labeled(const smg_grid_desc* grid, const uint8_t* labels, double eta, const double* gu,
                             const double* gv, const double* gw, double* b) {
    // assemble_rhs with general BoundaryData: every stencil leg of an active row into
    // a Dirichlet face moves to the right-hand side with the opposite sign of its matrix entry
    // (momentum: -eta/h^2 legs -> + eta/h^2 g; continuity: +1/h on the low face, -1/h on the high).
    if (!grid || !labels || !gu || !gv || !gw || !b || grid->dim != 3 || !(grid->h > 0)) return SMG_EINVAL;
    const size_t nc = static_cast<size_t>(grid->nx) * grid->ny * grid->nz;
    const auto mp = classify_labeled(std::vector<uint8_t>(labels, labels + nc), grid->nx, grid->ny, grid->nz, 1);
    const HostMap& m = *mp;
    const double e2 = eta / (grid->h * grid->h), ih = 1.0 / grid->h;
    const double* g[3] = {gu, gv, gw};
    const int n[3] = {m.nx, m.ny, m.nz};
    auto value = [&](int c, int x, int y, int z) {
        const int p[3] = {x, y, z};
        int e[3], q[3];
        for (int a = 0; a < 3; ++a) {
            e[a] = n[a] + (a == c ? 1 : 2);
            q[a] = p[a] + (a == c ? 0 : 1);
            if (q[a] < 0 || q[a] >= e[a]) return 0.0;
        }
        return g[c][(static_cast<size_t>(q[2]) * e[1] + q[1]) * e[0] + q[0]];
    };
    // status of a face anywhere (ring faces included): Dirichlet iff one of its two cells is
    auto dirichlet = [&](int c, int x, int y, int z) {
        return m.at(x - (c == 0), y - (c == 1), z - (c == 2)) == LAB_D || m.at(x, y, z) == LAB_D;
    };
    const int d[6][3] = {{-1, 0, 0}, {1, 0, 0}, {0, -1, 0}, {0, 1, 0}, {0, 0, -1}, {0, 0, 1}};
    for (int z = 0; z < m.nz; ++z)
        for (int y = 0; y < m.ny; ++y)
            for (int x = 0; x < m.nx; ++x) {
                const size_t q = m.ci(x, y, z);
                for (int c = 0; c < 3; ++c) {
                    const int32_t id = m.id[c][q];
                    if (id < 0) continue;
                    for (auto& k : d) {
                        const int fx = x + k[0], fy = y + k[1], fz = z + k[2];
                        if (!dirichlet(c, fx, fy, fz)) continue;
                        const double gval = value(c, fx, fy, fz);
                        if (gval != 0.0) b[id] = b[id] + e2 * gval;
                    }
                }
                const int32_t pid = m.id[3][q];
                if (pid < 0) continue;
                for (int c = 0; c < 3; ++c)
                    for (int side = 0; side < 2; ++side) {
                        const int fx = x + (c == 0) * side, fy = y + (c == 1) * side, fz = z + (c == 2) * side;
                        if (!dirichlet(c, fx, fy, fz)) continue;
                        const double gval = value(c, fx, fy, fz);
                        if (gval != 0.0) b[pid] = b[pid] - (side ? -ih : ih) * gval;
                    }
            }
    return 0;
}

int smg_forcing_labeled(const smg_grid_desc* grid, const uint8_t* labels, int kind, uint64_t seed, double* b) {
    if (!grid || !labels || !b || kind < 0 || kind > 2 || grid->dim != 3) return SMG_EINVAL;
    const size_t nc = static_cast<size_t>(grid->nx) * grid->ny * grid->nz;
    const auto m = classify_labeled(std::vector<uint8_t>(labels, labels + nc), grid->nx, grid->ny, grid->nz, 1);
    const Forcing f(kind, seed, grid->h);
    for (int z = 0; z < m->nz; ++z)
        for (int y = 0; y < m->ny; ++y)
            for (int x = 0; x < m->nx; ++x) {
                const size_t q = m->ci(x, y, z);
                for (int c = 0; c < 3; ++c)
                    if (m->id[c][q] >= 0) b[m->id[c][q]] = f(c, x, y, z);
                if (m->id[3][q] >= 0) b[m->id[3][q]] = 0.0;
            }
    return 0;
}

}  // extern "C"
