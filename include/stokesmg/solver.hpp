// stokesmg/solver.hpp — the SPEC-named host C++ API of the MG-preconditioned SQMR
// Stokes solver (arXiv 2312.10615), header-only, over the C-ABI of include/smg.h.
//
// The reference ships its solver only as a behavioural spec; this header
// gives the operations their SPEC names and argument meaning so a caller of the
// reference's C++ API (namespace stokesmg, proj/include/stokesmg/util.hpp) finds:
//
//   classify_dofs(CellGrid)                        SPEC:45-53   (host, any labelling)
//   partition_band(CellGrid, DofMap&, width)       SPEC:63-71   (host)
//   coarsen_grid(CellGrid)                         SPEC:54-62   (host)
//   build_hierarchy(grid, eta, gamma, n, cfg)      SPEC:361-369 (-> MgHierarchy, owns the GPU context)
//   apply(LevelOperator, FieldVector)
//   prolong / restrict_(TransferPair, FieldVector) SPEC:203-225 (`restrict` is a C keyword)
//   smooth(LevelOperator, x, b, cfg)
//   cycle(MgHierarchy, b, cfg)
//   mg_solve(MgHierarchy, b, tol, maxit)
//   sqmr_solve(L, precond, b, tol, maxit)          SPEC:422-430 (-> x, ResidualHistory, status)
//
// FieldVector is the SPEC's compact vector (u-lex, v-lex, w-lex, p-lex).
// Errors follow the SPEC: length mismatch throws std::invalid_argument (SPEC:125,
// 208, 216), the coarse dense cap throws std::length_error, other
// failures std::runtime_error carrying smg_last_error(); solver outcomes are a
// status, not an exception.  build_hierarchy takes any labelled CellGrid:
// the walled box (every cell Interior inside the implicit Dirichlet ring, the BASELINE
// configurations) runs the box kernels (smg_create); a grid with Dirichlet or Exterior cells
// runs the labelled-domain kernels (smg_create_labeled: obstacles, homogeneous-Neumann
// faces with dropped stencil legs).  Link with -lsmg (paper_2312_10615_b200/libsmg.so).
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../smg.h"  // NOLINT: the C-ABI this layer wraps
#include "util.hpp"

namespace stokesmg {

// ----------------------------------------------------------------- domain
enum class CellLabel : std::uint8_t { Dirichlet = 0, Interior = 1, Exterior = 2 };

struct CellGrid {  // SPEC:26-28; labels row-major, x fastest
    int dim = 3;
    int extents[3] = {1, 1, 1};
    double h = 1.0;
    std::vector<CellLabel> labels;
    CellLabel at(int x, int y, int z) const {  // outside the box: the implicit Dirichlet ring
        if (x < 0 || y < 0 || z < 0 || x >= extents[0] || y >= extents[1] || z >= extents[2])
            return CellLabel::Dirichlet;
        return labels[(static_cast<std::size_t>(z) * extents[1] + y) * extents[0] + x];
    }
    static CellGrid box(int nx, int ny, int nz, double h) {  // walled box (BASELINE configs)
        CellGrid g;
        g.extents[0] = nx;
        g.extents[1] = ny;
        g.extents[2] = nz;
        g.h = h;
        g.labels.assign(static_cast<std::size_t>(nx) * ny * nz, CellLabel::Interior);
        return g;
    }
};

struct DofStatus {  // Active(index) / DirichletValue / Inactive
    static constexpr std::int64_t Dirichlet = -1, Inactive = -2;
};

struct DofMap {
    int extents[3] = {1, 1, 1};
    std::vector<std::int64_t> face[3];  // per component: (n_x + (c==0)) x ... statuses
    std::vector<std::int64_t> cell;     // per cell
    std::int64_t count[4] = {0, 0, 0, 0};  // active u, v, w, p
    std::int64_t N = 0;
    std::vector<std::uint8_t> band;  // per active DOF: 1 = V1
    std::int64_t v1() const {
        std::int64_t s = 0;
        for (auto b : band) s += b;
        return s;
    }
};

// classify_dofs: faces of Dirichlet cells are DirichletValue, faces between two
// Interior cells Active, Interior|Exterior faces Inactive; pressures Active iff Interior;
// numbering u-lex, v-lex, w-lex, p-lex (x fastest).
inline DofMap classify_dofs(const CellGrid& g) {
    if (g.dim != 3) throw std::invalid_argument("classify_dofs: 3-D grids only");
    DofMap m;
    for (int a = 0; a < 3; ++a) m.extents[a] = g.extents[a];
    std::int64_t next = 0;
    for (int c = 0; c < 3; ++c) {
        const int ex = g.extents[0] + (c == 0), ey = g.extents[1] + (c == 1), ez = g.extents[2] + (c == 2);
        m.face[c].assign(static_cast<std::size_t>(ex) * ey * ez, DofStatus::Inactive);
        const std::int64_t first = next;
        for (int z = 0; z < ez; ++z)
            for (int y = 0; y < ey; ++y)
                for (int x = 0; x < ex; ++x) {
                    const CellLabel a = g.at(x - (c == 0), y - (c == 1), z - (c == 2)), b = g.at(x, y, z);
                    std::int64_t st;
                    if (a == CellLabel::Dirichlet || b == CellLabel::Dirichlet) st = DofStatus::Dirichlet;
                    else if (a == CellLabel::Interior && b == CellLabel::Interior) st = next++;
                    else st = DofStatus::Inactive;
                    m.face[c][(static_cast<std::size_t>(z) * ey + y) * ex + x] = st;
                }
        m.count[c] = next - first;
    }
    const std::size_t nc = g.labels.size();
    m.cell.assign(nc, DofStatus::Inactive);
    const std::int64_t first = next;
    for (std::size_t q = 0; q < nc; ++q)
        if (g.labels[q] == CellLabel::Interior) m.cell[q] = next++;
    m.count[3] = next - first;
    m.N = next;
    return m;
}

// partition_band: a cell is a band cell iff some cell within Chebyshev
// distance `width` is not Interior; the active DOFs on band-cell faces / centres form V1.
inline void partition_band(const CellGrid& g, DofMap& m, int width = 1) {
    if (width < 1) throw std::invalid_argument("partition_band: width >= 1");
    const int nx = g.extents[0], ny = g.extents[1], nz = g.extents[2];
    std::vector<std::uint8_t> bc(static_cast<std::size_t>(nx) * ny * nz, 0);
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x) {
                bool b = false;
                for (int k = -width; k <= width && !b; ++k)
                    for (int j = -width; j <= width && !b; ++j)
                        for (int i = -width; i <= width && !b; ++i) b = g.at(x + i, y + j, z + k) != CellLabel::Interior;
                bc[(static_cast<std::size_t>(z) * ny + y) * nx + x] = b;
            }
    auto band = [&](int x, int y, int z) {
        return x >= 0 && y >= 0 && z >= 0 && x < nx && y < ny && z < nz && bc[(static_cast<std::size_t>(z) * ny + y) * nx + x];
    };
    m.band.assign(static_cast<std::size_t>(m.N), 0);
    for (int c = 0; c < 3; ++c) {
        const int ex = nx + (c == 0), ey = ny + (c == 1), ez = nz + (c == 2);
        for (int z = 0; z < ez; ++z)
            for (int y = 0; y < ey; ++y)
                for (int x = 0; x < ex; ++x) {
                    const std::int64_t id = m.face[c][(static_cast<std::size_t>(z) * ey + y) * ex + x];
                    if (id >= 0) m.band[id] = band(x - (c == 0), y - (c == 1), z - (c == 2)) || band(x, y, z);
                }
    }
    for (std::size_t q = 0; q < m.cell.size(); ++q)
        if (m.cell[q] >= 0) m.band[m.cell[q]] = bc[q];
}

// coarsen_grid: D if any child D, else I if any child I, else E; odd extents
// padded with Exterior; an extent of 1 is rejected.
inline CellGrid coarsen_grid(const CellGrid& f) {
    CellGrid c;
    c.dim = f.dim;
    for (int a = 0; a < 3; ++a) {
        if (f.extents[a] < 2) throw std::invalid_argument("coarsen_grid: extent 1");
        c.extents[a] = (f.extents[a] + 1) / 2;
    }
    c.h = 2.0 * f.h;
    c.labels.assign(static_cast<std::size_t>(c.extents[0]) * c.extents[1] * c.extents[2], CellLabel::Exterior);
    for (int z = 0; z < c.extents[2]; ++z)
        for (int y = 0; y < c.extents[1]; ++y)
            for (int x = 0; x < c.extents[0]; ++x) {
                bool d = false, in = false;
                for (int k = 0; k < 2; ++k)
                    for (int j = 0; j < 2; ++j)
                        for (int i = 0; i < 2; ++i) {
                            const int fx = 2 * x + i, fy = 2 * y + j, fz = 2 * z + k;
                            if (fx >= f.extents[0] || fy >= f.extents[1] || fz >= f.extents[2]) continue;
                            const CellLabel l = f.at(fx, fy, fz);
                            d |= l == CellLabel::Dirichlet;
                            in |= l == CellLabel::Interior;
                        }
                c.labels[(static_cast<std::size_t>(z) * c.extents[1] + y) * c.extents[0] + x] =
                    d ? CellLabel::Dirichlet : (in ? CellLabel::Interior : CellLabel::Exterior);
            }
    return c;
}

// ------------------------------------------------------------ configuration
enum class BoundarySmoother { Multiplicative = 0, Additive = 1, Direct = 2 };  // Direct: SPEC:314, 333
struct SmootherConfig {
    BoundarySmoother kind = BoundarySmoother::Multiplicative;
    int nu = 1;          // boundary sweeps per side
    int band_width = 1;  // V1 band (Chebyshev)
    double omega = 1.0;  // additive damping
};
enum class CycleKind { V = 0, W = 1 };
struct CycleConfig {
    CycleKind kind = CycleKind::V;
    SmootherConfig smoother;
};

using FieldVector = std::vector<double>;

// ------------------------------------------------------------------ hierarchy
class MgHierarchy {
   public:
    // flags: SMG_FLAG_* (SMG_FLAG_NO_PRECOND: sqmr_solve on this hierarchy runs un-preconditioned)
    MgHierarchy(const CellGrid& g, double eta, double gamma, int n, const CycleConfig& cfg, int device = 0,
                int flags = 0) {
        if (g.labels.size() != static_cast<std::size_t>(g.extents[0]) * g.extents[1] * g.extents[2])
            throw std::invalid_argument("build_hierarchy: labels length != product of extents (SPEC:28)");
        bool box = true;
        for (auto l : g.labels) box = box && l == CellLabel::Interior;
        grid_ = smg_grid_desc{3, g.extents[0], g.extents[1], g.extents[2], g.h};
        prm_ = smg_params{eta,  gamma, n, cfg.smoother.nu, cfg.smoother.band_width, flags, static_cast<int>(cfg.kind),
                          static_cast<int>(cfg.smoother.kind), cfg.smoother.omega, 0};
        static_assert(sizeof(CellLabel) == 1, "CellLabel is the C-ABI's uint8 label");
        const int rc = box ? smg_create(&grid_, &prm_, 1, &device, &ctx_)
                           : smg_create_labeled(&grid_, reinterpret_cast<const std::uint8_t*>(g.labels.data()), &prm_,
                                                device, &ctx_);
        if (rc == SMG_ECAP) throw std::length_error("build_hierarchy: coarsest system above the dense cap (SPEC:365)");
        if (rc == SMG_EINVAL) throw std::invalid_argument("build_hierarchy: invalid grid / parameters");
        if (rc != 0) throw std::runtime_error("build_hierarchy: smg_create failed (" + std::to_string(rc) + ")");
    }
    MgHierarchy(const MgHierarchy&) = delete;
    MgHierarchy& operator=(const MgHierarchy&) = delete;
    MgHierarchy(MgHierarchy&& o) noexcept : ctx_(o.ctx_), grid_(o.grid_), prm_(o.prm_) { o.ctx_ = nullptr; }
    ~MgHierarchy() {
        if (ctx_) smg_destroy(ctx_);
    }
    smg_ctx* ctx() const { return ctx_; }
    int levels() const { return smg_num_levels(ctx_); }
    int flags() const { return prm_.flags; }
    std::int64_t ndof(int level = 0) const { return smg_level_ndof(ctx_, level, nullptr); }
    void check(int rc, const char* what) const {
        if (rc == 0) return;
        const std::string msg = std::string(what) + ": " + smg_last_error(ctx_);
        if (rc == SMG_EINVAL) throw std::invalid_argument(msg);
        throw std::runtime_error(msg);
    }
    void need(const FieldVector& v, int level, const char* what) const {
        if (static_cast<std::int64_t>(v.size()) != ndof(level))
            throw std::invalid_argument(std::string(what) + ": length mismatch (SPEC:125)");
    }

   private:
    smg_ctx* ctx_ = nullptr;
    smg_grid_desc grid_{};
    smg_params prm_{};
};

// build_hierarchy
inline MgHierarchy build_hierarchy(const CellGrid& g, double eta, double gamma, int n, const CycleConfig& cfg = {},
                                   int device = 0, int flags = 0) {
    return MgHierarchy(g, eta, gamma, n, cfg, device, flags);
}

// ----------------------------------------------------------- operators
struct LevelOperator {  // L (penalized = false) or L~ of one level
    const MgHierarchy* h;
    int level = 0;
    bool penalized = false;
};
struct TransferPair {  // level <-> level + 1
    const MgHierarchy* h;
    int level = 0;
};

// apply
inline FieldVector apply(const LevelOperator& op, const FieldVector& x) {
    op.h->need(x, op.level, "apply");
    FieldVector y(x.size());
    op.h->check(smg_apply(op.h->ctx(), op.level, op.penalized ? 1 : 0, x.data(), y.data()), "apply");
    return y;
}
// prolong: fine = P coarse
inline FieldVector prolong(const TransferPair& t, const FieldVector& xc) {
    t.h->need(xc, t.level + 1, "prolong");
    FieldVector xf(static_cast<std::size_t>(t.h->ndof(t.level)));
    t.h->check(smg_prolong(t.h->ctx(), t.level, xc.data(), xf.data()), "prolong");
    return xf;
}
// restrict: coarse = (1/8) P^T fine
inline FieldVector restrict_(const TransferPair& t, const FieldVector& rf) {
    t.h->need(rf, t.level, "restrict");
    FieldVector rc(static_cast<std::size_t>(t.h->ndof(t.level + 1)));
    t.h->check(smg_restrict(t.h->ctx(), t.level, rf.data(), rc.data()), "restrict");
    return rc;
}
// smooth, Alg. 3, with the hierarchy's SmootherConfig; x updated in place
inline void smooth(const LevelOperator& op, FieldVector& x, const FieldVector& b) {
    op.h->need(x, op.level, "smooth");
    op.h->need(b, op.level, "smooth");
    op.h->check(smg_smoother(op.h->ctx(), op.level, 4, 0, x.data(), b.data()), "smooth");
}
// symmetric_dgs and symmetric multiplicative Vanka alone
inline void symmetric_dgs(const LevelOperator& op, FieldVector& x, const FieldVector& b) {
    op.h->need(x, op.level, "symmetric_dgs");
    op.h->need(b, op.level, "symmetric_dgs");
    op.h->check(smg_smoother(op.h->ctx(), op.level, 1, 0, x.data(), b.data()), "symmetric_dgs");
}
inline void vanka_multiplicative_symmetric(const LevelOperator& op, FieldVector& x, const FieldVector& b) {
    op.h->need(x, op.level, "vanka");
    op.h->need(b, op.level, "vanka");
    op.h->check(smg_smoother(op.h->ctx(), op.level, 3, 0, x.data(), b.data()), "vanka");
}

// ------------------------------------------------------------ multigrid / krylov
// cycle: x = W^dagger b with x0 = 0
inline FieldVector cycle(const MgHierarchy& h, const FieldVector& b) {
    h.need(b, 0, "cycle");
    FieldVector x(b.size());
    h.check(smg_vcycle(h.ctx(), b.data(), x.data()), "cycle");
    return x;
}

enum class SolveStatus { Converged = SMG_CONVERGED, MaxIterations = SMG_MAX_ITERATIONS, Breakdown = SMG_BREAKDOWN };
struct HistoryRecord {
    int iteration;
    double rel_residual;
    double seconds;
};
using ResidualHistory = std::vector<HistoryRecord>;
struct SolveResult {
    FieldVector x;
    ResidualHistory history;
    SolveStatus status;
};

namespace detail {
template <class F>
SolveResult run_solver(const MgHierarchy& h, const FieldVector& b, int maxit, F&& call) {
    h.need(b, 0, "solve");
    SolveResult r{FieldVector(b.size()), {}, SolveStatus::MaxIterations};
    std::vector<double> rel(static_cast<std::size_t>(maxit > 0 ? maxit : 1)), sec(rel.size());
    smg_history hist{static_cast<int>(rel.size()), 0, rel.data(), sec.data()};
    int st = 0;
    h.check(call(h.ctx(), b.data(), r.x.data(), &hist, &st), "solve");
    for (int k = 0; k < hist.count; ++k) r.history.push_back({k + 1, rel[k], sec[k]});
    r.status = static_cast<SolveStatus>(st);
    return r;
}
}  // namespace detail

// mg_solve: x_j = x_{j-1} + cycle(b - L~ x_{j-1})
inline SolveResult mg_solve(const MgHierarchy& h, const FieldVector& b, double tol, int maxit) {
    return detail::run_solver(h, b, maxit, [&](smg_ctx* c, const double* bb, double* x, smg_history* hh, int* st) {
        return smg_mg_solve(c, bb, x, tol, maxit, hh, st);
    });
}

// sqmr_solve: L = the level-0 operator (unpenalized), precond = the V-cycle on L~
// of the same hierarchy (the mg-sqmr method); x0 = 0, true relative residuals.
inline SolveResult sqmr_solve(const LevelOperator& L, const MgHierarchy& precond, const FieldVector& b, double tol,
                              int maxit) {
    if (L.h != &precond || L.level != 0 || L.penalized)
        throw std::invalid_argument("sqmr_solve: L must be level 0 (unpenalized) of the preconditioner's hierarchy");
    return detail::run_solver(precond, b, maxit, [&](smg_ctx* c, const double* bb, double* x, smg_history* hh, int* st) {
        return smg_sqmr_solve(c, bb, x, tol, maxit, hh, st);
    });
}

// solve_driver: method mg = mg_solve on L~, mg-sqmr = sqmr_solve with the cycle,
// sqmr = Alg. 4 with the identity preconditioner (the hierarchy must carry SMG_FLAG_NO_PRECOND:
// the iteration is captured once per hierarchy, so the method is fixed at build time).
enum class Method { Mg, MgSqmr, Sqmr };
inline SolveResult solve_driver(const MgHierarchy& h, Method method, const FieldVector& b, double tol, int maxit) {
    const bool plain = (h.flags() & SMG_FLAG_NO_PRECOND) != 0;
    if (method == Method::Mg) return mg_solve(h, b, tol, maxit);
    if ((method == Method::Sqmr) != plain)
        throw std::invalid_argument("solve_driver: method sqmr needs a hierarchy built with SMG_FLAG_NO_PRECOND "
                                    "(and mg-sqmr one without)");
    return sqmr_solve(LevelOperator{&h, 0, false}, h, b, tol, maxit);
}

// assemble_rhs for the walled box: body force f (compact order, pressures
// 0) plus the Dirichlet contributions of the lid-driven cavity (lid = tangential u on y = ny).
inline FieldVector cavity_rhs(const CellGrid& g, double eta, double lid) {
    const smg_grid_desc d{3, g.extents[0], g.extents[1], g.extents[2], g.h};
    const std::int64_t n = smg_census(&d, 1, nullptr);
    FieldVector b(static_cast<std::size_t>(n), 0.0);
    if (smg_assemble_rhs(&d, eta, 0, lid, b.data()) != 0) throw std::runtime_error("assemble_rhs failed");
    return b;
}

}  // namespace stokesmg
