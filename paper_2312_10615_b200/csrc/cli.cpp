// cli.cpp — `solver` command line above the C-ABI (the
// reference's cli module restricted to the walled-box scenario of the hot path).
//
//   solver run <config.json>      solve; writes history_<method>.csv and summary.txt
//   solver census <config.json>   prints "N V1 pct%" (PAPER Table 1 layout)
//   solver verify [--max-n N]     symmetry of the materialised GPU smoother / V-cycle maps,
//                                 on the walled cube and on a labelled cube with an obstacle and an outflow
//   solver matrix <config.json>   dense L of the fine level (N <= 5000) as Matrix Market
//                                 coordinate text on stdout, materialised through smg_apply
//
// RunConfig (JSON, flat): nx, ny, nz (cells), h (default 1/nx), eta (1e-3),
// gamma (1e-3), levels, nu (1), band_width (1), cycle ("V"|"W"), method
// ("mg-sqmr"|"mg"), tol (1e-8), maxit (200), forcing ("uniform"|"fourier"|
// "channel"|"cavity": lid-driven, u = lid (1) on the top y face), seed (0), output_dir (env SMG_OUTPUT_DIR, else "."), devices ([0]),
// vanka ("multiplicative"|"additive"), omega (1), vtk (0; 1 writes fields.vtk),
// domain (path of a domain file: header line `dim nx ny nz h`, then one character per
// cell, D / I / E, row-major with x fastest, whitespace ignored -- a general labelled domain;
// nx, ny, nz, h then come from the file).
// Defaults follow SPEC:567-569.  Exit codes: 0 converged,
// 2 not converged, 1 usage/config error.
#include <algorithm>
#include <cerrno>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/smg.h"

namespace {

// Minimal JSON reader for one flat object of numbers, strings and number arrays.
struct Config {
    std::map<std::string, std::string> str;
    std::map<std::string, double> num;
    std::map<std::string, std::vector<double>> arr;
};

bool parse_json(const std::string& t, Config& c, std::string& err) {
    size_t i = 0;
    auto ws = [&] { while (i < t.size() && std::isspace(static_cast<unsigned char>(t[i]))) ++i; };
    auto str = [&](std::string& out) {
        if (t[i] != '"') return false;
        ++i;
        out.clear();
        while (i < t.size() && t[i] != '"') out += t[i++];
        if (i >= t.size()) return false;
        ++i;
        return true;
    };
    auto number = [&](double& v) {
        const char* b = t.c_str() + i;
        char* e = nullptr;
        errno = 0;
        v = std::strtod(b, &e);
        if (e == b || errno) return false;
        i += static_cast<size_t>(e - b);
        return true;
    };
    ws();
    if (i >= t.size() || t[i] != '{') { err = "expected '{'"; return false; }
    ++i;
    ws();
    if (t[i] == '}') return true;
    while (true) {
        ws();
        std::string key;
        if (!str(key)) { err = "expected a quoted key"; return false; }
        ws();
        if (t[i] != ':') { err = "expected ':' after " + key; return false; }
        ++i;
        ws();
        if (t[i] == '"') {
            std::string v;
            if (!str(v)) { err = "bad string for " + key; return false; }
            c.str[key] = v;
        } else if (t[i] == '[') {
            ++i;
            std::vector<double> a;
            ws();
            while (t[i] != ']') {
                double v;
                if (!number(v)) { err = "bad array for " + key; return false; }
                a.push_back(v);
                ws();
                if (t[i] == ',') { ++i; ws(); }
            }
            ++i;
            c.arr[key] = a;
        } else {
            double v;
            if (!number(v)) { err = "bad value for " + key; return false; }
            c.num[key] = v;
        }
        ws();
        if (t[i] == ',') { ++i; continue; }
        if (t[i] == '}') return true;
        err = "expected ',' or '}'";
        return false;
    }
}

// fields.vtk: legacy ASCII STRUCTURED_POINTS, pressure as CELL_DATA
// scalar, velocity averaged to cell centres (wall faces are 0, Dirichlet) as CELL_DATA
// vector.  x is the compact FieldVector: u (faces 1..nx-1), v, w, p, x fastest.
bool write_vtk(const std::string& path, int nx, int ny, int nz, double h, const std::vector<double>& x) {
    FILE* fo = std::fopen(path.c_str(), "w");
    if (!fo) return false;
    const int64_t nu = static_cast<int64_t>(nx - 1) * ny * nz, nv = static_cast<int64_t>(nx) * (ny - 1) * nz;
    const int64_t nw = static_cast<int64_t>(nx) * ny * (nz - 1);
    auto U = [&](int i, int y, int z) {  // u-face i (0..nx), 0 on the walls
        return (i <= 0 || i >= nx) ? 0.0 : x[(static_cast<int64_t>(z) * ny + y) * (nx - 1) + (i - 1)];
    };
    auto V = [&](int xx, int j, int z) {
        return (j <= 0 || j >= ny) ? 0.0 : x[nu + (static_cast<int64_t>(z) * (ny - 1) + (j - 1)) * nx + xx];
    };
    auto W = [&](int xx, int y, int k) {
        return (k <= 0 || k >= nz) ? 0.0 : x[nu + nv + (static_cast<int64_t>(k - 1) * ny + y) * nx + xx];
    };
    std::fprintf(fo, "# vtk DataFile Version 3.0\nstokes MG-SQMR solution\nASCII\nDATASET STRUCTURED_POINTS\n");
    std::fprintf(fo, "DIMENSIONS %d %d %d\nORIGIN 0 0 0\nSPACING %.17g %.17g %.17g\n", nx + 1, ny + 1, nz + 1, h, h, h);
    std::fprintf(fo, "CELL_DATA %lld\nSCALARS pressure double 1\nLOOKUP_TABLE default\n",
                 static_cast<long long>(nx) * ny * nz);
    for (int64_t k = 0; k < static_cast<int64_t>(nx) * ny * nz; ++k) std::fprintf(fo, "%.17g\n", x[nu + nv + nw + k]);
    std::fprintf(fo, "VECTORS velocity double\n");
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (int xx = 0; xx < nx; ++xx)
                std::fprintf(fo, "%.17g %.17g %.17g\n", 0.5 * (U(xx, y, z) + U(xx + 1, y, z)),
                             0.5 * (V(xx, y, z) + V(xx, y + 1, z)), 0.5 * (W(xx, y, z) + W(xx, y, z + 1)));
    const bool ok = std::ferror(fo) == 0;
    std::fclose(fo);
    return ok;
}

// Domain file: `3 nx ny nz h` then nx*ny*nz characters D / I / E (whitespace ignored).
bool read_domain(const std::string& path, smg_grid_desc& g, std::vector<uint8_t>& lab, std::string& err) {
    std::ifstream f(path);
    if (!f) { err = "cannot read " + path; return false; }
    int dim = 0;
    if (!(f >> dim >> g.nx >> g.ny >> g.nz >> g.h) || dim != 3 || g.nx < 1 || g.ny < 1 || g.nz < 1 || !(g.h > 0)) {
        err = "bad domain header (expected: 3 nx ny nz h)";
        return false;
    }
    g.dim = 3;
    const size_t nc = static_cast<size_t>(g.nx) * g.ny * g.nz;
    lab.clear();
    lab.reserve(nc);
    char ch;
    while (f.get(ch)) {
        if (std::isspace(static_cast<unsigned char>(ch))) continue;
        if (ch == 'D') lab.push_back(0);
        else if (ch == 'I') lab.push_back(1);
        else if (ch == 'E') lab.push_back(2);
        else { err = std::string("bad cell label '") + ch + "'"; return false; }
    }
    if (lab.size() != nc) { err = "label count != nx*ny*nz (SPEC:28)"; return false; }
    return true;
}

int usage() {
    std::fprintf(stderr, "usage: solver run <config.json> | solver census <config.json> | solver matrix <config.json> | "
                         "solver verify [--max-n N]\n");
    return 1;
}

// verify (AC 3/4): materialise b -> x of the GPU smoothers and the
// V-cycle on n^3 cubes (n = 4, 8, ... <= max_n, x0 = 0) and report ||C - C^T||_F / ||C||_F.
int verify(int max_n) {
    bool ok = true;
    for (int n = 4; n <= max_n; n *= 2) {
        smg_grid_desc g{3, n, n, n, 1.0 / n};
        for (int vk = 0; vk < 2; ++vk) {
            smg_params p{1.0, 1e-3, 2, 1, 1, 0, 0, vk, 0.5, 0};
            int dev = 0;
            smg_ctx* ctx = nullptr;
            if (smg_create(&g, &p, 1, &dev, &ctx) != SMG_OK) return 1;
            const int64_t N = smg_level_ndof(ctx, 0, nullptr);
            struct Map { const char* name; int op; };
            const Map maps[] = {{"smooth", 4}, {vk ? "vanka_additive" : "vanka_symmetric", vk ? 5 : 3}, {"vcycle", -1}};
            for (const Map& m : maps) {
                std::vector<double> C(static_cast<size_t>(N * N)), e(N, 0.0), col(N);
                for (int64_t j = 0; j < N; ++j) {
                    e[j] = 1.0;
                    int rc;
                    if (m.op < 0) {
                        rc = smg_vcycle(ctx, e.data(), col.data());
                    } else {
                        std::fill(col.begin(), col.end(), 0.0);
                        rc = smg_smoother(ctx, 0, m.op, 0, col.data(), e.data());
                    }
                    if (rc != SMG_OK) { smg_destroy(ctx); return 1; }
                    for (int64_t i = 0; i < N; ++i) C[static_cast<size_t>(i * N + j)] = col[i];
                    e[j] = 0.0;
                }
                double d = 0.0, a = 0.0;
                for (int64_t i = 0; i < N; ++i)
                    for (int64_t j = 0; j < N; ++j) {
                        const double c = C[static_cast<size_t>(i * N + j)], t = C[static_cast<size_t>(j * N + i)];
                        d += (c - t) * (c - t);
                        a += c * c;
                    }
                const double defect = std::sqrt(d) / std::fmax(std::sqrt(a), 1e-300);
                const bool pass = defect < 1e-10 && a > 0.0;
                ok = ok && pass;
                std::printf("n=%d vanka=%s %s symmetry_defect=%.3e %s\n", n, vk ? "additive" : "multiplicative",
                            m.name, defect, pass ? "PASS" : "FAIL");
            }
            smg_destroy(ctx);
        }
        if (n < 8) continue;
        // the same maps on a general labelled domain: a Dirichlet block and an Exterior outflow column
        std::vector<uint8_t> lab(static_cast<size_t>(n) * n * n, 1);
        for (int z = 0; z < n; ++z)
            for (int y = 0; y < n; ++y)
                for (int x = 0; x < n; ++x) {
                    uint8_t& l = lab[(static_cast<size_t>(z) * n + y) * n + x];
                    if (x >= n / 4 && x < n / 2 && y >= n / 4 && y < n / 2) l = 0;
                    if (x == n - 1) l = 2;
                }
        smg_params p{1.0, 1e-3, 2, 1, 1, 0, 0, 0, 1.0, -1};
        smg_ctx* ctx = nullptr;
        if (smg_create_labeled(&g, lab.data(), &p, 0, &ctx) != SMG_OK) return 1;
        const int64_t N = smg_level_ndof(ctx, 0, nullptr);
        struct Map { const char* name; int op; };
        const Map maps[] = {{"smooth", 4}, {"vanka_symmetric", 3}, {"vcycle", -1}};
        for (const Map& m : maps) {
            std::vector<double> C(static_cast<size_t>(N * N)), e(N, 0.0), col(N);
            for (int64_t j = 0; j < N; ++j) {
                e[j] = 1.0;
                int rc;
                if (m.op < 0) {
                    rc = smg_vcycle(ctx, e.data(), col.data());
                } else {
                    std::fill(col.begin(), col.end(), 0.0);
                    rc = smg_smoother(ctx, 0, m.op, 0, col.data(), e.data());
                }
                if (rc != SMG_OK) { smg_destroy(ctx); return 1; }
                for (int64_t i = 0; i < N; ++i) C[static_cast<size_t>(i * N + j)] = col[i];
                e[j] = 0.0;
            }
            double d = 0.0, a = 0.0;
            for (int64_t i = 0; i < N; ++i)
                for (int64_t j = 0; j < N; ++j) {
                    const double c = C[static_cast<size_t>(i * N + j)], t = C[static_cast<size_t>(j * N + i)];
                    d += (c - t) * (c - t);
                    a += c * c;
                }
            const double defect = std::sqrt(d) / std::fmax(std::sqrt(a), 1e-300);
            const bool pass = defect < 1e-10 && a > 0.0;
            ok = ok && pass;
            std::printf("n=%d labelled %s symmetry_defect=%.3e %s\n", n, m.name, defect, pass ? "PASS" : "FAIL");
        }
        smg_destroy(ctx);
    }
    return ok ? 0 : 2;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc >= 2 && std::string(argv[1]) == "verify") {
        int max_n = 8;
        if (argc == 4 && std::string(argv[2]) == "--max-n") max_n = std::atoi(argv[3]);
        else if (argc != 2) return usage();
        if (max_n < 4) return usage();
        return verify(max_n);
    }
    if (argc != 3) return usage();
    const std::string cmd = argv[1];
    std::ifstream f(argv[2]);
    if (!f) { std::fprintf(stderr, "cannot read %s\n", argv[2]); return 1; }
    std::stringstream ss;
    ss << f.rdbuf();
    Config c;
    std::string err;
    if (!parse_json(ss.str(), c, err)) { std::fprintf(stderr, "config error: %s\n", err.c_str()); return 1; }
    auto num = [&](const char* k, double d) { return c.num.count(k) ? c.num[k] : d; };
    auto str = [&](const char* k, const char* d) { return c.str.count(k) ? c.str[k] : std::string(d); };
    std::vector<uint8_t> labels;  // non-empty: a general labelled domain from the "domain" file
    smg_grid_desc g{3, static_cast<int>(num("nx", 0)), 0, 0, 0.0};
    if (c.str.count("domain")) {
        if (!read_domain(c.str["domain"], g, labels, err)) { std::fprintf(stderr, "config error: %s\n", err.c_str()); return 1; }
    } else {
        if (!c.num.count("nx")) { std::fprintf(stderr, "config error: nx (or domain) is required\n"); return 1; }
        g.ny = static_cast<int>(num("ny", g.nx));
        g.nz = static_cast<int>(num("nz", g.nx));
        g.h = num("h", 1.0 / g.nx);
    }
    const int bw = static_cast<int>(num("band_width", 1));
    if (cmd == "census" && !labels.empty()) {
        int64_t out[6];
        if (smg_census_labeled(&g, labels.data(), bw, out) < 0) { std::fprintf(stderr, "config error: bad grid\n"); return 1; }
        std::printf("%lld %lld %.2f%%\n", static_cast<long long>(out[0]), static_cast<long long>(out[1]),
                    out[0] ? 100.0 * static_cast<double>(out[1]) / static_cast<double>(out[0]) : 0.0);
        return 0;
    }
    if (cmd == "census") {
        int64_t out[2];
        if (smg_census(&g, bw, out) < 0) { std::fprintf(stderr, "config error: bad grid\n"); return 1; }
        std::printf("%lld %lld %.2f%%\n", static_cast<long long>(out[0]), static_cast<long long>(out[1]),
                    100.0 * static_cast<double>(out[1]) / static_cast<double>(out[0]));
        return 0;
    }
    if (cmd != "run" && cmd != "matrix") return usage();
    const std::string vk = str("vanka", "multiplicative");  // SmootherConfig.kind
    if (vk != "multiplicative" && vk != "additive") { std::fprintf(stderr, "config error: vanka\n"); return 1; }
    smg_params p{num("eta", 1e-3), num("gamma", 1e-3), static_cast<int>(num("levels", 2)),
                 static_cast<int>(num("nu", 1)), bw, 0, str("cycle", "V") == "W" ? 1 : 0,
                 vk == "additive" ? 1 : 0, num("omega", 1.0), static_cast<int64_t>(num("dgs_tile_min", 0))};
    const std::string method = str("method", "mg-sqmr");
    if (method != "mg-sqmr" && method != "mg") { std::fprintf(stderr, "config error: method\n"); return 1; }
    const std::string fk = str("forcing", "uniform");
    const int kind = fk == "fourier" ? 1 : fk == "channel" ? 2 : 0;
    const double tol = num("tol", 1e-8);
    const int maxit = static_cast<int>(num("maxit", 200));
    const char* envdir = std::getenv("SMG_OUTPUT_DIR");
    const std::string dir = str("output_dir", envdir ? envdir : ".");
    std::vector<int> devs;
    for (double d : c.arr.count("devices") ? c.arr["devices"] : std::vector<double>{0}) devs.push_back(static_cast<int>(d));
    smg_ctx* ctx = nullptr;
    if (!labels.empty()) {
        if (fk == "cavity" || num("vtk", 0) != 0 || devs.size() != 1) {
            std::fprintf(stderr, "config error: a domain file takes forcing uniform|fourier|channel, one device, no vtk\n");
            return 1;
        }
        p.dgs_tile_min = -1;
        if (smg_create_labeled(&g, labels.data(), &p, devs[0], &ctx) != SMG_OK) {
            std::fprintf(stderr, "config error: smg_create_labeled failed\n");
            return 1;
        }
    } else if (smg_create(&g, &p, static_cast<int>(devs.size()), devs.data(), &ctx) != SMG_OK) {
        std::fprintf(stderr, "config error: smg_create failed\n");
        return 1;
    }
    int64_t cnt[5];
    const int64_t n = smg_level_ndof(ctx, 0, cnt);
    if (cmd == "matrix") {  // assemble_dense through the GPU operator, Matrix Market out
        if (n > 5000) {
            std::fprintf(stderr, "matrix: N = %lld above the cap 5000 (SPEC:158)\n", static_cast<long long>(n));
            smg_destroy(ctx);
            return 1;
        }
        std::vector<double> e(n, 0.0), col(n);
        std::vector<std::vector<std::pair<int64_t, double>>> cols(n);
        int64_t nnz = 0;
        for (int64_t j = 0; j < n; ++j) {
            e[j] = 1.0;
            if (smg_apply(ctx, 0, 0, e.data(), col.data()) != SMG_OK) { smg_destroy(ctx); return 1; }
            e[j] = 0.0;
            for (int64_t i = 0; i < n; ++i)
                if (col[i] != 0.0) { cols[j].push_back({i, col[i]}); ++nnz; }
        }
        std::printf("%%%%MatrixMarket matrix coordinate real general\n%lld %lld %lld\n", static_cast<long long>(n),
                    static_cast<long long>(n), static_cast<long long>(nnz));
        for (int64_t j = 0; j < n; ++j)
            for (auto& en : cols[j]) std::printf("%lld %lld %.17g\n", static_cast<long long>(en.first + 1), static_cast<long long>(j + 1), en.second);
        smg_destroy(ctx);
        return 0;
    }
    std::vector<double> b(n), x(n), hist(maxit), secs(maxit), lx(n);
    if (!labels.empty()) smg_forcing_labeled(&g, labels.data(), kind, static_cast<uint64_t>(num("seed", 0)), b.data());
    else if (fk == "cavity") smg_assemble_rhs(&g, p.eta, 0, num("lid", 1.0), b.data());  // zero force, lid u
    else smg_forcing(&g, kind, static_cast<uint64_t>(num("seed", 0)), b.data(), 8);
    smg_history h{maxit, 0, hist.data(), secs.data()};
    int status = -1;
    const auto t0 = std::chrono::steady_clock::now();
    const int rc = method == "mg" ? smg_mg_solve(ctx, b.data(), x.data(), tol, maxit, &h, &status)
                                  : smg_sqmr_solve(ctx, b.data(), x.data(), tol, maxit, &h, &status);
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (rc != SMG_OK) {
        std::fprintf(stderr, "solve failed: %s\n", smg_last_error(ctx));
        smg_destroy(ctx);
        return 1;
    }
    // ||B u||_inf from the continuity rows of L x
    double bu = 0.0;
    if (smg_apply(ctx, 0, 0, x.data(), lx.data()) == SMG_OK)
        for (int64_t k = n - cnt[3]; k < n; ++k) bu = std::fmax(bu, std::fabs(lx[k]));
    const std::string csv = dir + "/history_" + method + ".csv", sum = dir + "/summary.txt";
    if (FILE* fo = std::fopen(csv.c_str(), "w")) {
        std::fprintf(fo, "iteration,rel_residual,seconds\n");
        for (int k = 0; k < h.count; ++k) std::fprintf(fo, "%d,%.17g,%.9g\n", k + 1, hist[k], secs[k]);
        std::fclose(fo);
    }
    if (FILE* fo = std::fopen(sum.c_str(), "w")) {
        std::fprintf(fo, "method: %s\nstatus: %s\niterations: %d\nfinal_rel_residual: %.17g\n"
                         "div_u_inf: %.17g\nwall_seconds: %.6f\ndof: %lld\n",
                     method.c_str(), status == SMG_CONVERGED ? "converged" : status == SMG_BREAKDOWN ? "breakdown" : "max-iterations",
                     h.count, h.count ? hist[h.count - 1] : 0.0, bu, wall, static_cast<long long>(n));
        std::fclose(fo);
    }
    smg_destroy(ctx);
    // emit flags: "vtk": 1 writes output_dir/fields.vtk
    if (num("vtk", 0) != 0 && !write_vtk(dir + "/fields.vtk", g.nx, g.ny, g.nz, g.h, x)) {
        std::fprintf(stderr, "cannot write %s/fields.vtk\n", dir.c_str());
        return 1;
    }
    return status == SMG_CONVERGED ? 0 : 2;
}
