// Probe of stokesmg::dot / norm2 / parallel_for (util.hpp:9-47): prints results that depend on the
// summation order (sequential, left to right), on norm2 = sqrt(dot(v, v)) and on the static block
// partition of parallel_for.  Compiled once against the reference's header (golden) and once
// against the repo's drop-in; the outputs must be identical.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <mutex>
#include <thread>
#include <vector>

#include "stokesmg/util.hpp"

int main() {
    // order-sensitive sums: a deterministic LCG with a wide dynamic range
    std::uint64_t st = 12345;
    auto next = [&] {
        st = st * 6364136223846793005ull + 1442695040888963407ull;
        const double u = static_cast<double>(st >> 11) * 0x1.0p-53 - 0.5;
        const int e = static_cast<int>((st >> 3) % 60) - 30;
        return std::ldexp(u, e);
    };
    for (int n : {0, 1, 2, 3, 17, 1000, 4099}) {
        std::vector<double> a(n), b(n);
        for (int i = 0; i < n; ++i) {
            a[i] = next();
            b[i] = next();
        }
        std::printf("n=%d dot=%.17g norm2=%.17g\n", n, stokesmg::dot(a, b), stokesmg::norm2(a));
    }
    std::vector<double> c{1e16, 1.0, -1e16, 3.0}, ones{1.0, 1.0, 1.0, 1.0};
    std::printf("absorb dot=%.17g norm2(3,4)=%.17g\n", stokesmg::dot(c, ones), stokesmg::norm2(std::vector<double>{3.0, 4.0}));
    // partition of parallel_for: which contiguous block each worker gets
    for (int threads : {1, 2, 3, 7, 16})
        for (std::int64_t n : {std::int64_t{1}, std::int64_t{5}, std::int64_t{16}, std::int64_t{1000}}) {
            std::vector<std::thread::id> who(static_cast<std::size_t>(n));
            std::vector<int> hit(static_cast<std::size_t>(n), 0);
            stokesmg::parallel_for(n, threads, [&](std::int64_t i) {
                who[static_cast<std::size_t>(i)] = std::this_thread::get_id();
                hit[static_cast<std::size_t>(i)] += 1;
            });
            int ok = 1;
            for (int h : hit) ok &= h == 1;
            std::printf("threads=%d n=%lld once=%d blocks:", threads, static_cast<long long>(n), ok);
            for (std::int64_t i = 1; i < n; ++i)
                if (who[static_cast<std::size_t>(i)] != who[static_cast<std::size_t>(i - 1)]) std::printf(" %lld", static_cast<long long>(i));
            std::printf("\n");
        }
    return 0;
}
