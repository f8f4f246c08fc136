// stokesmg/util.hpp — drop-in for /root/reference/proj/include/stokesmg/util.hpp:9-47.
//
// The three signatures below are the only compiled API the reference ships and
// are kept unchanged (namespace, names, argument and return types).  Semantics
// follow the reference contract:
//   * norm2 / dot: one sequential left-to-right accumulation in index order
//     (util.hpp:11-21), so results are bit-reproducible;
//   * parallel_for: synchronous, static contiguous blocks of ceil(n/workers)
//     items, at most min(threads, n) workers, and a plain sequential loop when
//     threads <= 1 or n < 2 (util.hpp:23-45).
// The GPU solver never calls these on its hot path; they serve the host side
// (CPU oracle, host setup) and keep the header a drop-in for callers.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <functional>
#include <thread>
#include <vector>

namespace stokesmg {

inline double dot(const std::vector<double>& a, const std::vector<double>& b) {
    const std::size_t n = a.size();
    const double* pa = a.data();
    const double* pb = b.data();
    double acc = 0.0;
    for (std::size_t k = 0; k != n; ++k) acc = acc + pa[k] * pb[k];
    return acc;
}

inline double norm2(const std::vector<double>& v) { return std::sqrt(dot(v, v)); }

inline void parallel_for(std::int64_t n, int threads,
                         const std::function<void(std::int64_t)>& body) {
    if (n < 2 || threads <= 1) {
        for (std::int64_t k = 0; k < n; ++k) body(k);
        return;
    }
    const std::int64_t nworkers = std::min<std::int64_t>(n, threads);
    const std::int64_t span = (n + nworkers - 1) / nworkers;
    std::vector<std::thread> crew;
    crew.reserve(static_cast<std::size_t>(nworkers));
    for (std::int64_t w = 0; w < nworkers; ++w) {
        const std::int64_t first = w * span;
        const std::int64_t last = std::min(n, first + span);
        crew.emplace_back([first, last, &body]() {
            for (std::int64_t k = first; k < last; ++k) body(k);
        });
    }
    for (std::thread& t : crew) t.join();
}

}  // namespace stokesmg
