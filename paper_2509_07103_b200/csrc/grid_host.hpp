// Host-side grid setup for the B200 lmKAN layer (product code, runs once per
// layer). Restates the reference grid construction so the device can locate
// cells without the reference library:
//   sigma            grid.hpp:14-17
//   build_grid       grid.hpp:44-68
//   interval_index   grid.hpp:72-75
// and derives the cell-locate threshold tables from interval_index itself
// (std::exp is glibc's here, exactly as in the reference build, so the tables
// reproduce the reference's ulp-level decisions; see DESIGN.md "Bit-exact cell
// indices").
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <vector>

namespace lmkan_b200 {
namespace host {

inline double sigma(double x) {
    const double t = std::exp(-std::fabs(x));
    return x > 0.0 ? 1.0 - 0.5 * t : 0.5 * t;
}

// Returns false when G < 3 (reference throws std::invalid_argument).
inline bool build_grid(int G, std::vector<double>& points, std::vector<double>& inv_areas) {
    if (G < 3) return false;
    points.assign(static_cast<std::size_t>(G) + 1, 0.0);
    for (int k = 1; 2 * k < G; ++k) {
        const double v = std::log(2.0 * k / G);
        points[k] = v;
        points[G - k] = -v;
    }
    if (G % 2 == 0) points[G / 2] = 0.0;
    points[0] = 2.0 * points[1] - points[2];
    points[G] = 2.0 * points[G - 1] - points[G - 2];
    inv_areas.assign(static_cast<std::size_t>(G) * G, 0.0);
    for (int i1 = 0; i1 < G; ++i1) {
        const double h1 = points[i1 + 1] - points[i1];
        for (int i2 = 0; i2 < G; ++i2) {
            const double h2 = points[i2 + 1] - points[i2];
            inv_areas[static_cast<std::size_t>(i1) * G + i2] = 1.0 / (h1 * h2);
        }
    }
    return true;
}

// floor(sigma(x) * G) clamped to [0, G-1]; NaN -> 0 (x86 cvttsd2si gives
// INT_MIN for NaN, which the reference clamp maps to 0).
inline int interval_index(int G, double x) {
    const double f = std::floor(sigma(x) * G);
    if (std::isnan(f)) return 0;
    const int i = static_cast<int>(f);
    return i < 0 ? 0 : (i >= G ? G - 1 : i);
}

inline uint64_t order_key(double x) {
    uint64_t u;
    std::memcpy(&u, &x, 8);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
inline double from_order_key(uint64_t k) {
    const uint64_t u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    double x;
    std::memcpy(&x, &u, 8);
    return x;
}

// t64[k-1] = min{double x : interval_index(x) >= k} by bisection over the
// total order of doubles (64 steps per threshold); t32[k-1] = smallest float
// >= t64[k-1], so for float x: x >= t32 <=> (double)x >= t64.
inline bool thresholds(int G, std::vector<double>& t64, std::vector<float>& t32) {
    if (G < 3) return false;
    t64.assign(G - 1, 0.0);
    t32.assign(G - 1, 0.0f);
    const double inf = std::numeric_limits<double>::infinity();
    for (int k = 1; k <= G - 1; ++k) {
        uint64_t lo = order_key(-inf), hi = order_key(inf);
        while (hi - lo > 1) {
            const uint64_t mid = lo + (hi - lo) / 2;
            if (interval_index(G, from_order_key(mid)) >= k) hi = mid; else lo = mid;
        }
        const double t = from_order_key(hi);
        t64[k - 1] = t;
        float f = static_cast<float>(t);  // round to nearest, then fix up to round-up
        if (static_cast<double>(f) < t) f = std::nextafter(f, std::numeric_limits<float>::infinity());
        t32[k - 1] = f;
    }
    return true;
}

}  // namespace host
}  // namespace lmkan_b200
