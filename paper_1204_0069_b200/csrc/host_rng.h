// host_rng.h -- host side of the reference's counter-based SplitMix64 streams
// (coopcg/rng.hpp:16-20 mix64, :40-70 Stream, :80-87 make_stream), shared by
// the generators of coopcg_gpu.cu (BASELINE inputs) and refgen.cu (the
// reference's own make_problem family).  Every arithmetic step is one IEEE
// operation (volatile keeps the host compiler from contracting), so the bytes
// equal the reference build's (-ffp-contract=off, CMakeLists.txt:25).
#pragma once
#include <cmath>
#include <cstdint>

namespace coopcg_gpu {
namespace host_rng {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
// make_stream(seed, id, extra) key (rng.hpp:80-87)
inline uint64_t key(uint64_t seed, uint64_t id, uint64_t extra) { return mix64(seed ^ mix64(id ^ mix64(extra))); }
// draw c (1-based counter) of a stream (rng.hpp:40)
inline uint64_t draw(uint64_t k, uint64_t c) { return mix64(k + c * kGolden); }
inline double unit(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }
// next_uniform(lo, hi) = lo + (hi - lo) * unit (rng.hpp:47-49)
inline double uniform(uint64_t k, uint64_t c, double lo, double hi) {
    volatile double span = hi - lo;
    volatile double t = span * unit(draw(k, c));
    return lo + t;
}
// next_normal (rng.hpp:62-70): normal number t (0-based) consumes draws 2t+1, 2t+2
inline double normal(uint64_t k, uint64_t t) {
    double u1 = unit(draw(k, 2 * t + 1));
    double u2 = unit(draw(k, 2 * t + 2));
    if (u1 <= 0.0) u1 = 0x1.0p-53;
    volatile double l = -2.0 * std::log(u1);
    const double r = std::sqrt(l);
    const double two_pi = 6.283185307179586476925286766559;
    volatile double ang = two_pi * u2;
    volatile double cs = std::cos(ang);
    return r * cs;
}

}  // namespace host_rng
}  // namespace coopcg_gpu
