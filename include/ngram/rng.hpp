// rng.hpp -- drop-in for proj/include/ngram/rng.hpp (rng.hpp:14-40): the seeded
// randomness that defines reference banks and token streams, reproduced exactly so
// make_bank<T> here yields bit-identical banks.
#pragma once
#include <cmath>
#include <cstdint>
#include <random>

namespace ngram {

using rng64 = std::mt19937_64;

inline double uniform01(rng64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }

inline std::uint64_t uniform_below(rng64& g, std::uint64_t bound) {
    const std::uint64_t cut = ~std::uint64_t(0) - (~std::uint64_t(0)) % bound;
    for (;;) {
        const std::uint64_t x = g();
        if (x < cut) return x % bound;
    }
}

inline double gaussian(rng64& g) {
    double u = 0.0;
    while (u <= 0.0) u = uniform01(g);
    const double v = uniform01(g);
    return std::sqrt(-2.0 * std::log(u)) * std::cos(2.0 * 3.141592653589793 * v);
}

}  // namespace ngram
