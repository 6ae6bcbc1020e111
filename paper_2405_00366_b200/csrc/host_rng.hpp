// host_rng.hpp -- the reference's seeded stream, product side.
//
// Rng semantics of rng.hpp:21-64 (std::mt19937_64, 53-bit uniform in (0,1],
// Box-Muller with two uniforms per normal, no caching) built on the C++
// standard library's std::mt19937_64 -- the same engine the reference uses.
// The oracle restates MT19937-64 independently in C; tests cross-check the
// two streams bit for bit.
#pragma once

#include <cmath>
#include <cstdint>
#include <numeric>
#include <random>
#include <vector>

namespace cimcs {

class HostRng {
public:
    explicit HostRng(uint64_t seed = 0) : eng_(seed) {}
    uint64_t raw() { return eng_(); }
    double uniform_open() {
        const uint64_t u = eng_() >> 11;
        return (static_cast<double>(u) + 1.0) * 0x1.0p-53;
    }
    uint64_t uniform_below(uint64_t bound) {
        const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
        uint64_t v;
        do {
            v = eng_();
        } while (v >= limit);
        return v % bound;
    }
    double gauss() {
        const double u1 = uniform_open();
        const double u2 = uniform_open();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * kPi * u2);
    }

private:
    static constexpr double kPi = 3.14159265358979323846;
    std::mt19937_64 eng_;
};

inline long long round_half_away(double v) {
    return static_cast<long long>(v < 0 ? std::ceil(v - 0.5) : std::floor(v + 0.5));
}

inline uint64_t mix_seed(uint64_t base, uint64_t salt) {
    uint64_t z = base + 0x9E3779B97F4A7C15ULL * (salt + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// 0 ok, 1 input_error (datagen.cpp:17-24)
inline int gen_dims(int N, double alpha, double a, int* M, int* K) {
    if (N < 1) return 1;
    if (!(alpha > 0.0) || alpha > 1.0) return 1;
    if (a < 0.0 || a > 1.0) return 1;
    const int m = static_cast<int>(round_half_away(alpha * static_cast<double>(N)));
    if (m < 1) return 1;
    if (M) *M = m;
    if (K) *K = static_cast<int>(round_half_away(a * static_cast<double>(N)));
    return 0;
}

// gen_instance (datagen.cpp:15-55): A (M x N column-major) drawn row-major,
// then x, then the support by partial Fisher-Yates, then the noise.
inline int gen_instance(int N, double alpha, double a, double nu, uint64_t seed, double* A,
                        double* y, double* x, int32_t* xi) {
    int M, K;
    if (gen_dims(N, alpha, a, &M, &K) || nu < 0.0) return 1;
    HostRng rng(seed);
    const double col_std = 1.0 / std::sqrt(static_cast<double>(M));
    for (int k = 0; k < M; ++k)
        for (int r = 0; r < N; ++r) A[static_cast<size_t>(r) * M + k] = col_std * rng.gauss();
    for (int r = 0; r < N; ++r) x[r] = rng.gauss();
    std::vector<int> idx(N);
    std::iota(idx.begin(), idx.end(), 0);
    for (int r = 0; r < N; ++r) xi[r] = 0;
    for (int i = 0; i < K; ++i) {
        const int pick = i + static_cast<int>(rng.uniform_below(static_cast<uint64_t>(N - i)));
        std::swap(idx[i], idx[pick]);
        xi[idx[i]] = 1;
    }
    for (int k = 0; k < M; ++k) y[k] = 0.0;
    for (int r = 0; r < N; ++r) {
        const double w = xi[r] ? x[r] : 0.0;
        const double* col = A + static_cast<size_t>(r) * M;
        for (int k = 0; k < M; ++k) y[k] = y[k] + col[k] * w;
    }
    for (int k = 0; k < M; ++k) y[k] += nu * rng.gauss();
    return 0;
}

}  // namespace cimcs
