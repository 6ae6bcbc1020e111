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
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <random>
#include <thread>
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
    // the same normal from two raw draws (gauss() == gauss_of(raw(), raw()))
    static double gauss_of(uint64_t r1, uint64_t r2) {
        const double u1 = (static_cast<double>(r1 >> 11) + 1.0) * 0x1.0p-53;
        const double u2 = (static_cast<double>(r2 >> 11) + 1.0) * 0x1.0p-53;
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * kPi * u2);
    }
    static constexpr double kPi = 3.14159265358979323846;

private:
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

// A of gen_instance with the same stream on `threads` host threads: the
// engine is inherently sequential (one thread draws the raw words, two per
// normal, in order), the Box-Muller transform and the column-major scatter of
// blocks of kb rows of A are spread over the workers (config 4: 5e9 normals).
inline void gen_matrix_parallel(HostRng& rng, int M, int N, double col_std, double* A,
                                int threads) {
    constexpr int kb = 64;  // rows of A (k) per chunk
    const int nchunks = (M + kb - 1) / kb;
    const int nbuf = 4;
    std::vector<std::vector<uint64_t>> buf(nbuf, std::vector<uint64_t>((size_t)2 * kb * N));
    std::vector<int> ready(nbuf, -1);  // chunk held by a buffer, -1 free
    std::vector<int> todo(nbuf, 0);    // workers still converting it
    std::mutex mu;
    std::condition_variable cv;
    auto produce = [&] {
        for (int c = 0; c < nchunks; ++c) {
            const int bi = c % nbuf;
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return ready[bi] < 0; });
            }
            const int rows = std::min(kb, M - c * kb);
            uint64_t* d = buf[bi].data();
            for (size_t t = 0; t < (size_t)2 * rows * N; ++t) d[t] = rng.raw();
            {
                std::lock_guard<std::mutex> lk(mu);
                ready[bi] = c;
                todo[bi] = threads;
            }
            cv.notify_all();
        }
    };
    auto consume = [&](int w) {
        for (int c = 0; c < nchunks; ++c) {
            const int bi = c % nbuf;
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return ready[bi] == c; });
            }
            const int k0 = c * kb, rows = std::min(kb, M - k0);
            const uint64_t* d = buf[bi].data();
            // worker w scatters columns r = w, w + threads, ... (contiguous runs of `rows`)
            for (int r = w; r < N; r += threads) {
                double* col = A + (size_t)r * M + k0;
                for (int k = 0; k < rows; ++k) {
                    const size_t t = 2 * ((size_t)k * N + r);
                    col[k] = col_std * HostRng::gauss_of(d[t], d[t + 1]);
                }
            }
            {
                std::lock_guard<std::mutex> lk(mu);
                if (--todo[bi] == 0) ready[bi] = -1;
            }
            cv.notify_all();
        }
    };
    std::vector<std::thread> pool;
    for (int w = 0; w < threads; ++w) pool.emplace_back(consume, w);
    produce();
    for (auto& th : pool) th.join();
}

// gen_instance (datagen.cpp:15-55): A (M x N column-major) drawn row-major,
// then x, then the support by partial Fisher-Yates, then the noise.
inline int gen_instance(int N, double alpha, double a, double nu, uint64_t seed, double* A,
                        double* y, double* x, int32_t* xi, int threads = 1) {
    int M, K;
    if (gen_dims(N, alpha, a, &M, &K) || nu < 0.0) return 1;
    HostRng rng(seed);
    const double col_std = 1.0 / std::sqrt(static_cast<double>(M));
    if (threads > 1 && (size_t)M * N >= ((size_t)1 << 22))
        gen_matrix_parallel(rng, M, N, col_std, A, threads);
    else
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
