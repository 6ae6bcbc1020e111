// extern "C" face of the reference's own Rng (rng.hpp) and gen_instance
// (datagen.cpp), compiled unmodified from /root/reference/proj.  Test
// infrastructure: the oracle's RNG/datagen restatement is checked against it.
#include <cstdint>
#include <cstring>

#include "cimcs/datagen.hpp"
#include "cimcs/rng.hpp"

extern "C" {
int ref_gen_instance(int N, double alpha, double a, double nu, uint64_t seed, double* A,
                     double* y, double* x, int32_t* xi, int* M_out) {
    try {
        const cimcs::ProblemInstance inst = cimcs::gen_instance(N, alpha, a, nu, seed);
        const int M = inst.M();
        if (M_out) *M_out = M;
        if (A) std::memcpy(A, inst.A.data(), sizeof(double) * static_cast<size_t>(M) * N);
        if (y) std::memcpy(y, inst.y.data(), sizeof(double) * static_cast<size_t>(M));
        if (x) std::memcpy(x, inst.x_true.data(), sizeof(double) * static_cast<size_t>(N));
        if (xi)
            for (int r = 0; r < N; ++r) xi[r] = inst.xi_true[r];
        return 0;
    } catch (...) {
        return 1;
    }
}

void ref_gauss(uint64_t seed, int n, double* out) {
    cimcs::Rng rng(seed);
    for (int i = 0; i < n; ++i) out[i] = rng.gauss();
}

void ref_raw(uint64_t seed, int n, uint64_t* out) {
    cimcs::Rng rng(seed);
    for (int i = 0; i < n; ++i) out[i] = rng.raw();
}

uint64_t ref_uniform_below(uint64_t seed, uint64_t bound) {
    cimcs::Rng rng(seed);
    return rng.uniform_below(bound);
}
}
