// extern "C" face of the reference's own io.cpp (bundles, CSV writer,
// format_double, fnv1a64), compiled unmodified from /root/reference/proj with
// the Eigen shim and the image's copy of nlohmann/json (the reference vendors
// it under vendor/, which is absent).  Test infrastructure only: pins
// csrc/io.hpp in both directions (tests/test_io.py).
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "cimcs/datagen.hpp"
#include "cimcs/io.hpp"

extern "C" {
int ref_format_double(double v, char* buf, int cap) {
    const std::string s = cimcs::format_double(v);
    if ((int)s.size() + 1 > cap) return 1;
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return 0;
}

uint64_t ref_fnv1a64(const char* p, uint64_t n) { return cimcs::fnv1a64(std::string(p, n)); }

int ref_save_generated(int N, double alpha, double a, double nu, uint64_t seed, int truth,
                       const char* dir) {
    try {
        cimcs::ProblemInstance inst = cimcs::gen_instance(N, alpha, a, nu, seed);
        if (!truth) {
            inst.x_true.resize(0);
            inst.xi_true.resize(0);
        }
        cimcs::save_instance(inst, dir);
        return 0;
    } catch (...) {
        return 1;
    }
}

// phase 1 (A == NULL): sizes + meta; phase 2: arrays.  1 = the reference threw.
int ref_load_instance(const char* dir, int* N, int* M, int* has_truth, double* meta4,
                      uint64_t* seed, double* A, double* y, double* x, int32_t* xi) {
    try {
        const cimcs::ProblemInstance inst = cimcs::load_instance(dir);
        *N = inst.N();
        *M = inst.M();
        *has_truth = inst.has_truth() ? 1 : 0;
        meta4[0] = inst.a;
        meta4[1] = inst.alpha;
        meta4[2] = inst.nu;
        *seed = inst.seed;
        if (A) {
            std::memcpy(A, inst.A.data(), sizeof(double) * (size_t)inst.M() * inst.N());
            std::memcpy(y, inst.y.data(), sizeof(double) * (size_t)inst.M());
            if (inst.has_truth() && x && xi) {
                std::memcpy(x, inst.x_true.data(), sizeof(double) * (size_t)inst.N());
                for (int r = 0; r < inst.N(); ++r) xi[r] = inst.xi_true[r];
            }
        }
        return 0;
    } catch (...) {
        return 1;
    }
}

// One table through the reference CsvWriter; cells row-major (nrows x ncells
// per row given by widths[]).  Returns the number of rows the writer rejected.
int ref_csv(const char* path, const char* const* comments, int nc, const char* const* cols,
            int ncol, const char* const* cells, const int* widths, int nrows) {
    std::vector<std::string> cm(comments, comments + nc), co(cols, cols + ncol);
    int rejected = 0;
    {
        cimcs::CsvWriter w(path, cm, co);
        const char* const* p = cells;
        for (int r = 0; r < nrows; ++r) {
            std::vector<std::string> row(p, p + widths[r]);
            p += widths[r];
            try {
                w.row(row);
            } catch (...) {
                ++rejected;
            }
        }
    }
    return rejected;
}
}
