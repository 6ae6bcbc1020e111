// io.hpp -- instance bundles and the CSV result contract (host C++).
//
// The data formats either side of the hot path: the
// reference hands instances between its CLI, tests and solver as bundles
// (io.hpp:20-29, io.cpp:86-167) and reports trials as CSV tables with a
// comment preamble (io.hpp:31-48, io.cpp:169-196; summary/history/failures
// columns tools/main.cpp:449-451, orchestrator.cpp:253-264, main.cpp:484).
// Doubles are written in the shortest decimal form that round-trips
// (io.cpp:18-25), so a bundle written here loads bit-exactly in the
// reference and vice versa (tests/test_io.py pins both directions against
// the reference's own io.cpp, built by oracle/Makefile.ref).
#pragma once

#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

namespace cimcs_io {

namespace fs = std::filesystem;

constexpr const char* kRngName = "mt19937_64-boxmuller-v1";  // rng.hpp:12

// Shortest "%.{15,16,17}g" text whose strtod is the same double (io.cpp:18-25).
inline std::string fmt_double(double v) {
    char buf[40];
    for (int p = 15; p <= 17; ++p) {
        std::snprintf(buf, sizeof buf, "%.*g", p, v);
        if (std::strtod(buf, nullptr) == v) break;
    }
    return buf;
}

// FNV-1a, 64-bit (io.cpp:27-34): offset basis 0xcbf29ce484222325, prime 2^40 + 0x1b3.
inline uint64_t fnv1a(const unsigned char* p, size_t n) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (size_t k = 0; k < n; ++k) h = (h ^ p[k]) * 0x100000001b3ull;
    return h;
}

inline bool put_file(const fs::path& p, const std::string& s, std::string* err) {
    std::ofstream f(p, std::ios::binary);
    if (f) f.write(s.data(), (std::streamsize)s.size());
    if (!f) {
        *err = "cannot write " + p.string();
        return false;
    }
    return true;
}

inline bool get_file(const fs::path& p, std::string* s, std::string* err) {
    std::ifstream f(p, std::ios::binary);
    if (!f) {
        *err = "cannot read " + p.string();
        return false;
    }
    std::ostringstream o;
    o << f.rdbuf();
    *s = o.str();
    return true;
}

// Numeric CSV rows: blank lines and '#' lines skipped, cells split on ',', ' '
// or '\t', each parsed with strtod until the first non-number (io.cpp:60-82).
// Calls row(k, values) per data row; returns the row count.
template <class F>
size_t scan_rows(const std::string& text, F&& row) {
    size_t nrow = 0, pos = 0;
    std::vector<double> v;
    std::string line;
    while (pos < text.size()) {
        size_t e = text.find('\n', pos);
        if (e == std::string::npos) e = text.size();
        line.assign(text, pos, e - pos);
        pos = e + 1;
        if (line.empty() || line[0] == '#') continue;
        v.clear();
        const char* p = line.c_str();
        while (*p) {
            char* end = nullptr;
            const double x = std::strtod(p, &end);
            if (end == p) break;
            v.push_back(x);
            p = end;
            while (*p == ',' || *p == ' ' || *p == '\t') ++p;
        }
        if (!v.empty()) row(nrow++, v);
    }
    return nrow;
}

struct Meta {
    int N = 0, M = 0;
    double a = 0, alpha = 0, nu = 0;
    uint64_t seed = 0;
};

// meta.json as the reference's json dump(2) lays it out: keys sorted, two-space
// indent (io.cpp:114-122).  Whole-valued doubles keep a ".0" like the json
// library's number formatter, so the reference reads them back as doubles.
inline std::string meta_json(const Meta& m) {
    auto d = [](double v) {
        std::string s = fmt_double(v);
        if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
        return s;
    };
    std::string s = "{\n";
    s += "  \"M\": " + std::to_string(m.M) + ",\n";
    s += "  \"N\": " + std::to_string(m.N) + ",\n";
    s += "  \"a\": " + d(m.a) + ",\n";
    s += "  \"alpha\": " + d(m.alpha) + ",\n";
    s += "  \"nu\": " + d(m.nu) + ",\n";
    s += std::string("  \"rng\": \"") + kRngName + "\",\n";
    s += "  \"seed\": " + std::to_string(m.seed) + "\n}\n";
    return s;
}

// The flat meta object: "key": number pairs (strings ignored).
inline bool parse_meta(const std::string& t, Meta* m, std::string* err) {
    auto num = [&](const char* key, bool* ok) -> std::string {
        const std::string k = std::string("\"") + key + "\"";
        size_t p = t.find(k);
        if (p == std::string::npos) {
            *ok = false;
            return "";
        }
        p = t.find(':', p + k.size());
        if (p == std::string::npos) {
            *ok = false;
            return "";
        }
        ++p;
        while (p < t.size() && (t[p] == ' ' || t[p] == '\n' || t[p] == '\t' || t[p] == '\r')) ++p;
        size_t e = p;
        while (e < t.size() && t[e] != ',' && t[e] != '}' && t[e] != '\n') ++e;
        return t.substr(p, e - p);
    };
    bool ok = true;
    const std::string N = num("N", &ok), M = num("M", &ok), a = num("a", &ok),
                      al = num("alpha", &ok), nu = num("nu", &ok), sd = num("seed", &ok);
    if (!ok) {
        *err = "meta.json: missing key";
        return false;
    }
    m->N = std::atoi(N.c_str());
    m->M = std::atoi(M.c_str());
    m->a = std::strtod(a.c_str(), nullptr);
    m->alpha = std::strtod(al.c_str(), nullptr);
    m->nu = std::strtod(nu.c_str(), nullptr);
    m->seed = std::strtoull(sd.c_str(), nullptr, 10);
    return true;
}

// save_instance (io.cpp:86-125): A.csv row-major (one observation per line),
// y.csv, truth.csv "x,xi" with a "# x,xi" header (only with ground truth),
// meta.json.  A is M x N column-major.
inline bool save_bundle(const fs::path& dir, const Meta& m, const double* A, const double* y,
                        const double* x, const int32_t* xi, std::string* err) {
    std::error_code ec;
    fs::create_directories(dir, ec);
    std::string s;
    s.reserve((size_t)m.M * m.N * 20);
    for (int k = 0; k < m.M; ++k) {
        for (int r = 0; r < m.N; ++r) {
            if (r) s += ',';
            s += fmt_double(A[(size_t)r * m.M + k]);
        }
        s += '\n';
    }
    if (!put_file(dir / "A.csv", s, err)) return false;
    s.clear();
    for (int k = 0; k < m.M; ++k) (s += fmt_double(y[k])) += '\n';
    if (!put_file(dir / "y.csv", s, err)) return false;
    if (x && xi) {
        s = "# x,xi\n";
        for (int r = 0; r < m.N; ++r) ((s += fmt_double(x[r])) += ',') += std::to_string(xi[r]) + "\n";
        if (!put_file(dir / "truth.csv", s, err)) return false;
    }
    return put_file(dir / "meta.json", meta_json(m), err);
}

// load_instance (io.cpp:127-167), phase 1: meta + whether truth.csv exists.
inline bool load_meta(const fs::path& dir, Meta* m, bool* truth, std::string* err) {
    std::string t;
    if (!get_file(dir / "meta.json", &t, err) || !parse_meta(t, m, err)) return false;
    if (m->N < 1 || m->M < 1) {
        *err = "meta.json: bad N/M";
        return false;
    }
    *truth = fs::exists(dir / "truth.csv");
    return true;
}

// phase 2: the arrays, with the reference's row/column count checks.
inline bool load_arrays(const fs::path& dir, const Meta& m, double* A, double* y, double* x,
                        int32_t* xi, std::string* err) {
    std::string t;
    if (!get_file(dir / "A.csv", &t, err)) return false;
    bool bad_cols = false;
    size_t n = scan_rows(t, [&](size_t k, const std::vector<double>& v) {
        if ((int)k >= m.M) return;
        if ((int)v.size() != m.N) {
            bad_cols = true;
            return;
        }
        for (int r = 0; r < m.N; ++r) A[(size_t)r * m.M + k] = v[r];
    });
    if ((int)n != m.M) {
        *err = "A.csv row count does not match meta.json";
        return false;
    }
    if (bad_cols) {
        *err = "A.csv column count does not match meta.json";
        return false;
    }
    if (!get_file(dir / "y.csv", &t, err)) return false;
    n = scan_rows(t, [&](size_t k, const std::vector<double>& v) {
        if ((int)k < m.M) y[k] = v[0];
    });
    if ((int)n != m.M) {
        *err = "y.csv row count mismatch";
        return false;
    }
    if (x && xi && fs::exists(dir / "truth.csv")) {
        if (!get_file(dir / "truth.csv", &t, err)) return false;
        bool short_row = false;
        n = scan_rows(t, [&](size_t r, const std::vector<double>& v) {
            if ((int)r >= m.N) return;
            if (v.size() < 2) {
                short_row = true;
                return;
            }
            x[r] = v[0];
            xi[r] = (int32_t)v[1];
        });
        if ((int)n != m.N || short_row) {
            *err = "truth.csv row count mismatch";
            return false;
        }
    }
    return true;
}

// CsvWriter (io.hpp:31-48, io.cpp:169-196): "# " comment lines, the header,
// then rows of exactly as many cells; the text is written on close.
struct Csv {
    std::string path, buf;
    size_t ncols = 0;
};

}  // namespace cimcs_io
