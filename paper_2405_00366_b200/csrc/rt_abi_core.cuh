// rt_abi_core.cuh -- part of the single runtime TU (runtime.cu includes the parts in
// order): C ABI: version, errors, hyper-parameters, orders, instance generation,
// bundles / CSV.
#pragma once

extern "C" {

// =================================================================== C ABI

int cimcs_abi_version(void) { return CIMCS_ABI_VERSION; }
const char* cimcs_last_error(void) { return g_err.c_str(); }

void cimcs_hyper_default(cimcs_hyper* h) {
    h->g2 = 1e-7;
    h->j = 1.0;
    h->K = 1.0;
    h->beta = 0.2;
    h->tau = 1.0;
    h->dt = 0.02;
    h->n_steps = 1000;
    h->p_thr = 1.0;
    h->d = 0.4;
    h->eta_init = 0.8;
    h->eta_end = 0.18;
    h->velo = 51;
    h->dt_c = 0.1;
    h->jacobi_iters = 100;
    h->cg_max_iters = 10000;
    h->cg_tol = 1e-10;
    h->gamma = 1e-4;
    h->mfz_loss_minus_j = 0;
    h->mu_abort = 100.0;
    h->pump_kind = CIMCS_PUMP_SIGMOID;
    h->pump_end = 1.2;
}

int cimcs_hyper_validate(const cimcs_hyper* h) { return validate(h); }
uint64_t cimcs_mix_seed(uint64_t base, uint64_t salt) { return mix_seed(base, salt); }

int cimcs_gemv_order(int dtype, int32_t* nseg, int32_t* gran) {
    (void)dtype;
    if (nseg) *nseg = kSeg;
    if (gran) *gran = kGran;
    return 0;
}

// The fp64 contraction order of the resident problem set (ORC_CANON's
// (nseg, gran)): the DMMA symmetric path sums 512-column segments, the grid and
// cluster kernels 8 interleaved segments of 8-column granules.
int cimcs_canon_order(const cimcs_ctx* c, int32_t* nseg, int32_t* gran) {
    if (!c || c->B < 1) return fail(CIMCS_INPUT_ERROR, "no problems set");
    const bool s64 = c->sym64;
    if (nseg) *nseg = s64 ? c->nSB6 : kSeg;
    if (gran) *gran = s64 ? kT6Seg : kGran;
    return 0;
}

int cimcs_gen_dims(int32_t N, double alpha, double a, int32_t* M, int32_t* K) {
    int m = 0, k = 0;
    if (gen_dims(N, alpha, a, &m, &k)) return fail(CIMCS_INPUT_ERROR, "gen_instance: bad dims");
    if (M) *M = m;
    if (K) *K = k;
    return 0;
}

// ------------------------------------------------ bundles and CSV (io.hpp)
int cimcs_format_double(double v, char* buf, int32_t cap) {
    const std::string s = cimcs_io::fmt_double(v);
    if (!buf || cap < (int32_t)s.size() + 1) return fail(CIMCS_INPUT_ERROR, "format_double: buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return 0;
}

uint64_t cimcs_fnv1a64(const char* bytes, uint64_t n) {
    return cimcs_io::fnv1a(reinterpret_cast<const unsigned char*>(bytes), (size_t)n);
}

int cimcs_save_instance(const char* dir, int32_t N, int32_t M, const double* A, const double* y,
                        const double* x_true, const int32_t* xi_true, double a, double alpha,
                        double nu, uint64_t seed) {
    if (!dir || N < 1 || M < 1 || !A || !y) return fail(CIMCS_INPUT_ERROR, "save_instance: bad arguments");
    cimcs_io::Meta m;
    m.N = N;
    m.M = M;
    m.a = a;
    m.alpha = alpha;
    m.nu = nu;
    m.seed = seed;
    std::string err;
    if (!cimcs_io::save_bundle(dir, m, A, y, x_true, xi_true, &err)) return fail(CIMCS_INPUT_ERROR, err);
    return 0;
}

int cimcs_load_instance(const char* dir, int32_t* N, int32_t* M, int32_t* has_truth, double* a,
                        double* alpha, double* nu, uint64_t* seed, double* A, double* y,
                        double* x_true, int32_t* xi_true) {
    if (!dir || !N || !M) return fail(CIMCS_INPUT_ERROR, "load_instance: bad arguments");
    cimcs_io::Meta m;
    bool truth = false;
    std::string err;
    if (!cimcs_io::load_meta(dir, &m, &truth, &err)) return fail(CIMCS_INPUT_ERROR, err);
    if (A) {  // phase 2: the caller sized the arrays from phase 1
        if (*N != m.N || *M != m.M) return fail(CIMCS_INPUT_ERROR, "load_instance: size mismatch");
        if (!y || !cimcs_io::load_arrays(dir, m, A, y, truth ? x_true : nullptr,
                                         truth ? xi_true : nullptr, &err))
            return fail(CIMCS_INPUT_ERROR, err.empty() ? "load_instance: bad arguments" : err);
    }
    *N = m.N;
    *M = m.M;
    if (has_truth) *has_truth = truth ? 1 : 0;
    if (a) *a = m.a;
    if (alpha) *alpha = m.alpha;
    if (nu) *nu = m.nu;
    if (seed) *seed = m.seed;
    return 0;
}

struct cimcs_csv : cimcs_io::Csv {};

int cimcs_csv_open(const char* path, const char* const* comments, int32_t ncomments,
                   const char* const* columns, int32_t ncols, cimcs_csv** out) {
    if (!path || !out || ncols < 0 || ncomments < 0) return fail(CIMCS_INPUT_ERROR, "csv_open: bad arguments");
    auto* w = new cimcs_csv();
    w->path = path;
    w->ncols = (size_t)ncols;
    for (int k = 0; k < ncomments; ++k) (w->buf += "# ") += std::string(comments[k]) + "\n";
    for (int k = 0; k < ncols; ++k) {
        if (k) w->buf += ',';
        w->buf += columns[k];
    }
    w->buf += '\n';
    *out = w;
    return 0;
}

int cimcs_csv_row(cimcs_csv* w, const char* const* cells, int32_t n) {
    if (!w || n < 0 || (size_t)n != w->ncols) return fail(CIMCS_INPUT_ERROR, "CsvWriter: cell count mismatch");
    for (int k = 0; k < n; ++k) {
        if (k) w->buf += ',';
        w->buf += cells[k];
    }
    w->buf += '\n';
    return 0;
}

int cimcs_csv_close(cimcs_csv* w) {
    if (!w) return 0;
    std::error_code ec;
    const std::filesystem::path p(w->path);
    std::filesystem::create_directories(p.parent_path().empty() ? "." : p.parent_path(), ec);
    std::string err;
    const bool ok = cimcs_io::put_file(p, w->buf, &err);
    delete w;
    return ok ? 0 : fail(CIMCS_INPUT_ERROR, err);
}

int cimcs_gen_instance(int32_t N, double alpha, double a, double nu, uint64_t seed, double* A,
                       double* y, double* x_true, int32_t* xi_true) {
    if (gen_instance(N, alpha, a, nu, seed, A, y, x_true, xi_true))
        return fail(CIMCS_INPUT_ERROR, "gen_instance: bad arguments");
    return 0;
}

int cimcs_gen_instances(int32_t B, int32_t N, const double* alpha, const double* a,
                        const double* nu, const uint64_t* seeds, double* const* A,
                        double* const* y, double* const* x_true, int32_t* const* xi_true,
                        int32_t threads) {
    std::atomic<int> next{0}, bad{0};
    if (threads <= 0) threads = (int)std::thread::hardware_concurrency();
    // fewer instances than threads: the spare threads transform each instance's A
    const int inner = std::max(1, threads / std::max(1, B));
    auto work = [&] {
        for (int b = next.fetch_add(1); b < B; b = next.fetch_add(1))
            if (gen_instance(N, alpha[b], a[b], nu[b], seeds[b], A[b], y[b], x_true[b],
                             xi_true[b], inner))
                bad = 1;
    };
    threads = std::max(1, std::min<int>(threads, B));
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(work);
    for (auto& th : pool) th.join();
    return bad ? fail(CIMCS_INPUT_ERROR, "gen_instance: bad arguments") : 0;
}

}  // extern "C"
