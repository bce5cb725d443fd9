// es_oracle.cpp — CPU FP64 restatement of the eventscope GMM hot path.
//
// TEST INFRASTRUCTURE ONLY (see es_oracle.h).  Every function follows the
// SPEC text it cites; nothing here is shared with the CUDA product.
//
// Algorithm sources:
//   densities          SPEC.md:261-279, PAPER.md:132,171 (Def. 1 density)
//   responsibilities   SPEC.md:281-289, Alg. 1 line 6
//   EM
//   BIC
//   detect             SPEC.md:357-365, 388-396; PAPER.md:183-199 (Alg. 2)
//   calibrate
//   errors             proj/include/eventscope/errors.hpp:13-37
//
// Determinism: rows are processed in fixed chunks of
// kChunk rows; per-chunk partial sums are combined in chunk order, so the
// result does not depend on the OpenMP thread count.

#include "es_oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

constexpr int64_t kChunk = 4096;
constexpr double kLog2Pi = 1.8378770664093454835606594728112;  // log(2*pi)

thread_local std::string g_err_name;
thread_local std::string g_err_msg;

enum Status { kOk = 0, kData = 1, kNumeric = 2, kIo = 3 };

int fail(int kind, const char* name, const std::string& msg) {
    g_err_name = name;
    g_err_msg = msg;
    return kind;
}

void set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
}

// ---------------------------------------------------------------- PRNG ----
// SplitMix64: host-side draws (init rows, collapse reseeds, k-means++).
struct SplitMix64 {
    uint64_t s;
    explicit SplitMix64(uint64_t seed) : s(seed) {}
    uint64_t next() {
        uint64_t z = (s += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    uint64_t below(uint64_t n) { return (uint64_t)(((unsigned __int128)next() * n) >> 64); }
    double uniform() { return (double)(next() >> 11) * 0x1.0p-53; }
};

// ------------------------------------------------------ dense helpers ----
// Lower Cholesky factor of a D x D SPD matrix (row-major). false if not PD.
// "Not PD" (SingularCovariance) is numerical: a pivot at or below
// D * 2^-46 of its diagonal entry (condition number beyond ~1e13 / D) counts as
// singular, so that an exactly rank-deficient covariance is rejected whatever
// the sign of the rounding noise in its pivots.
bool cholesky(const double* A, int D, double* L) {
    std::fill(L, L + (size_t)D * D, 0.0);
    for (int j = 0; j < D; ++j) {
        double s = A[(size_t)j * D + j];
        for (int p = 0; p < j; ++p) s -= L[(size_t)j * D + p] * L[(size_t)j * D + p];
        if (!(s > std::ldexp((double)D, -46) * A[(size_t)j * D + j]) || !std::isfinite(s)) return false;
        double ljj = std::sqrt(s);
        L[(size_t)j * D + j] = ljj;
        for (int i = j + 1; i < D; ++i) {
            double t = A[(size_t)i * D + j];
            for (int p = 0; p < j; ++p) t -= L[(size_t)i * D + p] * L[(size_t)j * D + p];
            L[(size_t)i * D + j] = t / ljj;
        }
    }
    return true;
}

// Factored model: per component L_k (Cholesky of Sigma_k) and log constants.
struct Factored {
    int K = 0, D = 0;
    std::vector<double> L;        // K*D*D
    std::vector<double> lognorm;  // -0.5*logdet - 0.5*D*log(2pi)
    std::vector<double> logpi;
    const double* mu = nullptr;
};

int factor(const double* pi, const double* mu, const double* cov, int K, int D, Factored& f) {
    f.K = K;
    f.D = D;
    f.mu = mu;
    f.L.assign((size_t)K * D * D, 0.0);
    f.lognorm.assign(K, 0.0);
    f.logpi.assign(K, 0.0);
    for (int k = 0; k < K; ++k) {
        double* Lk = f.L.data() + (size_t)k * D * D;
        if (!cholesky(cov + (size_t)k * D * D, D, Lk))
            return fail(kNumeric, "SingularCovariance",
                        "covariance of component " + std::to_string(k) + " is not positive definite");
        double logdet = 0.0;
        for (int d = 0; d < D; ++d) logdet += std::log(Lk[(size_t)d * D + d]);
        logdet *= 2.0;
        f.lognorm[k] = -0.5 * logdet - 0.5 * D * kLog2Pi;
        f.logpi[k] = std::log(pi[k]);
    }
    return kOk;
}

// log N(x | mu_k, Sigma_k) by forward substitution L z = x - mu.
double log_normal(const Factored& f, const double* x, int k, double* z) {
    const int D = f.D;
    const double* Lk = f.L.data() + (size_t)k * D * D;
    const double* mk = f.mu + (size_t)k * D;
    double q = 0.0;
    for (int r = 0; r < D; ++r) {
        double t = x[r] - mk[r];
        for (int j = 0; j < r; ++j) t -= Lk[(size_t)r * D + j] * z[j];
        z[r] = t / Lk[(size_t)r * D + r];
        q += z[r] * z[r];
    }
    return f.lognorm[k] - 0.5 * q;
}

struct RowScore {
    double ll;        // log-sum-exp over k of log pi_k + log N_ik
    int predict;      // argmax weighted
    int best;         // argmax unweighted
    double best_ld;   // log N_{i,best}
};

// Scores one row; w (K) receives log pi_k + log N_ik.
RowScore score_row(const Factored& f, const double* x, double* w, double* z) {
    RowScore r{};
    double m = -std::numeric_limits<double>::infinity();
    double bl = -std::numeric_limits<double>::infinity();
    r.predict = 0;
    r.best = 0;
    for (int k = 0; k < f.K; ++k) {
        double ln = log_normal(f, x, k, z);
        w[k] = f.logpi[k] + ln;
        if (w[k] > m) { m = w[k]; r.predict = k; }       // strict > : ties -> lowest k
        if (ln > bl) { bl = ln; r.best = k; }
    }
    double s = 0.0;
    for (int k = 0; k < f.K; ++k) s += std::exp(w[k] - m);  // max-shift
    r.ll = m + std::log(s);
    r.best_ld = bl;
    return r;
}

bool all_finite(const double* X, int64_t n) {
    for (int64_t i = 0; i < n; ++i)
        if (!std::isfinite(X[i])) return false;
    return true;
}

int64_t nchunks(int64_t N) { return (N + kChunk - 1) / kChunk; }

void data_stats(const double* X, int64_t N, int D, double* mean, double* S, double* mn, double* mx) {
    const int64_t C = nchunks(N);
    std::vector<double> part_sum((size_t)C * D, 0.0);
    std::vector<double> part_min((size_t)C * D), part_max((size_t)C * D);
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < C; ++c) {
        double* ps = &part_sum[(size_t)c * D];
        double* pmn = &part_min[(size_t)c * D];
        double* pmx = &part_max[(size_t)c * D];
        for (int d = 0; d < D; ++d) { pmn[d] = INFINITY; pmx[d] = -INFINITY; }
        for (int64_t i = c * kChunk; i < std::min(N, (c + 1) * kChunk); ++i)
            for (int d = 0; d < D; ++d) {
                double v = X[(size_t)i * D + d];
                ps[d] += v;
                pmn[d] = std::min(pmn[d], v);
                pmx[d] = std::max(pmx[d], v);
            }
    }
    for (int d = 0; d < D; ++d) { mean[d] = 0.0; mn[d] = INFINITY; mx[d] = -INFINITY; }
    for (int64_t c = 0; c < C; ++c)
        for (int d = 0; d < D; ++d) {
            mean[d] += part_sum[(size_t)c * D + d];
            mn[d] = std::min(mn[d], part_min[(size_t)c * D + d]);
            mx[d] = std::max(mx[d], part_max[(size_t)c * D + d]);
        }
    for (int d = 0; d < D; ++d) mean[d] /= (double)N;
    // second pass: centered covariance (biased, 1/N)
    std::vector<double> part_S((size_t)C * D * D, 0.0);
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < C; ++c) {
        double* pS = &part_S[(size_t)c * D * D];
        std::vector<double> y(D);
        for (int64_t i = c * kChunk; i < std::min(N, (c + 1) * kChunk); ++i) {
            for (int d = 0; d < D; ++d) y[d] = X[(size_t)i * D + d] - mean[d];
            for (int a = 0; a < D; ++a)
                for (int b = a; b < D; ++b) pS[(size_t)a * D + b] += y[a] * y[b];
        }
    }
    std::fill(S, S + (size_t)D * D, 0.0);
    for (int64_t c = 0; c < C; ++c)
        for (int a = 0; a < D; ++a)
            for (int b = a; b < D; ++b) S[(size_t)a * D + b] += part_S[(size_t)c * D * D + (size_t)a * D + b];
    for (int a = 0; a < D; ++a)
        for (int b = a; b < D; ++b) {
            S[(size_t)a * D + b] /= (double)N;
            S[(size_t)b * D + a] = S[(size_t)a * D + b];
        }
}

double default_reg(const double* S, int D) {
    double tr = 0.0;
    for (int d = 0; d < D; ++d) tr += S[(size_t)d * D + d];
    return 1e-6 * tr / D;
}

bool degenerate(const double* mn, const double* mx, int D) {
    for (int d = 0; d < D; ++d)
        if (mn[d] != mx[d]) return false;
    return true;
}

void set_cov_to(double* covk, const double* S, int D, double reg, bool diag = false) {
    for (int a = 0; a < D; ++a)
        for (int b = 0; b < D; ++b)
            covk[(size_t)a * D + b] = (diag && a != b) ? 0.0 : S[(size_t)a * D + b] + (a == b ? reg : 0.0);
}

// k-means++ seeding: first centre uniform, then
// D^2-weighted draws with the cumulative sum taken in row order.
void kmeanspp_rows(const double* X, int64_t N, int D, int K, SplitMix64& rng, std::vector<int64_t>& rows) {
    rows.clear();
    rows.push_back((int64_t)rng.below((uint64_t)N));
    std::vector<double> d2(N, INFINITY);
    const int64_t C = nchunks(N);
    std::vector<double> part(C);
    for (int j = 1; j < K; ++j) {
        const double* c = X + (size_t)rows.back() * D;
#pragma omp parallel for schedule(static)
        for (int64_t ch = 0; ch < C; ++ch) {
            double s = 0.0;
            for (int64_t i = ch * kChunk; i < std::min(N, (ch + 1) * kChunk); ++i) {
                double t = 0.0;
                for (int d = 0; d < D; ++d) {
                    double e = X[(size_t)i * D + d] - c[d];
                    t += e * e;
                }
                d2[i] = std::min(d2[i], t);
                s += d2[i];
            }
            part[ch] = s;
        }
        double total = 0.0;
        for (int64_t ch = 0; ch < C; ++ch) total += part[ch];
        double r = rng.uniform() * total;
        int64_t pick = N - 1;
        if (total > 0.0) {
            // locate chunk, then row, with the same chunked cumulative order
            double acc = 0.0;
            int64_t ch = 0;
            for (; ch < C; ++ch) {
                if (acc + part[ch] > r) break;
                acc += part[ch];
            }
            if (ch == C) ch = C - 1;
            double acc2 = acc;
            for (int64_t i = ch * kChunk; i < std::min(N, (ch + 1) * kChunk); ++i) {
                acc2 += d2[i];
                if (acc2 > r) { pick = i; break; }
            }
        } else {
            pick = (int64_t)rng.below((uint64_t)N);
        }
        rows.push_back(pick);
    }
}

}  // namespace

// =================================================================== API ===
extern "C" {

const char* eso_last_error_name(void) { return g_err_name.c_str(); }
const char* eso_last_error_message(void) { return g_err_msg.c_str(); }

int eso_component_log_density(const double* pi, const double* mu, const double* cov, int K, int D,
                              const double* x, int k, double* out) {
    if (k < 0 || k >= K) return fail(kData, "DimensionMismatch", "component index out of range");
    if (D <= 0) return fail(kData, "DimensionMismatch", "dimension must be positive");
    Factored f;
    if (int s = factor(pi, mu, cov, K, D, f)) return s;
    std::vector<double> z(D);
    *out = log_normal(f, x, k, z.data());
    return kOk;
}

int eso_mixture_log_density(const double* pi, const double* mu, const double* cov, int K, int D,
                            const double* x, double* out) {
    Factored f;
    if (int s = factor(pi, mu, cov, K, D, f)) return s;
    std::vector<double> z(D), w(K);
    *out = score_row(f, x, w.data(), z.data()).ll;
    return kOk;
}

int eso_score(const double* X, int64_t N, int D, const double* pi, const double* mu, const double* cov,
              int K, double* ll, int32_t* predict, int32_t* best_k, double* best_logdens, double* gamma,
              int nthreads) {
    set_threads(nthreads);
    Factored f;
    if (int s = factor(pi, mu, cov, K, D, f)) return s;
#pragma omp parallel
    {
        std::vector<double> z(D), w(K);
#pragma omp for schedule(static)
        for (int64_t i = 0; i < N; ++i) {
            RowScore r = score_row(f, X + (size_t)i * D, w.data(), z.data());
            if (ll) ll[i] = r.ll;
            if (predict) predict[i] = r.predict;
            if (best_k) best_k[i] = r.best;
            if (best_logdens) best_logdens[i] = r.best_ld;
            if (gamma)
                for (int k = 0; k < K; ++k) gamma[(size_t)i * K + k] = std::exp(w[k] - r.ll);
        }
    }
    return kOk;
}

int eso_data_stats(const double* X, int64_t N, int D, double* mean, double* S, double* colmin,
                   double* colmax, int nthreads) {
    if (N < 1) return fail(kData, "TooFewPoints", "empty matrix");
    set_threads(nthreads);
    data_stats(X, N, D, mean, S, colmin, colmax);
    return kOk;
}

int eso_random_init(const double* X, int64_t N, int D, int K, uint64_t seed, double reg, double* pi,
                    double* mu, double* cov, double* reg_used) {
    if (K < 1 || N < K) return fail(kData, "TooFewPoints", "need N >= K >= 1");
    std::vector<double> mean(D), S((size_t)D * D), mn(D), mx(D);
    data_stats(X, N, D, mean.data(), S.data(), mn.data(), mx.data());
    if (reg < 0) reg = default_reg(S.data(), D);
    SplitMix64 rng(seed);
    std::vector<int64_t> rows;
    while ((int)rows.size() < K) {
        int64_t r = (int64_t)rng.below((uint64_t)N);
        if (std::find(rows.begin(), rows.end(), r) == rows.end()) rows.push_back(r);
    }
    for (int k = 0; k < K; ++k) {
        pi[k] = 1.0 / K;
        std::memcpy(mu + (size_t)k * D, X + (size_t)rows[k] * D, sizeof(double) * D);
        set_cov_to(cov + (size_t)k * D * D, S.data(), D, reg);
    }
    if (reg_used) *reg_used = reg;
    return kOk;
}

}  // extern "C"

namespace {

// Work buffers of one EM iteration (gamma N x K and the chunk partials).
struct EmWork {
    std::vector<double> gamma, part_ll, part_nk, part_s1, part_s2;
    void size(int64_t N, int D, int K) {
        const int64_t C = nchunks(N);
        gamma.resize((size_t)N * K);
        part_ll.resize(C);
        part_nk.resize((size_t)C * K);
        part_s1.resize((size_t)C * K * D);
        part_s2.resize((size_t)C * K * D * D);
    }
};

// E-step: gamma (when kept) and logL = sum_i ll_i(theta), rows in
// chunks, chunk partials summed in chunk order.
int em_estep(const double* X, int64_t N, int D, int K, const double* pi, const double* mu, const double* cov,
             EmWork& w, bool keep_gamma, double& logL) {
    Factored f;
    if (int s = factor(pi, mu, cov, K, D, f)) return s;
    const int64_t C = nchunks(N);
#pragma omp parallel
    {
        std::vector<double> z(D), wk(K);
#pragma omp for schedule(static)
        for (int64_t c = 0; c < C; ++c) {
            double s = 0.0;
            for (int64_t i = c * kChunk; i < std::min(N, (c + 1) * kChunk); ++i) {
                RowScore r = score_row(f, X + (size_t)i * D, wk.data(), z.data());
                s += r.ll;
                if (keep_gamma)
                    for (int k = 0; k < K; ++k) w.gamma[(size_t)i * K + k] = std::exp(wk[k] - r.ll);
            }
            w.part_ll[c] = s;
        }
    }
    logL = 0.0;
    for (int64_t c = 0; c < C; ++c) logL += w.part_ll[c];
    return kOk;
}

// M-step, literal two-pass form of SPEC.md:294 (mean first, then the covariance about the
// NEW mean); Nk receives sum_i gamma_ik.  Collapse handling is the caller's.
void em_mstep(const double* X, int64_t N, int D, int K, double reg, bool diag, double* pi, double* mu, double* cov,
              EmWork& w, std::vector<double>& Nk) {
    const int64_t C = nchunks(N);
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < C; ++c) {
        double* nk = &w.part_nk[(size_t)c * K];
        double* s1 = &w.part_s1[(size_t)c * K * D];
        std::fill(nk, nk + K, 0.0);
        std::fill(s1, s1 + (size_t)K * D, 0.0);
        for (int64_t i = c * kChunk; i < std::min(N, (c + 1) * kChunk); ++i)
            for (int k = 0; k < K; ++k) {
                double g = w.gamma[(size_t)i * K + k];
                nk[k] += g;
                for (int d = 0; d < D; ++d) s1[(size_t)k * D + d] += g * X[(size_t)i * D + d];
            }
    }
    Nk.assign(K, 0.0);
    for (int64_t c = 0; c < C; ++c)
        for (int k = 0; k < K; ++k) Nk[k] += w.part_nk[(size_t)c * K + k];
    for (int k = 0; k < K; ++k) {
        for (int d = 0; d < D; ++d) {
            double s = 0.0;
            for (int64_t c = 0; c < C; ++c) s += w.part_s1[(size_t)c * K * D + (size_t)k * D + d];
            mu[(size_t)k * D + d] = Nk[k] > 0 ? s / Nk[k] : mu[(size_t)k * D + d];
        }
        pi[k] = Nk[k] / (double)N;
    }
#pragma omp parallel
    {
        std::vector<double> y(D);
#pragma omp for schedule(static)
        for (int64_t c = 0; c < C; ++c) {
            double* s2 = &w.part_s2[(size_t)c * K * D * D];
            std::fill(s2, s2 + (size_t)K * D * D, 0.0);
            for (int64_t i = c * kChunk; i < std::min(N, (c + 1) * kChunk); ++i)
                for (int k = 0; k < K; ++k) {
                    double g = w.gamma[(size_t)i * K + k];
                    for (int d = 0; d < D; ++d) y[d] = X[(size_t)i * D + d] - mu[(size_t)k * D + d];
                    for (int a = 0; a < D; ++a)
                        for (int b = a; b < (diag ? a + 1 : D); ++b)
                            s2[(size_t)k * D * D + (size_t)a * D + b] += g * y[a] * y[b];
                }
        }
    }
    for (int k = 0; k < K; ++k) {
        double* ck = cov + (size_t)k * D * D;
        for (int a = 0; a < D; ++a)
            for (int b = a; b < D; ++b) {
                double s = 0.0;
                for (int64_t c = 0; c < C; ++c)
                    s += w.part_s2[(size_t)c * K * D * D + (size_t)k * D * D + (size_t)a * D + b];
                double v = Nk[k] > 0 ? s / Nk[k] : 0.0;
                if (diag && a != b) v = 0.0;
                ck[(size_t)a * D + b] = v + (a == b ? reg : 0.0);
                ck[(size_t)b * D + a] = ck[(size_t)a * D + b];
            }
    }
}

}  // namespace

extern "C" {

int eso_fit_em(const double* X, int64_t N, int D, int K, const eso_fit_opts* opts, const double* pi_init,
               const double* mu_init, const double* cov_init, double* pi, double* mu, double* cov,
               eso_fit_report* rep, double* per_iter) {
    // ---- validation
    if (K < 1 || N < K) return fail(kData, "TooFewPoints", "fit_em requires N >= K >= 1");
    if (D < 1) return fail(kData, "DimensionMismatch", "dimension must be positive");
    if (!all_finite(X, N * D)) return fail(kData, "NonFiniteInput", "X contains non-finite entries");
    set_threads(opts->nthreads);
    std::vector<double> mean(D), S((size_t)D * D), mn(D), mx(D);
    data_stats(X, N, D, mean.data(), S.data(), mn.data(), mx.data());
    if (K > 1 && degenerate(mn.data(), mx.data(), D))
        return fail(kData, "DegenerateData", "all points identical and K > 1");
    const double reg = opts->reg < 0 ? default_reg(S.data(), D) : opts->reg;
    const bool diag = opts->cov_type == 1;  // diagonal extension: same M-step restricted to diag(Sigma)

    // ---- init
    SplitMix64 rng(opts->seed);
    if (opts->init == 2) {
        std::memcpy(pi, pi_init, sizeof(double) * K);
        std::memcpy(mu, mu_init, sizeof(double) * K * D);
        std::memcpy(cov, cov_init, sizeof(double) * K * D * D);
    } else {
        std::vector<int64_t> rows;
        if (opts->init == 1) {
            kmeanspp_rows(X, N, D, K, rng, rows);
        } else {
            while ((int)rows.size() < K) {
                int64_t r = (int64_t)rng.below((uint64_t)N);
                if (std::find(rows.begin(), rows.end(), r) == rows.end()) rows.push_back(r);
            }
        }
        for (int k = 0; k < K; ++k) {
            pi[k] = 1.0 / K;
            std::memcpy(mu + (size_t)k * D, X + (size_t)rows[k] * D, sizeof(double) * D);
            set_cov_to(cov + (size_t)k * D * D, S.data(), D, reg, diag);
        }
    }

    EmWork w;
    w.size(N, D, K);
    std::vector<double> Nk;
    int collapses = 0;
    int iterations = 0;
    bool converged = false;
    int nrec = 0;
    double prev = 0.0, cur = 0.0;

    for (int t = 0; t < opts->max_iter; ++t) {
        // ---- E-step: gamma and logL_t = sum_i ll_i(theta_t)
        if (int s = em_estep(X, N, D, K, pi, mu, cov, w, true, cur)) return s;
        per_iter[nrec++] = cur;
        if (t >= 1 && std::fabs(cur - prev) < opts->tol * (1.0 + std::fabs(cur))) {
            converged = true;  // theta_t is returned; final logL = logL_t
            break;
        }
        prev = cur;
        // ---- M-step, literal two-pass form of SPEC.md:294
        em_mstep(X, N, D, K, reg, diag, pi, mu, cov, w, Nk);
        // ---- collapse handling: N*pi_k < 1 -> reseed
        bool any = false;
        for (int k = 0; k < K; ++k) {
            if (Nk[k] < 1.0) {
                if (++collapses > 2)
                    return fail(kNumeric, "RepeatedCollapse", "component collapsed more than twice");
                int64_t r = (int64_t)rng.below((uint64_t)N);
                std::memcpy(mu + (size_t)k * D, X + (size_t)r * D, sizeof(double) * D);
                set_cov_to(cov + (size_t)k * D * D, S.data(), D, reg, diag);
                pi[k] = 1.0 / K;
                any = true;
            }
        }
        if (any) {
            double z = 0.0;
            for (int k = 0; k < K; ++k) z += pi[k];
            for (int k = 0; k < K; ++k) pi[k] /= z;
        }
        iterations = t + 1;
    }
    double final_ll = cur;
    if (!converged) {
        if (int s = em_estep(X, N, D, K, pi, mu, cov, w, false, final_ll)) return s;
    }
    if (rep) {
        rep->iterations = iterations;
        rep->final_log_likelihood = final_ll;
        rep->converged = converged ? 1 : 0;
        rep->seed = opts->seed;
        rep->n_per_iter = nrec;
        rep->collapses = collapses;
        rep->reg_used = reg;
    }
    return kOk;
}

// One EM iteration in place (bench.py --impl reference: the timed unit of the metric): the
// E-step of fit_em and its literal two-pass M-step, no collapse reseed (collapsed components
// are counted in *n_collapsed).  Work buffers persist per thread across calls.
int eso_em_step(const double* X, int64_t N, int D, int K, double reg, int cov_type, double* pi, double* mu,
                double* cov, double* logL, int* n_collapsed, int nthreads) {
    if (K < 1 || N < K) return fail(kData, "TooFewPoints", "em_step requires N >= K >= 1");
    set_threads(nthreads);
    static thread_local EmWork w;
    w.size(N, D, K);
    std::vector<double> Nk;
    double ll = 0.0;
    if (int s = em_estep(X, N, D, K, pi, mu, cov, w, true, ll)) return s;
    em_mstep(X, N, D, K, reg, cov_type == 1, pi, mu, cov, w, Nk);
    if (logL) *logL = ll;
    if (n_collapsed) {
        int c = 0;
        for (int k = 0; k < K; ++k) c += Nk[k] < 1.0;
        *n_collapsed = c;
    }
    return kOk;
}

int eso_detect(const double* X, int64_t N, int D, const double* pi, const double* mu, const double* cov, int K,
               double log_delta, int mode, uint8_t* flags, int32_t* best_k, double* best_logdens,
               int64_t* n_flagged, int nthreads) {
    set_threads(nthreads);
    Factored f;
    if (int s = factor(pi, mu, cov, K, D, f)) return s;
    int64_t cnt = 0;
#pragma omp parallel
    {
        std::vector<double> z(D), w(K);
#pragma omp for schedule(static) reduction(+ : cnt)
        for (int64_t i = 0; i < N; ++i) {
            RowScore r = score_row(f, X + (size_t)i * D, w.data(), z.data());
            double v = mode == 1 ? r.ll : r.best_ld;
            uint8_t fl = v < log_delta ? 1 : 0;  // strict '<'
            if (flags) flags[i] = fl;
            if (best_k) best_k[i] = r.best;
            if (best_logdens) best_logdens[i] = r.best_ld;
            cnt += fl;
        }
    }
    if (n_flagged) *n_flagged = cnt;
    return kOk;
}

int eso_calibrate(const double* X, int64_t n_train, int D, const double* pi, const double* mu, const double* cov,
                  int K, double q, int mode, double* delta, double* log_delta, int nthreads) {
    if (n_train < 1) return fail(kData, "EmptyTraining", "training split is empty");
    if (!(q > 0.0 && q < 1.0)) return fail(kData, "RangeViolation", "q must be in (0,1)");
    set_threads(nthreads);
    Factored f;
    if (int s = factor(pi, mu, cov, K, D, f)) return s;
    std::vector<double> v(n_train);
#pragma omp parallel
    {
        std::vector<double> z(D), w(K);
#pragma omp for schedule(static)
        for (int64_t i = 0; i < n_train; ++i) {
            RowScore r = score_row(f, X + (size_t)i * D, w.data(), z.data());
            v[i] = mode == 1 ? r.ll : r.best_ld;  // log densities; exp is monotone
        }
    }
    // q-quantile with linear interpolation between order statistics, h = (n-1) q
    const double h = (double)(n_train - 1) * q;
    const int64_t lo = (int64_t)std::floor(h);
    const int64_t hi = std::min<int64_t>(lo + 1, n_train - 1);
    std::nth_element(v.begin(), v.begin() + lo, v.end());
    const double vlo = v[lo];
    double vhi = vlo;
    if (hi != lo) vhi = *std::min_element(v.begin() + lo + 1, v.end());
    const double dlo = std::exp(vlo), dhi = std::exp(vhi);  // interpolate in density space
    const double frac = h - (double)lo;
    double d = dlo + frac * (dhi - dlo);
    *delta = d;
    // log delta computed once and shared by every comparison;
    // exact endpoints keep their log so no exp/log round trip moves a flag.
    *log_delta = (d == dlo) ? vlo : (d == dhi) ? vhi : std::log(d);
    return kOk;
}


// k-means baseline (eval-bench): k-means++ seeding as fit_em's, Lloyd's
// algorithm on the train split (first floor(train_window N) rows) until no assignment
// changes or max_iter steps (<= 0: 100); empty clusters keep their centroid; distance
// squared as an FMA chain over features in order (ties -> lowest k); score = distance;
// threshold = (1-q)-quantile of train scores (h = (n_train-1)(1-q), linear interpolation);
// flag iff score > threshold.
int eso_kmeans_baseline(const double* X, int64_t N, int D, int K, double q, double train_window, uint64_t seed,
                        int max_iter, double* centroids, double* threshold, uint8_t* flags, double* scores,
                        int64_t* n_flagged, int* iterations, int nthreads) {
    if (K < 1) return fail(kData, "InvalidK", "K must be >= 1");
    if (!(q > 0.0 && q < 1.0)) return fail(kData, "RangeViolation", "q must be in (0,1)");
    if (!(train_window > 0.0 && train_window <= 1.0))
        return fail(kData, "RangeViolation", "train_window must be in (0,1]");
    const int64_t nt = (int64_t)std::floor(train_window * (double)N);
    if (nt < K) return fail(kData, "TooFewPoints", "training split has fewer rows than K");
    if (max_iter <= 0) max_iter = 100;
    set_threads(nthreads);
    SplitMix64 rng(seed);
    std::vector<int64_t> rows;
    kmeanspp_rows(X, nt, D, K, rng, rows);
    std::vector<double> cen((size_t)K * D);
    for (int k = 0; k < K; ++k)
        for (int a = 0; a < D; ++a) cen[(size_t)k * D + a] = X[(size_t)rows[k] * D + a];
    auto nearest = [&](const double* x, double* best) {
        double b = INFINITY;
        int bk = 0;
        for (int k = 0; k < K; ++k) {
            double d2 = 0.0;
            for (int a = 0; a < D; ++a) {
                const double e = x[a] - cen[(size_t)k * D + a];
                d2 = std::fma(e, e, d2);
            }
            if (d2 < b) {
                b = d2;
                bk = k;
            }
        }
        *best = b;
        return bk;
    };
    std::vector<int> asg(nt, -1);
    int it = 0;
    while (it < max_iter) {
        int64_t changed = 0;
#pragma omp parallel for schedule(static) reduction(+ : changed)
        for (int64_t i = 0; i < nt; ++i) {
            double b;
            const int k = nearest(X + (size_t)i * D, &b);
            if (asg[i] != k) ++changed;
            asg[i] = k;
        }
        std::vector<double> sum((size_t)K * D, 0.0), cnt(K, 0.0);
        for (int64_t i = 0; i < nt; ++i) {
            const int k = asg[i];
            cnt[k] += 1.0;
            for (int a = 0; a < D; ++a) sum[(size_t)k * D + a] += X[(size_t)i * D + a];
        }
        ++it;
        for (int k = 0; k < K; ++k)
            if (cnt[k] > 0.0)
                for (int a = 0; a < D; ++a) cen[(size_t)k * D + a] = sum[(size_t)k * D + a] / cnt[k];
        if (changed == 0) break;
    }
    std::vector<double> sc(N);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; ++i) {
        double b;
        nearest(X + (size_t)i * D, &b);
        sc[i] = std::sqrt(b);
    }
    std::vector<double> v(sc.begin(), sc.begin() + nt);
    const double h = (double)(nt - 1) * (1.0 - q);
    const int64_t lo = (int64_t)std::floor(h);
    const int64_t hi = std::min<int64_t>(lo + 1, nt - 1);
    std::nth_element(v.begin(), v.begin() + lo, v.end());
    const double vlo = v[lo];
    double vhi = vlo;
    if (hi != lo) vhi = *std::min_element(v.begin() + lo + 1, v.end());
    const double thr = vlo + (h - (double)lo) * (vhi - vlo);
    int64_t nf = 0;
    for (int64_t i = 0; i < N; ++i) {
        const uint8_t f = sc[i] > thr ? 1 : 0;
        if (flags) flags[i] = f;
        nf += f;
    }
    if (scores) std::copy(sc.begin(), sc.end(), scores);
    if (centroids) std::copy(cen.begin(), cen.end(), centroids);
    *threshold = thr;
    *n_flagged = nf;
    *iterations = it;
    return kOk;
}

// Lloyd's iterations from given centroids (the kmeans_baseline inner loop), for pinning the
// restatement against an external implementation (tests/test_eval_bench.py vs sklearn).
int eso_lloyd(const double* X, int64_t N, int D, int K, double* centroids, int max_iter, int* iterations) {
    std::vector<int> asg(N, -1);
    int it = 0;
    while (it < max_iter) {
        int64_t changed = 0;
        std::vector<double> sum((size_t)K * D, 0.0), cnt(K, 0.0);
        for (int64_t i = 0; i < N; ++i) {
            double b = INFINITY;
            int bk = 0;
            for (int k = 0; k < K; ++k) {
                double d2 = 0.0;
                for (int a = 0; a < D; ++a) {
                    const double e = X[(size_t)i * D + a] - centroids[(size_t)k * D + a];
                    d2 = std::fma(e, e, d2);
                }
                if (d2 < b) {
                    b = d2;
                    bk = k;
                }
            }
            if (asg[i] != bk) ++changed;
            asg[i] = bk;
            cnt[bk] += 1.0;
            for (int a = 0; a < D; ++a) sum[(size_t)bk * D + a] += X[(size_t)i * D + a];
        }
        ++it;
        for (int k = 0; k < K; ++k)
            if (cnt[k] > 0.0)
                for (int a = 0; a < D; ++a) centroids[(size_t)k * D + a] = sum[(size_t)k * D + a] / cnt[k];
        if (changed == 0) break;
    }
    *iterations = it;
    return kOk;
}

// confusion: out = {tp, fp, tn, fn}, anomaly = positive class
int eso_confusion(const uint8_t* labels, const uint8_t* flags, int64_t n, int64_t* out) {
    out[0] = out[1] = out[2] = out[3] = 0;
    for (int64_t i = 0; i < n; ++i) {
        const int l = labels[i] != 0, f = flags[i] != 0;
        ++out[l ? (f ? 0 : 3) : (f ? 1 : 2)];
    }
    return kOk;
}

int eso_select_k_bic(const double* X, int64_t N, int D, const int* k_range, int n_k, const eso_fit_opts* opts,
                     int* best_k, double* bic) {
    if (n_k < 1) return fail(kData, "EmptyRange", "k_range is empty");
    int best = -1;
    double best_bic = INFINITY;
    std::string last_name, last_msg;
    int last_status = kOk;
    for (int j = 0; j < n_k; ++j) {
        const int K = k_range[j];
        std::vector<double> pi(K), mu((size_t)K * D), cov((size_t)K * D * D), per(opts->max_iter + 1);
        eso_fit_report rep{};
        int s = eso_fit_em(X, N, D, K, opts, nullptr, nullptr, nullptr, pi.data(), mu.data(), cov.data(), &rep,
                           per.data());
        if (s != kOk) {  // skip failed K
            bic[j] = NAN;
            last_status = s;
            last_name = g_err_name;
            last_msg = g_err_msg;
            continue;
        }
        const double p = (K - 1) + (double)K * D +
                         (opts->cov_type == 1 ? (double)K * D : (double)K * D * (D + 1) / 2.0);
        bic[j] = -2.0 * rep.final_log_likelihood + p * std::log((double)N);
        if (bic[j] < best_bic) { best_bic = bic[j]; best = K; }
    }
    if (best < 0) return fail(last_status, last_name.c_str(), last_msg);
    *best_k = best;
    return kOk;
}

// ------------------------------------------------------------- SYN-v1 ----
void eso_philox4x32(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        uint32_t n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        uint32_t n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

int eso_syn_model(uint64_t seed, int D, int K, double* pi_true, double* mu_true, double* chol_true) {
    if (K < 1 || D < 1) return fail(kData, "DimensionMismatch", "K and D must be positive");
    SplitMix64 rng(seed ^ 0x5359'4E2D'7631'0000ull);  // "SYN-v1"
    auto normal = [&]() {
        double u1 = 1.0 - rng.uniform(), u2 = rng.uniform();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
    };
    double z = 0.0;
    for (int k = 0; k < K; ++k) z += (double)(k + 1);
    for (int k = 0; k < K; ++k) pi_true[k] = (double)(k + 1) / z;
    std::vector<double> B((size_t)D * D), Sg((size_t)D * D);
    for (int k = 0; k < K; ++k) {
        for (int d = 0; d < D; ++d) mu_true[(size_t)k * D + d] = -3.0 + 6.0 * rng.uniform();
        for (auto& b : B) b = normal();
        for (int a = 0; a < D; ++a)
            for (int c = 0; c < D; ++c) {
                double s = 0.0;
                for (int p = 0; p < D; ++p) s += B[(size_t)a * D + p] * B[(size_t)c * D + p];
                Sg[(size_t)a * D + c] = s / D + (a == c ? 0.05 : 0.0);
            }
        if (!cholesky(Sg.data(), D, chol_true + (size_t)k * D * D))
            return fail(kNumeric, "SingularCovariance", "synthetic covariance not PD");
    }
    return kOk;
}

int eso_syn_rows(uint64_t seed, int D, int K, const double* pi_true, const double* mu_true, const double* chol_true,
                 int64_t row0, int64_t n, double* X, int32_t* comp, uint8_t* anomaly, int nthreads) {
    set_threads(nthreads);
    std::vector<double> cum(K);
    double acc = 0.0;
    for (int k = 0; k < K; ++k) { acc += pi_true[k]; cum[k] = acc; }
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    const uint32_t kStream = 0x53594E31u;  // 'SYN1'
#pragma omp parallel
    {
        std::vector<double> z(D + 1);
#pragma omp for schedule(static)
        for (int64_t j = 0; j < n; ++j) {
            const uint64_t i = (uint64_t)(row0 + j);
            uint32_t ctr[4] = {(uint32_t)i, (uint32_t)(i >> 32), 0u, kStream}, o[4];
            eso_philox4x32(ctr, key, o);
            double uc = (double)((((uint64_t)o[0] << 32) | o[1]) >> 11) * 0x1.0p-53;
            double ua = (double)((((uint64_t)o[2] << 32) | o[3]) >> 11) * 0x1.0p-53;
            int k = K - 1;
            for (int t = 0; t < K - 1; ++t)
                if (uc < cum[t]) { k = t; break; }
            const bool anom = ua < (1.0 / 6.0);
            for (int p = 0; 2 * p < D; ++p) {
                ctr[2] = (uint32_t)(p + 1);
                eso_philox4x32(ctr, key, o);
                double u1 = 1.0 - (double)((((uint64_t)o[0] << 32) | o[1]) >> 11) * 0x1.0p-53;
                double u2 = (double)((((uint64_t)o[2] << 32) | o[3]) >> 11) * 0x1.0p-53;
                double r = std::sqrt(-2.0 * std::log(u1));
                z[2 * p] = r * std::cos(2.0 * M_PI * u2);
                z[2 * p + 1] = r * std::sin(2.0 * M_PI * u2);
            }
            const double s = anom ? 4.0 : 1.0;
            const double* C = chol_true + (size_t)k * D * D;
            for (int a = 0; a < D; ++a) {
                double t = 0.0;
                for (int b = 0; b <= a; ++b) t += C[(size_t)a * D + b] * z[b];
                X[(size_t)j * D + a] = mu_true[(size_t)k * D + a] + s * t;
            }
            if (comp) comp[j] = k;
            if (anomaly) anomaly[j] = anom ? 1 : 0;
        }
    }
    return kOk;
}

}  // extern "C"
