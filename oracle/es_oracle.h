/*
 * es_oracle.h — CPU restatement of the eventscope GMM hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  The product (paper_2506_02007_b200/) never links or calls it.
 *
 * Parity pinning: the reference ships no implementation (proj/src is absent,
 * /root/reference/proj/CMakeLists.txt:16-18) and its linear-algebra dependency
 * (Eigen3 >= 3.3, CMakeLists.txt:12) is not installed and has no version pin.
 * This oracle is therefore pinned by (1) every closed-form example of
 * SPEC.md gmm-core / anomaly-detect (tests/test_oracle_golden.py) and (2)
 * scikit-learn 1.9.0 GaussianMixture fixtures committed under tests/golden/
 * (tests/golden/make_sklearn_golden.py).  At the Eigen boundary parity is
 * "unpinned" (no reference-produced vectors exist) — see DESIGN.md.
 *
 * Conventions: all matrices row-major FP64; X is N x D (row i = x_i,
 * SPEC.md:41); covariances are K x D x D.  Status codes mirror errors.hpp
 * ErrorKind (/root/reference/proj/include/eventscope/errors.hpp:13-17):
 * 0 ok, 1 Data, 2 Numeric, 3 Io; eso_last_error_name() gives the stable name.
 */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int init;          /* 0 = Random, 1 = KMeansPP, 2 = user supplied */
    double tol;        /* SPEC.md:321 default 1e-6 */
    int max_iter;      /* SPEC.md:321 default 200 */
    double reg;        /* < 0 => default 1e-6*tr(S)/d; 0 => disabled */
    uint64_t seed;
    int nthreads;      /* 0 => OpenMP default */
    int cov_type;      /* 0 = full (SPEC), 1 = diagonal (extension) */
} eso_fit_opts;

typedef struct {
    int iterations;
    double final_log_likelihood;
    int converged;
    uint64_t seed;
    int n_per_iter;    /* entries written to per_iter */
    int collapses;
    double reg_used;
} eso_fit_report;

const char* eso_last_error_name(void);
const char* eso_last_error_message(void);

/* SPEC.md:261-269 */
int eso_component_log_density(const double* pi, const double* mu, const double* cov,
                              int K, int D, const double* x, int k, double* out);
/* SPEC.md:271-279 (log form: log p(x)) */
int eso_mixture_log_density(const double* pi, const double* mu, const double* cov,
                            int K, int D, const double* x, double* out);

/* Per-event scoring over X: any output pointer may be NULL.
 *   ll[i]           = log p(x_i)                              (score_samples)
 *   predict[i]      = argmax_k log pi_k + log N_ik, ties -> lowest k
 *   best_k[i]       = argmax_k log N_ik (unweighted), ties -> lowest k
 *   best_logdens[i] = log N_{i,best_k}
 *   gamma[i*K+k]    = responsibilities                      */
int eso_score(const double* X, int64_t N, int D, const double* pi, const double* mu,
              const double* cov, int K, double* ll, int32_t* predict, int32_t* best_k,
              double* best_logdens, double* gamma, int nthreads);

/* Data statistics: mean (D), biased covariance S (D x D), per-column min/max. */
int eso_data_stats(const double* X, int64_t N, int D, double* mean, double* S,
                   double* colmin, double* colmax, int nthreads);

/* Random init (SPEC.md:335 + DESIGN.md "Random init"): K distinct rows drawn by
 * SplitMix64(seed), pi = 1/K, Sigma = S + reg I.  reg < 0 => default.        */
int eso_random_init(const double* X, int64_t N, int D, int K, uint64_t seed, double reg,
                    double* pi, double* mu, double* cov, double* reg_used);

/* EM fit (Alg. 1).  If opts->init == 2, pi/mu/cov
 * in *_init are used.  per_iter must hold max_iter+1 doubles.               */
int eso_fit_em(const double* X, int64_t N, int D, int K, const eso_fit_opts* opts,
               const double* pi_init, const double* mu_init, const double* cov_init,
               double* pi, double* mu, double* cov, eso_fit_report* rep, double* per_iter);

/* One EM iteration in place (E-step + literal two-pass M-step of eso_fit_em, no
 * collapse reseed): the timed unit of bench.py --impl reference.  *logL = logL of
 * the parameters on entry; *n_collapsed = components with N_k < 1. */
int eso_em_step(const double* X, int64_t N, int D, int K, double reg, int cov_type, double* pi, double* mu,
                double* cov, double* logL, int* n_collapsed, int nthreads);

/* detect: mode 0 = best-component density (Def. 1), mode 1 =
 * mixture density.  flag iff log p < log_delta.                */
int eso_detect(const double* X, int64_t N, int D, const double* pi, const double* mu,
               const double* cov, int K, double log_delta, int mode, uint8_t* flags,
               int32_t* best_k, double* best_logdens, int64_t* n_flagged, int nthreads);

/* calibrate_threshold: q-quantile (linear interpolation between
 * order statistics, h = (n-1) q) of best-component densities over rows [0,n_train). */
int eso_kmeans_baseline(const double* X, int64_t N, int D, int K, double q, double train_window, uint64_t seed,
                        int max_iter, double* centroids, double* threshold, uint8_t* flags, double* scores,
                        int64_t* n_flagged, int* iterations, int nthreads);
int eso_lloyd(const double* X, int64_t N, int D, int K, double* centroids, int max_iter, int* iterations);
int eso_confusion(const uint8_t* labels, const uint8_t* flags, int64_t n, int64_t* out);
int eso_calibrate(const double* X, int64_t n_train, int D, const double* pi,
                  const double* mu, const double* cov, int K, double q, int mode,
                  double* delta, double* log_delta, int nthreads);

/* select_k_bic. bic must hold n_k doubles (NaN for failed K). */
int eso_select_k_bic(const double* X, int64_t N, int D, const int* k_range, int n_k,
                     const eso_fit_opts* opts, int* best_k, double* bic);

/* SYN-v1 synthetic generator: true model + rows [row0,row0+n). */
int eso_syn_model(uint64_t seed, int D, int K, double* pi_true, double* mu_true,
                  double* chol_true);
int eso_syn_rows(uint64_t seed, int D, int K, const double* pi_true, const double* mu_true,
                 const double* chol_true, int64_t row0, int64_t n, double* X,
                 int32_t* comp, uint8_t* anomaly, int nthreads);

/* Philox4x32-10 block (exposed for cross-checks against the device generator). */
void eso_philox4x32(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

#ifdef __cplusplus
}
#endif
