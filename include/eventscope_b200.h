/*
 * eventscope_b200.h — C-ABI of the B200-native eventscope GMM hot path.
 *
 * This is the drop-in boundary.  The reference ships its interface only as
 * SPEC op signatures plus the error type in proj/include/eventscope/errors.hpp
 * (no gmm.hpp / detect.hpp exists under /root/reference/proj/include).  Every
 * entry point below replaces one of those ops; the C++ API in
 * include/eventscope/{gmm,detect}.hpp calls through here and re-throws
 * failures as eventscope::Error with the same stable names.
 *
 *   es_gmm_fit               <- fit_em
 *   es_gmm_em_begin/step/end <- fit_em (stepwise engine; same semantics)
 *   es_gmm_score             <- mixture_density (log form, batched) SPEC.md:271-279
 *                               + predict (argmax responsibility)
 *   es_gmm_responsibilities  <- responsibilities
 *   es_gmm_component_log_density <- component_log_density SPEC.md:261-269
 *   es_gmm_detect            <- detect
 *   es_gmm_calibrate         <- calibrate_threshold
 *   es_gmm_select_k_bic      <- select_k_bic
 *   es_run_pipeline          <- run_pipeline
 *   es_kmeans_baseline       <- kmeans_baseline
 *   es_confusion             <- confusion
 *   es_events_extract        <- extract_features        SPEC.md:62-70 (+ validate_event :52-60)
 *
 * Conventions
 *  - Plain pointers and sizes only.  Parameters are host FP64 arrays, row-major:
 *    weights[K], means[K*D], covariances[K*D*D].
 *  - Outputs may be host or device pointers (detected per call); the library
 *    never retains caller pointers after return.  Datasets are copied into
 *    library-owned HBM once (es_dataset_*), so repeated fit/score calls do not
 *    re-upload the event matrix.
 *  - Return value: 0 ok, else an ErrorKind-mirroring class (errors.hpp:13-17):
 *    ES_ERR_DATA, ES_ERR_NUMERIC, ES_ERR_IO, plus ES_ERR_RUNTIME for CUDA/NCCL
 *    failures.  es_last_error_name()/es_last_error_message() (thread-local)
 *    give the stable name ("TooFewPoints", "SingularCovariance", ...).
 *  - Multi-GPU: one context per GPU/process.  A dataset is that rank's
 *    contiguous block of event rows; ranks exchange only sufficient
 *    statistics (NCCL all-gather over NVLink, reduced in rank order).
 *  - A context is driven by one host thread at a time.
 */
#ifndef EVENTSCOPE_B200_H
#define EVENTSCOPE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ES_OK 0
#define ES_ERR_DATA 1
#define ES_ERR_NUMERIC 2
#define ES_ERR_IO 3
#define ES_ERR_RUNTIME 4

#define ES_INIT_RANDOM 0
#define ES_INIT_KMEANSPP 1 /* SPEC.md:291,319 (default of the C++ API) */
#define ES_INIT_GIVEN 2    /* warm start from es_gmm_params */

#define ES_COV_FULL 0
#define ES_COV_DIAG 1 /* diagonal covariances (not in the reference) */

#define ES_DETECT_COMPONENT 0 /* Def. 1: best-component density */
#define ES_DETECT_MIXTURE 1   /* mixture density ablation */

typedef struct es_ctx es_ctx;
typedef struct es_dataset es_dataset;
typedef struct es_em_state es_em_state;

typedef struct {
    int32_t K;
    int32_t D;
    double* weights;     /* K          */
    double* means;       /* K*D        */
    double* covariances; /* K*D*D      */
} es_gmm_params;

typedef struct {
    int32_t init;     /* ES_INIT_* */
    double tol;       /* SPEC.md:321 default 1e-6 */
    int32_t max_iter; /* SPEC.md:321 default 200 */
    double reg;       /* < 0: default 1e-6*tr(S)/d; 0: disabled */
    uint64_t seed;
    int32_t covariance_type; /* ES_COV_FULL (SPEC) or ES_COV_DIAG (extension) */
} es_fit_opts;

typedef struct {
    int32_t iterations;
    double final_log_likelihood;
    int32_t converged;
    uint64_t seed;
    int32_t n_per_iter;
    int32_t collapses;
    double reg_used;
} es_fit_report;

/* Host-side exchange for multi-rank runs without NCCL (e.g. several ranks
 * sharing one GPU in tests).  Buffers are host memory.  dtype: 0 f64, 1 i64;
 * op: 0 sum, 1 min, 2 max.  Return 0 on success. */
typedef struct {
    void* user;
    int (*allgather)(void* user, const void* send, void* recv, size_t bytes_per_rank);
    int (*allreduce)(void* user, void* buf, size_t count, int dtype, int op);
} es_exchange;

/* ------------------------------------------------------------ errors ---- */
const char* es_last_error_name(void);
const char* es_last_error_message(void);
const char* es_version(void);

/* ----------------------------------------------------------- context ---- */
int es_ctx_create(int device, es_ctx** out);
int es_nccl_unique_id(unsigned char id[128]);
int es_ctx_create_nccl(int device, int rank, int world, const unsigned char id[128], es_ctx** out);
int es_ctx_create_exchange(int device, int rank, int world, const es_exchange* ex, es_ctx** out);
int es_ctx_destroy(es_ctx* ctx);
/* CUDA stream (cudaStream_t) all of this context's work is enqueued on. */
int es_ctx_stream(es_ctx* ctx, void** stream);
/* Kernel-launch counter (for launch accounting in benchmarks). */
int es_ctx_launch_count(es_ctx* ctx, int64_t* count);
/* NCCL collectives this context issued (0 for a single-GPU context; a context made by
 * es_ctx_create_nccl, including a one-rank one under ES_FORCE_NCCL=1, exchanges through NCCL). */
int es_ctx_collective_count(es_ctx* ctx, int64_t* count);
/* Arithmetic of the hot kernels: 0 (default) = mixed — FP32 whitening, FP64
 * statistics / log-likelihoods, FP64 recomputation of every component that
 * can change an output at the 1e-6 level; 1 = strict FP64 everywhere. */
int es_ctx_set_precision(es_ctx* ctx, int mode);
/* CUDA-event timing of the hot kernels on the context stream (resets the
 * accumulators).  which: 0 = fused EM pass, 1 = scoring pass. */
int es_ctx_set_timing(es_ctx* ctx, int enable);
int es_ctx_kernel_time(es_ctx* ctx, int which, double* ms, int64_t* launches);

/* ----------------------------------------------------------- dataset ---- */
/* Copies this rank's rows; element (i,j) at X[i*row_stride + j*col_stride].
 * X may be host (pageable or pinned) or device memory. */
int es_dataset_create(es_ctx* ctx, const double* X, int64_t n_local, int32_t D, int64_t row_stride,
                      int64_t col_stride, es_dataset** out);
/* SYN-v1 synthetic events generated in place on the device:
 * this rank receives global rows [r*n/G, (r+1)*n/G). */
int es_dataset_generate(es_ctx* ctx, uint64_t seed, int64_t n_global, int32_t D, int32_t K_true,
                        es_dataset** out);
/* Rows [row0, row0 + n_global) of the same SYN-v1 stream (a slice of a larger
 * generated matrix, e.g. 2^26 rows at offset 2^29 of the 2^30-event c4 stream);
 * this rank receives [row0 + r*n/G, row0 + (r+1)*n/G); row indices of the
 * dataset are relative to row0. */
int es_dataset_generate_range(es_ctx* ctx, uint64_t seed, int64_t row0, int64_t n_global, int32_t D,
                              int32_t K_true, es_dataset** out);
int es_dataset_destroy(es_dataset* ds);
int es_dataset_info(es_dataset* ds, int64_t* n_local, int64_t* n_global, int64_t* row_offset, int32_t* D);
/* Copies local rows [row0,row0+n) back out, row-major (tests / inspection). */
int es_dataset_read_rows(es_dataset* ds, int64_t row0, int64_t n, double* out);

/* --------------------------------------------------------------- fit ---- */
int es_gmm_fit(es_ctx* ctx, es_dataset* ds, int32_t K, const es_fit_opts* opts, const es_gmm_params* init,
               es_gmm_params* out, es_fit_report* rep, double* per_iter /* max_iter+1, nullable */);
/* Stepwise engine: begin (validation, data statistics, init), step (n EM
 * iterations, stops early on convergence), end (final logL, copy-out). */
int es_gmm_em_begin(es_ctx* ctx, es_dataset* ds, int32_t K, const es_fit_opts* opts, const es_gmm_params* init,
                    es_em_state** out);
int es_gmm_em_step(es_em_state* st, int32_t n_iter, int32_t* done);
int es_gmm_em_end(es_em_state* st, es_gmm_params* out, es_fit_report* rep, double* per_iter);
int es_gmm_em_free(es_em_state* st);
/* Record precision of the last fused (tcgen05) E+M pass: 1 = single fp16 record
 * (every component had >= 2^20 events), 2 = fp16 hi + lo records, 0 = another kernel. */
int es_gmm_em_record_passes(const es_em_state* st, int32_t* passes);
/* Name of the EM pass kernel the last iteration ran ("k_em_mma<1>", "k_em_diag_mixed",
 * "strict FP64 (...)", ...; static storage). */
int es_gmm_em_last_kernel(const es_em_state* st, const char** name);

/* ------------------------------------------------------------- score ---- */
/* Per local event (any output nullable): ll = log p(x); predict = argmax
 * posterior; best_k = argmax_k log N_ik (unweighted);
 * best_logdens = log N_{i,best_k}.  total_ll (nullable) = global sum of ll. */
int es_gmm_score(es_ctx* ctx, es_dataset* ds, const es_gmm_params* p, double* ll, int32_t* predict,
                 int32_t* best_k, double* best_logdens, double* total_ll);
int es_gmm_responsibilities(es_ctx* ctx, es_dataset* ds, const es_gmm_params* p, double* gamma /* n_local*K */);
int es_gmm_component_log_density(es_ctx* ctx, const es_gmm_params* p, const double* x, int32_t k, double* out);
int es_gmm_mixture_log_density(es_ctx* ctx, const es_gmm_params* p, const double* x, double* out);

/* ------------------------------------------------------------ detect ---- */
/* flag_i = (mode value) < log_delta (strict).  anomaly_indices receives the
 * GLOBAL indices of this rank's flagged events in order (capacity n_local).
 * n_flagged = global count; n_local_flagged = this rank's count. */
int es_gmm_detect(es_ctx* ctx, es_dataset* ds, const es_gmm_params* p, double log_delta, int32_t mode,
                  uint8_t* flags, int32_t* best_k, double* best_logdens, int64_t* anomaly_indices,
                  int64_t* n_local_flagged, int64_t* n_flagged);
/* delta = q-quantile (h = (n-1)q, linear interpolation in density space) of
 * the mode values over the GLOBAL rows [0, n_train). */
int es_gmm_calibrate(es_ctx* ctx, es_dataset* ds, const es_gmm_params* p, int64_t n_train, double q, int32_t mode,
                     double* delta, double* log_delta);

/* ---------------------------------------------------------------- BIC ---- */
/* bic[j] = NaN for a K that failed. */
int es_gmm_select_k_bic(es_ctx* ctx, es_dataset* ds, const int32_t* k_range, int32_t n_k, const es_fit_opts* opts,
                        int32_t* best_k, double* bic);

/* ---------------------------------------------------------- pipeline ---- */
/* run_pipeline over a time-ordered feature matrix (row order = event
 * order): the first floor(train_window * N) rows are the training split; columns are
 * z-scored with the training split's mean and population standard deviation (a zero-
 * variance column is centred only); a K-component GMM is fitted on the
 * standardized training split; delta is the quantile_q-quantile of the training split's
 * best-component densities, or cfg->delta when quantile_q <= 0; every
 * row is then scored per detect.  InsufficientTraining if the training
 * split has fewer than 10*K rows.  The model is in standardized space. */
typedef struct {
    int32_t K;
    double train_window;   /* fraction of the earliest events used for fitting, SPEC.md:347 (0.5) */
    double quantile_q;     /* > 0: calibrate delta (SPEC.md:394 default 0.01); <= 0: use delta */
    double delta;          /* density threshold when quantile_q <= 0 */
    int32_t standardize;   /* 1: z-score with training-split statistics */
    int32_t mode;          /* 0: best-component density (Def. 1), 1: mixture density */
    es_fit_opts fit;
} es_pipeline_cfg;
int es_run_pipeline(es_ctx* ctx, es_dataset* ds, const es_pipeline_cfg* cfg, es_gmm_params* model /* out */,
                    es_fit_report* rep, double* std_mean /* D, nullable */, double* std_scale /* D, nullable */,
                    double* delta, double* log_delta, uint8_t* flags /* n_local, nullable */,
                    int32_t* best_k /* n_local, nullable */, double* best_logdens /* n_local, nullable */,
                    int64_t* anomaly_indices /* n_local capacity, nullable */, int64_t* n_local_flagged,
                    int64_t* n_flagged);

/* eval-bench.  k-means baseline: k-means++ seeding (seed) and Lloyd's
 * algorithm on the train split (first floor(train_window N) rows), stopping when no
 * assignment changes or after max_iter steps (<= 0: 100); score = Euclidean distance to
 * the nearest centroid; threshold = (1-q)-quantile of the train scores; flag iff score >
 * threshold.  D <= 64.  Errors: TooFewPoints (n_train < K), RangeViolation. */
int es_kmeans_baseline(es_ctx* ctx, es_dataset* ds, int32_t K, double q, double train_window, uint64_t seed,
                       int32_t max_iter, double* centroids /* K*D, nullable */, double* threshold,
                       uint8_t* flags /* n_local, nullable */, double* scores /* n_local, nullable */,
                       int64_t* n_flagged, int32_t* iterations);
/* Columnar events (SPEC.md:32-38 TraceEvent numeric fields; the attrs this build uses as
 * columns, NaN = absent).  Layers: */
enum { ES_LAYER_CUDA = 0, ES_LAYER_PYTHON = 1, ES_LAYER_TORCH = 2, ES_LAYER_NCCL = 3, ES_LAYER_GPU_SAMPLE = 4 };
typedef struct es_event_columns {
    const uint8_t* layer;        /* n, ES_LAYER_* */
    const int64_t* ts_start;     /* n, ns since epoch, > 0 */
    const int64_t* duration_ns;  /* n, >= 0 */
    const double* message_bytes; /* n or NULL: Nccl attr, >= 0 */
    const double* util_pct;      /* n or NULL: GpuSample attrs */
    const double* mem_used_mb;
    const double* temp_c;
} es_event_columns;
/* extract_features on the device: validates every event (first violation -> Data error
 * RangeViolation / UnknownLayer / MissingField, its row in *bad_row), keeps `layer`'s
 * events in order and writes the layer's default features (Cuda/Python/Torch:
 * log10(duration_ns+1); Nccl: + log10(message_bytes+1); GpuSample: util, mem, temp) into a
 * new dataset; event_index (n capacity, nullable) receives the source event of each row.
 * EmptyLayer when no event has the layer. */
int es_events_extract(es_ctx* ctx, const es_event_columns* cols, int64_t n, int32_t layer, es_dataset** out,
                      int64_t* event_index, int64_t* bad_row);
/* out = {tp, fp, tn, fn}, anomaly = positive class; labels / flags host or device. */
int es_confusion(es_ctx* ctx, const uint8_t* labels, const uint8_t* flags, int64_t n, int64_t* out);

#ifdef __cplusplus
}
#endif
#endif /* EVENTSCOPE_B200_H */
