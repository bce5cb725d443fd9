// es_kernels.h — launchers for the sm_100a kernels (es_kernels.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "es_layout.h"

namespace es {

constexpr int kBlock = 256;

// Per-event outputs of a scoring pass; any pointer may be null.
struct ScoreOut {
    double* ll = nullptr;          // log p(x_i)
    int32_t* predict = nullptr;    // argmax_k log pi_k + log N_ik
    int32_t* best_k = nullptr;     // argmax_k log N_ik
    double* best_ld = nullptr;     // log N_{i,best_k}
    uint8_t* flags = nullptr;      // (mode value) < log_delta
    double* gamma = nullptr;       // n x K responsibilities
    double* lnk = nullptr;         // n x K component log densities
    double log_delta = 0.0;
    int mode = 0;                  // 0 component, 1 mixture
    int sum_ll = 1;                // the per-CTA sum of ll is used (0: detect / calibrate skip ll)
};

struct LaunchStats {
    int64_t launches = 0;
};

// Which EM pass implementation a (D, K) shape uses.
enum class EmPath { Team4, Team8, Team16, Generic };
EmPath em_path(int D, int K);
// Number of CTA partial blocks the EM pass writes for this shape.
int em_grid(int D, int K, int num_sms);
int score_grid(int D, int K, int num_sms);

// EM E+M pass: writes grid partial stat blocks (stat_total(D,K) doubles each)
// into `partial`; returns the grid size through *nblk.  `whitened` reports
// the coordinate system of the statistics.
void launch_em_pass(const double* X, int64_t n, int64_t ld, int D, int K, const double* model, double* partial,
                    int num_sms, int* nblk, bool* whitened, cudaStream_t s, LaunchStats& ls);
// Unit-weight statistics about `center` (K = 1): data covariance pass.
void launch_unit_stats(const double* X, int64_t n, int64_t ld, int D, const double* center, double* partial,
                       int num_sms, int* nblk, cudaStream_t s, LaunchStats& ls);
// Z = (X - mean) * inv_scale per feature plane (run_pipeline standardization).
void launch_standardize(const double* X, int64_t n, int64_t ld, int D, const double* mean, const double* inv_scale,
                        double* Z, int64_t zld, int num_sms, cudaStream_t s, LaunchStats& ls);
// Fixed-order sum of nblk partial blocks of length len -> out.
void launch_reduce_blocks(const double* partial, int nblk, int len, double* out, cudaStream_t s, LaunchStats& ls);
// Column sum/min/max/non-finite count: out[4*D] = sum | min | max | nonfinite.
void launch_col_stats(const double* X, int64_t n, int64_t ld, int D, double* scratch, double* out, int num_sms,
                      cudaStream_t s, LaunchStats& ls);
// M-step finalize from G rank blocks of statistics (summed in rank order),
// updating the model in place and writing IterStatus (+ logL record[t]).
// whitened: 0 raw statistics, 1 whitened (team kernels), 2 raw + diagonal covariance
// whitened 3: raw statistics about c + fp32((mu_k - c) xs) / xs (k_em_mma), needs center and xs;
// whitened 4: as 3 with diagonal covariances (k_em_diag_mixed, xs = 1).
// G < 0: the -G per-CTA partial blocks of a one-rank pass, reduced inside (no k_reduce_blocks).
// model_in -> model_out (may alias; a collapsed component is carried over unchanged).
// G < 0 also needs `red` (K * stat_k(D) + 1 doubles) and `tick` (K zeroed ints, left zeroed).
void launch_finalize(const double* stats, int G, int D, int K, int64_t n_global, double reg, int whitened,
                     const double* model_in, double* model_out, IterRecord* st, double* record, int t,
                     cudaStream_t s, LaunchStats& ls, const double* center = nullptr, double xs = 1.0,
                     double* red = nullptr, int* tick = nullptr);
// Diagonal-covariance E+M pass (FP64 team kernel, D <= 32, K <= 32).
void launch_em_diag(const double* X, int64_t n, int64_t ld, int D, int K, const double* model, double* partial,
                    int num_sms, int* nblk, cudaStream_t s, LaunchStats& ls);
// Mixed-precision diagonal E+M pass (es_em_diag.cu): FP32 packed arithmetic with per-component
// centring, FP64 accumulation every 32 events per lane; statistics for finalize mode 4 (diagonal,
// about center + fp32(mu_k - center)).  D <= 16, K <= 16.
bool em_diag_mixed_supported(int D, int K);
void launch_em_diag_mixed(const double* X, int64_t n, int64_t ld, int D, int K, const double* model,
                          const double* center, double* partial, int num_sms, int* nblk, cudaStream_t s,
                          LaunchStats& ls);
// Mixed-precision full-covariance E+M pass (es_em_full.cu) for the shapes the tensor-core pass
// does not take (D <= 32, K <= 32): FP32 packed arithmetic with per-component centring, FP64
// statistics; finalize mode 3 (about center + fp32((mu_k - center) xs) / xs).
// Full-covariance E+M pass on tcgen05 for D <= 32, K <= 32 (es_em_wide.cu; BASELINE c5):
// E-step whitening and M-step Gram on the tensor cores in groups of 4 components; npass = 1
// one fp16 record per value (>= kOnePassMinNk events per component), 2 fp16 hi + lo records;
// finalize mode 3.  `workspace`
// holds em_wide_workspace_bytes() (the per-pass operand images); two launches.
bool em_wide_supported(int D, int K);
size_t em_wide_workspace_bytes();
void launch_em_wide(const double* X, int64_t n, int64_t ld, int D, int K, const double* model, const double* center,
                    const double* center_host, double xs, bool f32conv, int npass, void* workspace, double* partial,
                    int num_sms, int* nblk, cudaStream_t s, LaunchStats& ls);
// Diagonal E+M pass on tcgen05 (es_em_diag_tc.cu; BASELINE c3): per-event fp16 records of
// (x^2, x, 1) serve as the E-step A operand (w = A Theta) and the M-step A operand (A^T Gamma);
// D <= 16, K <= 16, >= kOnePassMinNk events per component; finalize mode 2.  ES_EM_DIAG_TC=0 off.
bool em_diag_tc_enabled(int D, int K);
int em_diag_tc_mode();
void launch_em_diag_tc(const CUtensorMap* xmap, int64_t n, int D, int K, const double* model, const double* center,
                       const double* center_host, double xs, double* partial, int num_sms, int* nblk, cudaStream_t s,
                       LaunchStats& ls);
bool em_full_mixed_supported(int D, int K);
void launch_em_full_mixed(const double* X, int64_t n, int64_t ld, int D, int K, const double* model,
                          const double* center, double xs, double* partial, int num_sms, int* nblk, cudaStream_t s,
                          LaunchStats& ls);
// Derive L, W, lognorm, logpi from pi, mu, cov in `model` (all components).
void launch_derive(double* model, int D, int K, IterStatus* st, cudaStream_t s, LaunchStats& ls);
// Scoring pass; `blocksum` receives per-CTA [ll_sum, flag_count] pairs.
void launch_score(const double* X, int64_t n, int64_t ld, int D, int K, const double* model, const ScoreOut& o,
                  double* blocksum, int num_sms, int* nblk, cudaStream_t s, LaunchStats& ls);
// Order-preserving radix select helpers on FP64 keys.
void launch_hist8(const double* keys, int64_t n, int shift, uint64_t prefix_mask, uint64_t prefix_val,
                  unsigned long long* hist, int num_sms, cudaStream_t s, LaunchStats& ls);
// Anomaly-index compaction (order preserving).
void launch_compact(const uint8_t* flags, int64_t n, int64_t index_base, int64_t* counts_scratch,
                    int64_t* out_idx, int64_t* out_count, cudaStream_t s, LaunchStats& ls);
// Row-major staging -> planar transpose for rows [row0, row0+n).
void launch_rows_to_planar(const double* rows, int64_t n, int D, double* X, int64_t ld, int64_t row0,
                           cudaStream_t s, LaunchStats& ls);
// Planar -> row-major for rows [row0, row0+n).
void launch_planar_to_rows(const double* X, int64_t ld, int D, int64_t row0, int64_t n, double* rows,
                           cudaStream_t s, LaunchStats& ls);
// k-means++ distance update: d2[i] = min(d2[i], ||x_i - c||^2) (first: assign),
// parts[chunk] = fixed-order sum of d2 over 4096-row chunks.
void launch_kpp_update(const double* X, int64_t n, int64_t ld, int D, const double* center, double* d2,
                       double* parts, bool first, cudaStream_t s, LaunchStats& ls);
// Shapes of the fused tensor-core passes (D <= 16, K <= 8): the mixed-precision path's domain.
bool em_mixed_supported(int D, int K);
// Fused pass with E-step and M-step Gram on tcgen05 (es_em_mma.cu), the mixed-precision EM
// pass for D <= 16, K <= 8.  Writes finalize mode-3 statistics.
bool em_mma_enabled();
// Record precision: npass 2 (fp16 hi + lo records) or 1 (single fp16 record, used when
// every component has >= kOnePassMinNk events); ES_EM_MMA_PASSES=1|2 overrides.
constexpr double kOnePassMinNk = 1048576.0;
// Mixed-precision (tcgen05 E-step) EM passes run only when every component has at least
// this many events; below, the iteration uses the strict FP64 kernel.
constexpr double kMixedMinNk = 16384.0;
int em_mma_passes();
// f32conv: max|x| <= 4 max|x - c| over the data, so x^ = (x - c) xs may be formed on the FP32
// pipe (error <= 2^-24 * 64 in x^ units) instead of an FP64 fma per value (ES_EM_F32CONV=0 off).
void launch_em_mma(const CUtensorMap* xmap, int64_t n, int D, int K, const double* model, const double* center,
                   const double* center_host, double xs, bool f32conv, int npass, double* partial, int num_sms,
                   int* nblk, cudaStream_t s, LaunchStats& ls);
// Builds that tensor map (driver entry point resolved through the runtime).
bool make_event_tmap(CUtensorMap* map, const double* X, int64_t n, int64_t ld, int D);
// Fused-pipeline scoring pass (es_score_mma.cu), the default for D <= 16, K <= 8:
// center_host / xs as for launch_em_mma (x^ = (x - c) xs, xs a power of two).
bool score_mma_enabled(int D, int K, const ScoreOut& o);
void launch_score_mma(const CUtensorMap* xmap, int64_t n, int D, int K, const double* model, const double* center,
                      const double* center_host, double xs, const ScoreOut& o, double* blocksum, int num_sms,
                      int* nblk, cudaStream_t s, LaunchStats& ls);
// SYN-v1 rows [grow0, grow0+n) written into planar X (local row = global - grow0).
void launch_synth(double* X, int64_t ld, int64_t n, int64_t grow0, int D, int K, const double* syn_model,
                  uint64_t seed, cudaStream_t s, LaunchStats& ls);


// k-means baseline (eval-bench): Lloyd step (mode 0: partial[blk][K (D + 1) + 1] = per
// centroid row sums | count, then changed assignments) or scoring (mode 1: score[i] =
// distance to the nearest centroid), D <= 64; grid from lloyd_grid (fixed row order).
int lloyd_grid(int64_t n, int num_sms);
void launch_lloyd(const double* X, int64_t n, int64_t ld, int D, int K, const double* cen, int32_t* assign,
                  double* partial, double* score, int mode, int grid, cudaStream_t s, LaunchStats& ls);
void launch_flag_gt(const double* score, int64_t n, double thr, uint8_t* flags, unsigned long long* count,
                    int num_sms, cudaStream_t s, LaunchStats& ls);
void launch_confusion(const uint8_t* labels, const uint8_t* flags, int64_t n, unsigned long long* out, int num_sms,
                      cudaStream_t s, LaunchStats& ls);

// event features (extract_features): validation + layer filter, then the layer's features
void launch_event_keep(const uint8_t* layer, const int64_t* ts, const int64_t* dur, const double* mb,
                       const double* util, const double* mem, const double* temp, int64_t n, int L, uint8_t* keep,
                       unsigned long long* bad, int num_sms, cudaStream_t s, LaunchStats& ls);
void launch_event_features(const int64_t* idx, int64_t m, const int64_t* dur, const double* mb, const double* util,
                           const double* mem, const double* temp, int L, double* X, int64_t ld, int num_sms,
                           cudaStream_t s, LaunchStats& ls);

}  // namespace es
