// es_layout.h — HBM layouts shared by the kernels and the host runtime.
//
// Event matrix (this rank's shard): feature-planar FP64, plane j holds
// x_{i,j} for all local rows i at X[j*ld + i]; ld is the row count rounded up
// to 32 so every plane starts 256-byte aligned.  Column-major is what an
// Eigen-backed FeatureMatrix (Eigen default storage) already
// is, and it makes the thread-per-event loads fully coalesced.
//
// Model ("derived") block, FP64, for K components of dimension D:
//   pi[K] | logpi[K] | lognorm[K] | mu[K*D] | cov[K*D*D] | L[K*D*D] | W[K*D*D]
// L = chol(cov_k) (lower), W = L^-1 (lower, zeros above the diagonal),
// lognorm = -1/2 log|Sigma_k| - D/2 log(2 pi).
//
// Sufficient-statistics block (one per CTA partial / per rank), FP64:
//   for k: [ N_k | s1_k[D] | s2_k[D(D+1)/2 packed upper, row-major] ] ... | logL
// Statistics are taken about c_k = mu_k of the current model; "whitened"
// blocks hold them in z = W_k (x - mu_k) coordinates (team kernels), raw
// blocks in d = x - mu_k coordinates (generic kernel).
#pragma once
#include <stdint.h>

namespace es {

constexpr double kLog2Pi = 1.8378770664093454835606594728112;

inline __host__ __device__ int64_t plane_ld(int64_t n) { return (n + 31) / 32 * 32; }
inline __host__ __device__ int packed_size(int D) { return D * (D + 1) / 2; }
inline __host__ __device__ int packed_index(int a, int b, int D) {  // a <= b
    return a * D - (a * (a - 1)) / 2 + (b - a);
}
inline __host__ __device__ int stat_k(int D) { return 1 + D + packed_size(D); }
inline __host__ __device__ int stat_total(int D, int K) { return K * stat_k(D) + 1; }

struct ModelView {
    int K, D;
    double* base;
    __host__ __device__ double* pi() const { return base; }
    __host__ __device__ double* logpi() const { return base + K; }
    __host__ __device__ double* lognorm() const { return base + 2 * K; }
    __host__ __device__ double* mu() const { return base + 3 * K; }
    __host__ __device__ double* cov() const { return mu() + (int64_t)K * D; }
    __host__ __device__ double* L() const { return cov() + (int64_t)K * D * D; }
    __host__ __device__ double* W() const { return L() + (int64_t)K * D * D; }
    static __host__ __device__ int64_t size(int K, int D) { return 3 * (int64_t)K + (int64_t)K * D + 3 * (int64_t)K * D * D; }
};

// Device-side status written by the M-step finalize, read by the host once
// per EM iteration (the only device->host crossing in the loop).
struct IterStatus {
    double logL;             // logL of the model the E-step just used
    uint64_t collapse_lo;    // components 0..63 with N_k < 1
    uint64_t collapse_hi;    // components 64..127
    int32_t not_pd;          // a new covariance failed Cholesky
    int32_t pad;
    uint64_t min_nk_inv;     // ~bits(min_k N_k) (max-reduced; 0 = none): picks the record precision
};

// Per-iteration record of k_finalize, written straight into mapped pinned host memory
// (no memset, no copy node): every component's entry is written unconditionally.
constexpr int kMaxK = 128;
struct IterRecord {
    double logL;            // logL of the model the E-step just used
    double nk[kMaxK];       // N_k of the statistics
    int32_t flags[kMaxK];   // bit 0: collapse (N_k < 1), bit 1: new covariance not positive definite
};

}  // namespace es
