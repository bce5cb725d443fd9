// es_chol.cuh — warp-level FP64 Cholesky factorisation and triangular inverse of one D x D
// covariance (the M-step's finalize, derive): L = chol(A), W = L^-1, log|A|; the pinned
// numerical-singularity rule of the oracle (a pivot at or below D 2^-46 of its diagonal entry).
#pragma once
#include <cmath>

namespace es {

__device__ __forceinline__ double chol_warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// CTA form (every thread of the block calls it; thread = matrix element): the finalize runs once
// per EM iteration right after a pass that streamed gigabytes through L2, so its code is fetched
// cold and its critical path is a chain of dependent shared-memory round trips; here each
// column j costs one rsqrt and two barriers.  Step j scales column j of L (and row j of
// W = L^-1, now final), then every element updates once: L[i][c] -= L[i][j] L[c][j] (j < c <= i)
// and W[i][c] -= L[i][j] W[j][c] (c <= j < i).  D <= 32; same pinned pivot rule as chol_inv_warp.
// (scripts/chol_probe.cu: warm / cold cycles of the forms; scripts/fin_trace.py: in the M-step.)
__device__ __noinline__ bool chol_inv_cta(const double* A, double* L, double* W, int D, int ld, double* logdet,
                                          double* scratch) {
    const int t = threadIdx.x, nt = blockDim.x, n2 = D * D;
    const double thr = ldexp((double)D, -46);
    bool ok = true;
    if (n2 <= nt) {  // one element per thread (D <= 16 with 256 threads): indices hoisted
        const bool on = t < n2;
        const int i = on ? t / D : 0, c = on ? t - i * D : 0, o = i * ld + c;
        if (on) {
            L[o] = c <= i ? A[o] : 0.0;
            W[o] = c == i ? 1.0 : 0.0;
        }
        __syncthreads();
        for (int j = 0; j < D; ++j) {
            const double piv = L[j * ld + j];
            if (!(piv > thr * A[j * ld + j]) || !isfinite(piv)) ok = false;
            const double rl = rsqrt(fmax(piv, 0.0));
            if (on) {
                if (c == j && i > j) L[o] *= rl;
                if (i == j && c <= j) W[o] *= rl;
                if (i == j && c == j) L[o] = piv * rl;
            }
            __syncthreads();
            if (on && i > j) {
                const double lij = L[i * ld + j];
                if (c > j && c <= i) L[o] = fma(-lij, L[c * ld + j], L[o]);
                if (c <= j) W[o] = fma(-lij, W[j * ld + c], W[o]);
            }
            __syncthreads();
        }
        if (t < 32) {
            double v = 0.0;
            for (int r = t; r < D; r += 32) v += log(L[r * ld + r]);
            v = chol_warp_sum(v);
            if (t == 0) scratch[0] = v;
        }
        __syncthreads();
        *logdet = 2.0 * scratch[0];
        __syncthreads();
        return ok;
    }
    for (int e = t; e < n2; e += nt) {
        const int i = e / D, c = e % D;
        L[i * ld + c] = c <= i ? A[i * ld + c] : 0.0;
        W[i * ld + c] = c == i ? 1.0 : 0.0;
    }
    __syncthreads();
    for (int j = 0; j < D; ++j) {
        const double piv = L[j * ld + j];
        // numerical singularity: pivot at or below D 2^-46 of its diagonal entry (as the oracle)
        if (!(piv > thr * A[j * ld + j]) || !isfinite(piv)) ok = false;
        const double rl = rsqrt(fmax(piv, 0.0));
        for (int e = t; e < n2; e += nt) {
            const int i = e / D, c = e % D;
            if (c == j && i > j) L[i * ld + j] *= rl;
            if (i == j && c < j) W[j * ld + c] *= rl;
            if (i == j && c == j) {
                L[j * ld + j] = piv * rl;
                W[j * ld + j] *= rl;
            }
        }
        __syncthreads();
        for (int e = t; e < n2; e += nt) {
            const int i = e / D, c = e % D;
            if (i > j) {
                const double lij = L[i * ld + j];
                if (c > j && c <= i) L[i * ld + c] = fma(-lij, L[c * ld + j], L[i * ld + c]);
                if (c <= j) W[i * ld + c] = fma(-lij, W[j * ld + c], W[i * ld + c]);
            }
        }
        __syncthreads();
    }
    if (t < 32) {
        double v = 0.0;
        for (int i = t; i < D; i += 32) v += log(L[i * ld + i]);
        v = chol_warp_sum(v);
        if (t == 0) scratch[0] = v;
    }
    __syncthreads();
    *logdet = 2.0 * scratch[0];
    __syncthreads();
    return ok;
}

__device__ bool chol_inv_warp(const double* A, double* L, double* W, int D, int ld, double* logdet) {
    const int lane = threadIdx.x & 31;
    bool ok = true;
    for (int e = lane; e < D * ld; e += 32) {
        L[e] = 0.0;
        W[e] = 0.0;
    }
    __syncwarp();
    // left-looking, lanes over rows i >= j: t_i = A[i][j] - sum_{p<j} L[i][p] L[j][p] (four
    // independent partial sums); lane j's t_j is the pivot, broadcast by a shuffle
    for (int j = 0; j < D; ++j) {
        double tv[2] = {0.0, 0.0};
        for (int h = 0; h < 2; ++h) {
            const int i = j + lane + 32 * h;
            if (i >= D || (h == 1 && D <= 32)) continue;
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            int p = 0;
            for (; p + 4 <= j; p += 4) {
                s0 = fma(L[i * ld + p], L[j * ld + p], s0);
                s1 = fma(L[i * ld + p + 1], L[j * ld + p + 1], s1);
                s2 = fma(L[i * ld + p + 2], L[j * ld + p + 2], s2);
                s3 = fma(L[i * ld + p + 3], L[j * ld + p + 3], s3);
            }
            for (; p < j; ++p) s0 = fma(L[i * ld + p], L[j * ld + p], s0);
            tv[h] = A[i * ld + j] - ((s0 + s1) + (s2 + s3));
        }
        const double dj = __shfl_sync(0xffffffffu, tv[0], 0);  // row i = j sits in lane 0
        // numerical singularity: pivot at or below D 2^-46 of its diagonal entry (as the oracle)
        if (!(dj > ldexp((double)D, -46) * A[j * ld + j]) || !isfinite(dj)) ok = false;
        const double ljj = sqrt(fmax(dj, 0.0));
        const double rl = 1.0 / ljj;
        __syncwarp();
        for (int h = 0; h < 2; ++h) {
            const int i = j + lane + 32 * h;
            if (i >= D || (h == 1 && D <= 32)) continue;
            L[i * ld + j] = i == j ? ljj : tv[h] * rl;
        }
        if (lane == 0) L[j * ld + D] = rl;
        __syncwarp();
    }
    // W = L^-1 by columns (lane c): W[r][c] = (delta_rc - sum_{p=c}^{r-1} L[r][p] W[p][c]) / L[r][r]
    for (int c = lane; c < D; c += 32) {
        for (int r = c; r < D; ++r) {
            double s0 = (r == c) ? 1.0 : 0.0, s1 = 0.0;
            int p = c;
            for (; p + 2 <= r; p += 2) {
                s0 -= L[r * ld + p] * W[p * ld + c];
                s1 -= L[r * ld + p + 1] * W[(p + 1) * ld + c];
            }
            if (p < r) s0 -= L[r * ld + p] * W[p * ld + c];
            W[r * ld + c] = (s0 + s1) * L[r * ld + D];
        }
    }
    __syncwarp();
    double ldt = 0.0;
    for (int j = lane; j < D; j += 32) ldt += log(L[j * ld + j]);
    ldt = chol_warp_sum(ldt);
    *logdet = 2.0 * ldt;
    for (int j = lane; j < D; j += 32) L[j * ld + D] = 0.0;
    return ok;
}

// Every thread of the block calls it.  scratch: one double of shared memory.
__device__ bool chol_inv_any(const double* A, double* L, double* W, int D, int ld, double* logdet,
                             double* scratch) {
    if (D <= 32) return chol_inv_cta(A, L, W, D, ld, logdet, scratch);
    bool ok = true;
    if (threadIdx.x < 32) {
        ok = chol_inv_warp(A, L, W, D, ld, logdet);
        if (threadIdx.x == 0) {
            scratch[0] = *logdet;
            scratch[1] = ok ? 1.0 : 0.0;
        }
    }
    __syncthreads();
    *logdet = scratch[0];
    ok = scratch[1] != 0.0;
    __syncthreads();
    return ok;
}

}  // namespace es
