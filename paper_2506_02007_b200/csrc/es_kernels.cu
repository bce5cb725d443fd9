// es_kernels.cu — sm_100a kernels of the eventscope GMM hot path.
//
// Hot kernels (see DESIGN.md for the roofline of each):
//   k_em_team<DM,H>   fused E-step + M-step sufficient statistics, one pass over
//                     the event matrix (Alg. 1);
//                     responsibilities never touch HBM.
//   k_score_team<DM>  streaming score_samples / predict / detect flags
//                     (Alg. 2).
// Both map one "team" of K*H lanes onto one event: lane (k,h) whitens the
// event against component k (W_k = L_k^-1 held in shared memory), the team
// does a butterfly log-sum-exp over k, and (EM) lane (k,h) accumulates its
// 1/H share of component k's statistics in registers for every event the
// thread ever sees.  All reductions are fixed-order (no floating-point
// atomics): bit-reproducible runs.
//
// Everything is FP64: the parity contract is 1e-6 relative per-event ll and
// 1e-5 relative parameters with FP64 statistics accumulation.
#include <cfloat>
#include <cmath>

#include "es_chol.cuh"
#include "es_kernels.h"

namespace es {

// Opt a kernel into the largest dynamic shared memory it can use: the
// device's per-block opt-in limit minus the kernel's own static __shared__.
template <class F>
static void allow_max_smem(F* f) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes a{};
    cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(f));
    cudaFuncSetAttribute(reinterpret_cast<const void*>(f), cudaFuncAttributeMaxDynamicSharedMemorySize,
                         optin - (int)a.sharedSizeBytes);
}

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Fixed-order block sum (tree over smem); result valid in thread 0.
__device__ double block_sum(double v, double* red) {
    const int t = threadIdx.x;
    red[t] = v;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (t < s) red[t] += red[t + s];
        __syncthreads();
    }
    double r = red[0];
    __syncthreads();
    return r;
}

__device__ __forceinline__ int decode_pair(int p, int D, int* b) {
    int a = 0;
    while (p >= D - a) {
        p -= D - a;
        ++a;
    }
    *b = a + p;
    return a;
}

// ----------------------------------------------------------- Philox4x32-10
__device__ __forceinline__ void philox(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
        uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
        uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0;
        c[1] = lo1;
        c[2] = n2;
        c[3] = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

__device__ __forceinline__ double u53(uint32_t a, uint32_t b) {
    return (double)((((uint64_t)a << 32) | b) >> 11) * 0x1.0p-53;
}

}  // namespace

// ===================================================================== synth
// SYN-v1: syn_model = cum_pi[K] | mu[K*D] | chol[K*D*D].
__global__ void k_synth(double* __restrict__ X, int64_t ld, int64_t n, int64_t grow0, int D, int K,
                        const double* __restrict__ sm, uint32_t key0, uint32_t key1) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const uint64_t i = (uint64_t)(grow0 + j);
    const double* cum = sm;
    const double* mu = sm + K;
    const double* ch = mu + (int64_t)K * D;
    uint32_t c[4] = {(uint32_t)i, (uint32_t)(i >> 32), 0u, 0x53594E31u};
    philox(c, key0, key1);
    const double uc = u53(c[0], c[1]);
    const double ua = u53(c[2], c[3]);
    int k = K - 1;
    for (int t = 0; t < K - 1; ++t)
        if (uc < cum[t]) {
            k = t;
            break;
        }
    const double s = ua < (1.0 / 6.0) ? 4.0 : 1.0;
    double z[64];
    for (int p = 0; 2 * p < D; ++p) {
        uint32_t d[4] = {(uint32_t)i, (uint32_t)(i >> 32), (uint32_t)(p + 1), 0x53594E31u};
        philox(d, key0, key1);
        const double u1 = 1.0 - u53(d[0], d[1]);
        const double u2 = u53(d[2], d[3]);
        const double r = sqrt(-2.0 * log(u1));
        z[2 * p] = r * cos(2.0 * M_PI * u2);
        if (2 * p + 1 < 64) z[2 * p + 1] = r * sin(2.0 * M_PI * u2);
    }
    const double* C = ch + (int64_t)k * D * D;
    for (int a = 0; a < D; ++a) {
        double t = 0.0;
        for (int b = 0; b <= a; ++b) t += C[a * D + b] * z[b];
        X[(int64_t)a * ld + j] = mu[k * D + a] + s * t;
    }
}

void launch_synth(double* X, int64_t ld, int64_t n, int64_t grow0, int D, int K, const double* syn_model,
                  uint64_t seed, cudaStream_t s, LaunchStats& ls) {
    if (n <= 0) return;
    const int64_t g = (n + kBlock - 1) / kBlock;
    k_synth<<<(unsigned)g, kBlock, 0, s>>>(X, ld, n, grow0, D, K, syn_model, (uint32_t)seed, (uint32_t)(seed >> 32));
    ++ls.launches;
}

// ================================================================ layouts
// rows (row-major n x D) -> planar X[j*ld + row0 + i]; 128 rows per CTA.
__global__ void k_rows_to_planar(const double* __restrict__ rows, int64_t n, int D, double* __restrict__ X,
                                 int64_t ld, int64_t row0) {
    extern __shared__ double tile[];  // 128 x (D+1)
    const int64_t r0 = (int64_t)blockIdx.x * 128;
    const int nr = (int)min((int64_t)128, n - r0);
    for (int e = threadIdx.x; e < nr * D; e += blockDim.x) {
        const int i = e / D, j = e % D;
        tile[i * (D + 1) + j] = rows[(r0 + i) * D + j];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nr * D; e += blockDim.x) {
        const int j = e / nr, i = e % nr;
        X[(int64_t)j * ld + row0 + r0 + i] = tile[i * (D + 1) + j];
    }
}

void launch_rows_to_planar(const double* rows, int64_t n, int D, double* X, int64_t ld, int64_t row0,
                           cudaStream_t s, LaunchStats& ls) {
    if (n <= 0) return;
    static bool attr = false;
    if (!attr) {
        allow_max_smem(k_rows_to_planar);
        attr = true;
    }
    const int64_t g = (n + 127) / 128;
    k_rows_to_planar<<<(unsigned)g, kBlock, 128 * (D + 1) * sizeof(double), s>>>(rows, n, D, X, ld, row0);
    ++ls.launches;
}

__global__ void k_planar_to_rows(const double* __restrict__ X, int64_t ld, int D, int64_t row0, int64_t n,
                                 double* __restrict__ rows) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * D) return;
    const int64_t i = e / D;
    const int j = (int)(e % D);
    rows[e] = X[(int64_t)j * ld + row0 + i];
}

void launch_planar_to_rows(const double* X, int64_t ld, int D, int64_t row0, int64_t n, double* rows,
                           cudaStream_t s, LaunchStats& ls) {
    if (n <= 0) return;
    const int64_t g = (n * D + kBlock - 1) / kBlock;
    k_planar_to_rows<<<(unsigned)g, kBlock, 0, s>>>(X, ld, D, row0, n, rows);
    ++ls.launches;
}

// ============================================================ column stats
// grid (bx, D): plane j, rows strided by bx; scratch[(j*bx_total + b)*4 + {sum,min,max,nonfinite}]
__global__ void k_col_stats(const double* __restrict__ X, int64_t n, int64_t ld, double* __restrict__ scratch) {
    __shared__ double red[kBlock];
    const int j = blockIdx.y;
    const double* p = X + (int64_t)j * ld;
    double s = 0.0, mn = INFINITY, mx = -INFINITY, nf = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = p[i];
        if (!isfinite(v)) nf += 1.0;
        s += v;
        mn = fmin(mn, v);
        mx = fmax(mx, v);
    }
    double* o = scratch + ((int64_t)j * gridDim.x + blockIdx.x) * 4;
    const double bs = block_sum(s, red);
    const double bn = block_sum(nf, red);
    // min / max trees
    red[threadIdx.x] = mn;
    __syncthreads();
    for (int t = blockDim.x / 2; t > 0; t >>= 1) {
        if (threadIdx.x < t) red[threadIdx.x] = fmin(red[threadIdx.x], red[threadIdx.x + t]);
        __syncthreads();
    }
    const double bmn = red[0];
    __syncthreads();
    red[threadIdx.x] = mx;
    __syncthreads();
    for (int t = blockDim.x / 2; t > 0; t >>= 1) {
        if (threadIdx.x < t) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + t]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        o[0] = bs;
        o[1] = bmn;
        o[2] = red[0];
        o[3] = bn;
    }
}

__global__ void k_col_stats_reduce(const double* __restrict__ scratch, int nb, int D, double* __restrict__ out) {
    const int j = threadIdx.x;
    if (j >= D) return;
    double s = 0.0, mn = INFINITY, mx = -INFINITY, nf = 0.0;
    for (int b = 0; b < nb; ++b) {
        const double* o = scratch + ((int64_t)j * nb + b) * 4;
        s += o[0];
        mn = fmin(mn, o[1]);
        mx = fmax(mx, o[2]);
        nf += o[3];
    }
    out[j] = s;
    out[D + j] = mn;
    out[2 * D + j] = mx;
    out[3 * D + j] = nf;
}

void launch_col_stats(const double* X, int64_t n, int64_t ld, int D, double* scratch, double* out, int num_sms,
                      cudaStream_t s, LaunchStats& ls) {
    const int bx = max(1, min(num_sms * 4 / max(D, 1) + 1, 1024));
    k_col_stats<<<dim3(bx, D), kBlock, 0, s>>>(X, n, ld, scratch);
    k_col_stats_reduce<<<1, 64, 0, s>>>(scratch, bx, D, out);
    ls.launches += 2;
}

// ======================================================= fixed-order reduce
// One warp per output entry: lane l sums blocks l, l + 32, ... in order, then a fixed xor
// tree across the lanes (deterministic; ~5 loads deep instead of a 148-long serial chain).
__global__ void k_reduce_blocks(const double* __restrict__ partial, int nblk, int len, double* __restrict__ out) {
    const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (e >= len) return;
    double s = 0.0;
#pragma unroll 4
    for (int b = lane; b < nblk; b += 32) s += partial[(int64_t)b * len + e];
    s = warp_sum(s);
    if (lane == 0) out[e] = s;
}

void launch_reduce_blocks(const double* partial, int nblk, int len, double* out, cudaStream_t s, LaunchStats& ls) {
    k_reduce_blocks<<<(len + 7) / 8, 256, 0, s>>>(partial, nblk, len, out);
    ++ls.launches;
}

// ========================================================== generic E + M
// Any D <= 64, K <= 128.  One tile of T events at a time: planar tile in
// smem, (event,k) work items for the E-step, per-event LSE, then every
// thread owns stat entries (k, r) and adds the tile's contribution into its
// CTA's private partial block.  Statistics in raw d = x - c_k coordinates.
template <bool UNIT>
__global__ void __launch_bounds__(kBlock) k_em_generic(const double* __restrict__ X, int64_t n, int64_t ld, int D,
                                                       int K, const double* __restrict__ model,
                                                       const double* __restrict__ centers,
                                                       double* __restrict__ partial, int T) {
    extern __shared__ double sm[];
    __shared__ double red[kBlock];
    const int TP = T + 1;
    double* xs = sm;            // D x TP
    double* gs = xs + D * TP;   // K x TP
    const int SK = stat_k(D);
    const int NE = K * SK;
    ModelView mv{K, D, const_cast<double*>(model)};
    double* myp = partial + (int64_t)blockIdx.x * (NE + 1);
    for (int e = threadIdx.x; e < NE + 1; e += blockDim.x) myp[e] = 0.0;
    double ll_acc = 0.0;
    __syncthreads();
    for (int64_t t0 = (int64_t)blockIdx.x * T; t0 < n; t0 += (int64_t)gridDim.x * T) {
        const int nt = (int)min((int64_t)T, n - t0);
        for (int e = threadIdx.x; e < D * T; e += blockDim.x) {
            const int j = e / T, t = e % T;
            xs[j * TP + t] = t < nt ? X[(int64_t)j * ld + t0 + t] : 0.0;
        }
        __syncthreads();
        if (!UNIT) {
            for (int e = threadIdx.x; e < K * T; e += blockDim.x) {
                const int k = e / T, t = e % T;
                if (t >= nt) continue;
                const double* W = mv.W() + (int64_t)k * D * D;
                const double* mu = mv.mu() + (int64_t)k * D;
                double q = 0.0;
                for (int r = 0; r < D; ++r) {
                    double z = 0.0;
                    for (int j = 0; j <= r; ++j) z = fma(W[r * D + j], xs[j * TP + t] - mu[j], z);
                    q = fma(z, z, q);
                }
                gs[k * TP + t] = mv.logpi()[k] + mv.lognorm()[k] - 0.5 * q;
            }
            __syncthreads();
            for (int t = threadIdx.x; t < nt; t += blockDim.x) {
                double m = -INFINITY;
                for (int k = 0; k < K; ++k) m = fmax(m, gs[k * TP + t]);
                double s = 0.0;
                for (int k = 0; k < K; ++k) s += exp(gs[k * TP + t] - m);
                const double ll = m + log(s);
                ll_acc += ll;
                for (int k = 0; k < K; ++k) gs[k * TP + t] = exp(gs[k * TP + t] - ll);
            }
            __syncthreads();
        }
        for (int e = threadIdx.x; e < NE; e += blockDim.x) {
            const int k = e / SK, r = e % SK;
            const double* c = centers + (int64_t)k * D;
            const double* g = gs + k * TP;
            double acc = 0.0;
            if (r == 0) {
                for (int t = 0; t < nt; ++t) acc += UNIT ? 1.0 : g[t];
            } else if (r <= D) {
                const int a = r - 1;
                const double ca = c[a];
                for (int t = 0; t < nt; ++t) acc = fma(UNIT ? 1.0 : g[t], xs[a * TP + t] - ca, acc);
            } else {
                int b;
                const int a = decode_pair(r - 1 - D, D, &b);
                const double ca = c[a], cb = c[b];
                for (int t = 0; t < nt; ++t)
                    acc = fma((UNIT ? 1.0 : g[t]) * (xs[a * TP + t] - ca), xs[b * TP + t] - cb, acc);
            }
            myp[e] += acc;
        }
        __syncthreads();
    }
    const double bl = block_sum(ll_acc, red);
    if (threadIdx.x == 0) myp[NE] = bl;
}

static int generic_tile(int D, int K) {
    int T = 12288 / (D + K);  // (D+K)*(T+1)*8 bytes <= ~96 KB
    T = max(16, min(256, T));
    return T;
}

// ================================================================ team path
// Team of TS = next_pow2(K*H) lanes per event; lane tl -> (k = tl/H, h = tl%H).
// DM = padded dimension (multiple of 4); H in {1,2}.
template <int DM, int H>
struct TeamCfg {
    static constexpr int HALF = DM / 2;
    static constexpr int P = DM * (DM + 1) / 2;
    static constexpr int PH = HALF * (HALF + 1) / 2;
    static constexpr int NACC = (H == 1) ? (1 + DM + P) : (1 + HALF + 2 * PH);
    static constexpr int WS = DM * DM + 2;   // W stride (doubles): 16-byte skew between components
    static constexpr int MS = DM + 2;        // mu stride
};

__host__ __device__ inline int next_pow2(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}

// Stage W_k (padded DM x DM, zeros outside D), mu_k, logpi, lognorm into smem.
template <int DM, int H>
__device__ void team_stage(const ModelView& mv, double* sW, double* sMu, double* sC) {
    using C = TeamCfg<DM, H>;
    const int K = mv.K, D = mv.D;
    for (int e = threadIdx.x; e < K * DM * DM; e += blockDim.x) {
        const int k = e / (DM * DM), rc = e % (DM * DM), r = rc / DM, c = rc % DM;
        sW[k * C::WS + rc] = (r < D && c < D) ? mv.W()[(int64_t)k * D * D + r * D + c] : 0.0;
    }
    for (int e = threadIdx.x; e < K * DM; e += blockDim.x) {
        const int k = e / DM, c = e % DM;
        sMu[k * C::MS + c] = c < D ? mv.mu()[k * D + c] : 0.0;
    }
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
        sC[2 * k] = mv.logpi()[k];
        sC[2 * k + 1] = mv.lognorm()[k];
    }
}

// Whitening of one event against component k: returns q = ||W_k (x - mu_k)||^2
// and leaves z (H==1: all DM coordinates; H==2: assembled after exchange) in z[].
template <int DM, int H>
__device__ __forceinline__ double team_whiten(const double* __restrict__ Wk, const double* __restrict__ muk,
                                              const double (&x)[DM], double (&z)[DM], int h) {
    double d[DM];
#pragma unroll
    for (int j = 0; j < DM; j += 2) {
        const double2 m = *reinterpret_cast<const double2*>(muk + j);
        d[j] = x[j] - m.x;
        d[j + 1] = x[j + 1] - m.y;
    }
    if constexpr (H == 1) {
        double q = 0.0;
#pragma unroll
        for (int r = DM - 1; r >= 0; --r) {
            const double* Wr = Wk + r * DM;
            double acc = 0.0;
#pragma unroll
            for (int j = 0; j <= r; j += 2) {
                const double2 w = *reinterpret_cast<const double2*>(Wr + j);
                acc = fma(w.x, d[j], acc);
                if (j + 1 <= r) acc = fma(w.y, d[j + 1], acc);
            }
            z[r] = acc;
        }
#pragma unroll
        for (int r = 0; r < DM; ++r) q = fma(z[r], z[r], q);
        return q;
    } else {
        // rows owned: 4m+h and 4m+3-h (balanced: 2(4m+4) multiply-adds per block m)
        double zo[DM / 2];
        double qo = 0.0;
#pragma unroll
        for (int m = 0; m < DM / 4; ++m) {
            const double* W0 = Wk + (4 * m + h) * DM;
            const double* W1 = Wk + (4 * m + 3 - h) * DM;
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int j = 0; j < 4 * m + 4; j += 2) {
                const double2 w0 = *reinterpret_cast<const double2*>(W0 + j);
                const double2 w1 = *reinterpret_cast<const double2*>(W1 + j);
                a0 = fma(w0.x, d[j], a0);
                a0 = fma(w0.y, d[j + 1], a0);
                a1 = fma(w1.x, d[j], a1);
                a1 = fma(w1.y, d[j + 1], a1);
            }
            zo[2 * m] = a0;
            zo[2 * m + 1] = a1;
            qo = fma(a0, a0, qo);
            qo = fma(a1, a1, qo);
        }
        const double q = qo + __shfl_xor_sync(0xffffffffu, qo, 1);
#pragma unroll
        for (int m = 0; m < DM / 4; ++m) {
            const double p0 = __shfl_xor_sync(0xffffffffu, zo[2 * m], 1);
            const double p1 = __shfl_xor_sync(0xffffffffu, zo[2 * m + 1], 1);
            z[4 * m + 0] = h ? p0 : zo[2 * m];
            z[4 * m + 3] = h ? p1 : zo[2 * m + 1];
            z[4 * m + 1] = h ? zo[2 * m] : p0;
            z[4 * m + 2] = h ? zo[2 * m + 1] : p1;
        }
        return q;
    }
}

// Team log-sum-exp / argmax over components (butterfly on lane offsets H..TS/2;
// commutative adds make every lane's result bit-identical).
struct TeamLse {
    double ll;
    int predict;
    int best;
    double best_ld;
};

template <int H>
__device__ __forceinline__ TeamLse team_lse(double w, double ln, int k, int TS) {
    double m = w;
    int am = k;
    double bl = ln;
    int ab = k;
    for (int off = H; off < TS; off <<= 1) {
        const double mo = __shfl_xor_sync(0xffffffffu, m, off);
        const int ao = __shfl_xor_sync(0xffffffffu, am, off);
        if (mo > m || (mo == m && ao < am)) {
            m = mo;
            am = ao;
        }
        const double bo = __shfl_xor_sync(0xffffffffu, bl, off);
        const int abo = __shfl_xor_sync(0xffffffffu, ab, off);
        if (bo > bl || (bo == bl && abo < ab)) {
            bl = bo;
            ab = abo;
        }
    }
    double s = (w == -INFINITY) ? 0.0 : exp(w - m);
    for (int off = H; off < TS; off <<= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    return TeamLse{m + log(s), am, ab, bl};
}

// Accumulator index of global stat entry r of component k for team role h;
// -1 if role h does not own it.  (Inverse of the accumulation pattern below.)
template <int DM, int H>
__host__ __device__ int team_source(int r, int D, int h) {
    using C = TeamCfg<DM, H>;
    if (H == 1) {
        if (r <= D) return r;  // N, s1[a] = acc[1+a]
        int b, p = r - 1 - D, a = 0;
        while (p >= D - a) {
            p -= D - a;
            ++a;
        }
        b = a + p;
        return 1 + DM + (a * DM - (a * (a - 1)) / 2 + (b - a));
    } else {
        const int HF = C::HALF;
        if (r == 0) return h == 0 ? 0 : -1;
        if (r <= D) {
            const int a = r - 1;
            if (a < HF) return h == 0 ? 1 + a : -1;
            return h == 1 ? 1 + (a - HF) : -1;
        }
        int p = r - 1 - D, a = 0;
        while (p >= D - a) {
            p -= D - a;
            ++a;
        }
        const int b = a + p;
        auto pk = [&](int x, int y) { return x * HF - (x * (x - 1)) / 2 + (y - x); };
        if (b < HF) return h == 0 ? 1 + HF + pk(a, b) : -1;
        if (a >= HF) return h == 1 ? 1 + HF + pk(a - HF, b - HF) : -1;
        const int c = b - HF;
        if (c >= a) return h == 0 ? 1 + HF + C::PH + pk(a, c) : -1;
        return h == 1 ? 1 + HF + C::PH + pk(c, a) : -1;
    }
}

template <int DM, int H>
__global__ void __launch_bounds__(kBlock, 1) k_em_team(const double* __restrict__ X, int64_t n, int64_t ld, int D,
                                                        int K, const double* __restrict__ model,
                                                        double* __restrict__ partial) {
    using C = TeamCfg<DM, H>;
    extern __shared__ __align__(16) double sm[];
    double* sW = sm;                       // K * WS
    double* sMu = sW + K * C::WS;          // K * MS
    double* sC = sMu + K * C::MS;          // 2K (+pad)
    double* sRed = sm;  // 8 * TS * NACC, aliases the staged model after the event loop
    const int TS = next_pow2(K * H);
    const int EPW = 32 / TS;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tl = lane % TS, slot = lane / TS;
    const int k = tl / H, h = tl % H;
    const bool kact = k < K;
    const int kk = kact ? k : 0;
    ModelView mv{K, D, const_cast<double*>(model)};
    team_stage<DM, H>(mv, sW, sMu, sC);
    __syncthreads();
    const double* Wk = sW + kk * C::WS;
    const double* muk = sMu + kk * C::MS;
    const double logpi = kact ? sC[2 * kk] : -INFINITY;
    const double lognorm = sC[2 * kk + 1];

    double acc[C::NACC];
#pragma unroll
    for (int j = 0; j < C::NACC; ++j) acc[j] = 0.0;
    double ll_acc = 0.0;

    for (int64_t it = 0;; ++it) {
        const int64_t wbase = ((it * gridDim.x + blockIdx.x) * 8 + warp) * EPW;
        if (wbase >= n) break;
        const int64_t i = wbase + slot;
        const bool valid = i < n;
        double x[DM];
#pragma unroll
        for (int j = 0; j < DM; ++j) x[j] = (valid && j < D) ? __ldg(X + (int64_t)j * ld + i) : 0.0;
        double z[DM];
        const double q = team_whiten<DM, H>(Wk, muk, x, z, h);
        const double ln = lognorm - 0.5 * q;
        const double w = kact ? logpi + ln : -INFINITY;
        const TeamLse r = team_lse<H>(w, kact ? ln : -INFINITY, k, TS);
        const double g = (valid && kact) ? exp(w - r.ll) : 0.0;
        if (valid && tl == 0) ll_acc += r.ll;
        if constexpr (H == 1) {
            acc[0] += g;
            int p = 1 + DM;
#pragma unroll
            for (int a = 0; a < DM; ++a) {
                const double ga = g * z[a];
                acc[1 + a] += ga;
#pragma unroll
                for (int b = a; b < DM; ++b) {
                    acc[p] = fma(ga, z[b], acc[p]);
                    ++p;
                }
            }
        } else {
            constexpr int HF = C::HALF;
            double u[DM];
#pragma unroll
            for (int j = 0; j < DM; ++j) u[j] = h ? z[(j + HF) % DM] : z[j];
            acc[0] += g;
            int p = 1 + HF;
            int o = 1 + HF + C::PH;
#pragma unroll
            for (int a = 0; a < HF; ++a) {
                const double ga = g * u[a];
                acc[1 + a] += ga;
#pragma unroll
                for (int b = a; b < HF; ++b) {
                    acc[p] = fma(ga, u[b], acc[p]);
                    ++p;
                }
#pragma unroll
                for (int c = a; c < HF; ++c) {
                    acc[o] = fma(ga, u[HF + c], acc[o]);
                    ++o;
                }
            }
        }
    }
    // ---- reduction: slots within the warp (butterfly), then warps in order
    __syncthreads();  // every warp is done with the staged model: sRed may alias it
#pragma unroll
    for (int j = 0; j < C::NACC; ++j)
        for (int off = TS; off < 32; off <<= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], off);
    for (int off = TS; off < 32; off <<= 1) ll_acc += __shfl_xor_sync(0xffffffffu, ll_acc, off);
    if (slot == 0) {
        double* dst = sRed + ((int64_t)warp * TS + tl) * C::NACC;
#pragma unroll
        for (int j = 0; j < C::NACC; ++j) dst[j] = acc[j];
    }
    __shared__ double sLL[8];
    if (lane == 0) sLL[warp] = ll_acc;
    __syncthreads();
    const int SK = stat_k(D);
    const int NE = K * SK;
    double* myp = partial + (int64_t)blockIdx.x * (NE + 1);
    for (int e = threadIdx.x; e < NE; e += blockDim.x) {
        const int kc = e / SK, rr = e % SK;
        int src_h = 0, j = team_source<DM, H>(rr, D, 0);
        if (j < 0) {
            src_h = 1;
            j = team_source<DM, H>(rr, D, 1);
        }
        const int role = kc * H + src_h;
        double s = 0.0;
        for (int wv = 0; wv < 8; ++wv) s += sRed[((int64_t)wv * TS + role) * C::NACC + j];
        myp[e] = s;
    }
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int wv = 0; wv < 8; ++wv) s += sLL[wv];
        myp[NE] = s;
    }
}

template <int DM>
__global__ void __launch_bounds__(kBlock) k_score_team(const double* __restrict__ X, int64_t n, int64_t ld, int D,
                                                        int K, const double* __restrict__ model, ScoreOut o,
                                                        double* __restrict__ blocksum) {
    using C = TeamCfg<DM, 1>;
    extern __shared__ __align__(16) double sm[];
    __shared__ double red[kBlock];
    double* sW = sm;
    double* sMu = sW + K * C::WS;
    double* sC = sMu + K * C::MS;
    const int TS = next_pow2(K);
    const int EPW = 32 / TS;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tl = lane % TS, slot = lane / TS;
    const int k = tl;
    const bool kact = k < K;
    const int kk = kact ? k : 0;
    ModelView mv{K, D, const_cast<double*>(model)};
    team_stage<DM, 1>(mv, sW, sMu, sC);
    __syncthreads();
    const double* Wk = sW + kk * C::WS;
    const double* muk = sMu + kk * C::MS;
    const double logpi = kact ? sC[2 * kk] : -INFINITY;
    const double lognorm = sC[2 * kk + 1];
    double ll_acc = 0.0, nflag = 0.0;
    for (int64_t it = 0;; ++it) {
        const int64_t wbase = ((it * gridDim.x + blockIdx.x) * 8 + warp) * EPW;
        if (wbase >= n) break;
        const int64_t i = wbase + slot;
        const bool valid = i < n;
        double x[DM];
#pragma unroll
        for (int j = 0; j < DM; ++j) x[j] = (valid && j < D) ? __ldg(X + (int64_t)j * ld + i) : 0.0;
        double z[DM];
        const double q = team_whiten<DM, 1>(Wk, muk, x, z, 0);
        const double ln = lognorm - 0.5 * q;
        const double w = kact ? logpi + ln : -INFINITY;
        const TeamLse r = team_lse<1>(w, kact ? ln : -INFINITY, k, TS);
        if (!valid) continue;
        if (kact) {
            if (o.gamma) o.gamma[i * K + k] = exp(w - r.ll);
            if (o.lnk) o.lnk[i * K + k] = ln;
        }
        if (tl == 0) {
            ll_acc += r.ll;
            const uint8_t f = ((o.mode == 1) ? r.ll : r.best_ld) < o.log_delta ? 1 : 0;
            nflag += f;
            if (o.ll) o.ll[i] = r.ll;
            if (o.predict) o.predict[i] = r.predict;
            if (o.best_k) o.best_k[i] = r.best;
            if (o.best_ld) o.best_ld[i] = r.best_ld;
            if (o.flags) o.flags[i] = f;
        }
    }
    const double a = block_sum(ll_acc, red);
    const double b = block_sum(nflag, red);
    if (threadIdx.x == 0) {
        blocksum[2 * blockIdx.x] = a;
        blocksum[2 * blockIdx.x + 1] = b;
    }
}

// Generic scorer: thread per event, any D <= 64, K <= 128 (slow path).
__device__ double gen_lnk(const ModelView& mv, const double* X, int64_t ld, int64_t i, int k) {
    const int D = mv.D;
    const double* W = mv.W() + (int64_t)k * D * D;
    const double* mu = mv.mu() + (int64_t)k * D;
    double q = 0.0;
    for (int r = 0; r < D; ++r) {
        double z = 0.0;
        for (int j = 0; j <= r; ++j) z = fma(W[r * D + j], X[(int64_t)j * ld + i] - mu[j], z);
        q = fma(z, z, q);
    }
    return mv.lognorm()[k] - 0.5 * q;
}

__global__ void __launch_bounds__(kBlock) k_score_generic(const double* __restrict__ X, int64_t n, int64_t ld, int D,
                                                           int K, const double* __restrict__ model, ScoreOut o,
                                                           double* __restrict__ blocksum) {
    __shared__ double red[kBlock];
    ModelView mv{K, D, const_cast<double*>(model)};
    double ll_acc = 0.0, nflag = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double m = -INFINITY, bl = -INFINITY;
        int am = 0, ab = 0;
        for (int k = 0; k < K; ++k) {
            const double ln = gen_lnk(mv, X, ld, i, k);
            const double w = mv.logpi()[k] + ln;
            if (o.lnk) o.lnk[i * K + k] = ln;
            if (w > m) { m = w; am = k; }
            if (ln > bl) { bl = ln; ab = k; }
        }
        double s = 0.0;
        for (int k = 0; k < K; ++k) s += exp(mv.logpi()[k] + gen_lnk(mv, X, ld, i, k) - m);
        const double ll = m + log(s);
        if (o.gamma)
            for (int k = 0; k < K; ++k) o.gamma[i * K + k] = exp(mv.logpi()[k] + gen_lnk(mv, X, ld, i, k) - ll);
        ll_acc += ll;
        const uint8_t f = ((o.mode == 1) ? ll : bl) < o.log_delta ? 1 : 0;
        nflag += f;
        if (o.ll) o.ll[i] = ll;
        if (o.predict) o.predict[i] = am;
        if (o.best_k) o.best_k[i] = ab;
        if (o.best_ld) o.best_ld[i] = bl;
        if (o.flags) o.flags[i] = f;
    }
    const double a = block_sum(ll_acc, red);
    const double b = block_sum(nflag, red);
    if (threadIdx.x == 0) {
        blocksum[2 * blockIdx.x] = a;
        blocksum[2 * blockIdx.x + 1] = b;
    }
}

// ------------------------------------------------------------ dispatch
EmPath em_path(int D, int K) {
    if (D <= 4 && K <= 32) return EmPath::Team4;
    if (D <= 8 && K <= 32) return EmPath::Team8;
    if (D <= 16 && K <= 16) return EmPath::Team16;
    return EmPath::Generic;
}

template <int DM, int H>
static size_t team_smem(int K, bool em) {
    using C = TeamCfg<DM, H>;
    size_t s = (size_t)K * C::WS + (size_t)K * C::MS + ((2 * K + 1) & ~1);
    if (em) s = s > (size_t)8 * next_pow2(K * H) * C::NACC ? s : (size_t)8 * next_pow2(K * H) * C::NACC;
    return s * sizeof(double);
}

template <int DM, int H>
static void set_team_attrs(int K) {
    static bool done = false;
    if (!done) {
        allow_max_smem(k_em_team<DM, H>);
        done = true;
    }
    (void)K;
}

int em_grid(int D, int K, int num_sms) {
    switch (em_path(D, K)) {
        case EmPath::Generic: return num_sms * 2;
        default: return num_sms;  // one register-heavy CTA per SM
    }
}

template <int DM, int H>
static void run_em_team(const double* X, int64_t n, int64_t ld, int D, int K, const double* model, double* partial,
                        int grid, cudaStream_t s) {
    set_team_attrs<DM, H>(K);
    k_em_team<DM, H><<<grid, kBlock, team_smem<DM, H>(K, true), s>>>(X, n, ld, D, K, model, partial);
}

void launch_em_pass(const double* X, int64_t n, int64_t ld, int D, int K, const double* model, double* partial,
                    int num_sms, int* nblk, bool* whitened, cudaStream_t s, LaunchStats& ls) {
    const int grid = em_grid(D, K, num_sms);
    *nblk = grid;
    *whitened = true;
    switch (em_path(D, K)) {
        case EmPath::Team4: run_em_team<4, 1>(X, n, ld, D, K, model, partial, grid, s); break;
        case EmPath::Team8: run_em_team<8, 1>(X, n, ld, D, K, model, partial, grid, s); break;
        case EmPath::Team16: run_em_team<16, 2>(X, n, ld, D, K, model, partial, grid, s); break;
        case EmPath::Generic: {
            *whitened = false;
            const int T = generic_tile(D, K);
            const size_t smem = (size_t)(D + K) * (T + 1) * sizeof(double);
            static bool attr = false;
            if (!attr) {
                allow_max_smem(k_em_generic<false>);
                allow_max_smem(k_em_generic<true>);
                attr = true;
            }
            k_em_generic<false><<<grid, kBlock, smem, s>>>(X, n, ld, D, K, model, model + 3 * K, partial, T);
            break;
        }
    }
    ++ls.launches;
}

// Unit-weight statistics about `center` for D <= 16 on the FP64 tensor pipe: per warp, a
// contiguous event range; per 4 events one mma.sync m8n8k4 f64 k-step of the Gram
// G = D^T D (D = centred rows), blocks (0,0), (0,1), (1,1) of the 16 x 16 matrix; the A and
// B fragments are the same loaded values (thread t: feature t/4 + 8 m, event t%4).  Four
// k-steps in flight per warp (independent accumulators).  FP64 products and sums.
__global__ void __launch_bounds__(256) k_unit_gram(const double* __restrict__ X, int64_t n, int64_t ld, int D,
                                                    const double* __restrict__ center, double* __restrict__ partial) {
    constexpr int U = 4;
    __shared__ double red[8][16 * 16 + 16];
    const int t = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * 8 + warp, nw = (int64_t)gridDim.x * 8;
    const int64_t chunk = ((n + nw - 1) / nw + 4 * U - 1) / (4 * U) * (4 * U);
    const int64_t e0 = gw * chunk, e1 = min(n, e0 + chunk);
    const int f0 = t >> 2, f1 = f0 + 8, ev = t & 3;
    const double c0 = f0 < D ? center[f0] : 0.0, c1 = f1 < D ? center[f1] : 0.0;
    const double* x0 = X + (int64_t)f0 * ld;
    const double* x1 = X + (int64_t)f1 * ld;
    double acc[U][3][2];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
        for (int b = 0; b < 3; ++b) acc[u][b][0] = acc[u][b][1] = 0.0;
    double s0 = 0.0, s1 = 0.0;
    for (int64_t e = e0; e < e1; e += 4 * U) {
        double d0[U], d1[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = e + 4 * u + ev;
            const bool ok = i < e1;
            d0[u] = (ok && f0 < D) ? __ldg(x0 + i) - c0 : 0.0;
            d1[u] = (ok && f1 < D) ? __ldg(x1 + i) - c1 : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            s0 += d0[u];
            s1 += d1[u];
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[u][0][0]), "+d"(acc[u][0][1]) : "d"(d0[u]), "d"(d0[u]));
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[u][1][0]), "+d"(acc[u][1][1]) : "d"(d0[u]), "d"(d1[u]));
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[u][2][0]), "+d"(acc[u][2][1]) : "d"(d1[u]), "d"(d1[u]));
        }
    }
    // C fragment: row f0 (+8), columns 2 (t & 3) + {0, 1} (+8); fixed-order sums
    double* r = red[warp];
    const int cn = 2 * (t & 3);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        double g00 = 0.0, g01 = 0.0, g11 = 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            g00 += acc[u][0][h];
            g01 += acc[u][1][h];
            g11 += acc[u][2][h];
        }
        r[f0 * 16 + cn + h] = g00;
        r[f0 * 16 + 8 + cn + h] = g01;
        r[(8 + cn + h) * 16 + f0] = g01;  // (1,0) = (0,1)^T
        r[f1 * 16 + 8 + cn + h] = g11;
    }
    s0 += __shfl_xor_sync(0xffffffffu, s0, 1);
    s0 += __shfl_xor_sync(0xffffffffu, s0, 2);
    s1 += __shfl_xor_sync(0xffffffffu, s1, 1);
    s1 += __shfl_xor_sync(0xffffffffu, s1, 2);
    if ((t & 3) == 0) {
        r[256 + f0] = s0;
        r[256 + f1] = s1;
    }
    __syncthreads();
    // block partial: [N | s1[D] | s2 packed upper | logL = 0]
    const int SK = stat_k(D);
    double* out = partial + (int64_t)blockIdx.x * (SK + 1);
    for (int j = threadIdx.x; j < SK + 1; j += blockDim.x) {
        double v = 0.0;
        if (j == 0) {
            for (int w = 0; w < 8; ++w) {
                const int64_t a = ((int64_t)blockIdx.x * 8 + w) * chunk;
                const int64_t lo = a < n ? a : n, hi = a + chunk < n ? a + chunk : n;
                v += (double)(hi - lo);
            }
        } else if (j <= D) {
            for (int w = 0; w < 8; ++w) v += red[w][256 + j - 1];
        } else if (j < SK) {
            int pp = j - 1 - D, a = 0;
            while (pp >= D - a) {
                pp -= D - a;
                ++a;
            }
            const int b = a + pp;
            for (int w = 0; w < 8; ++w) v += red[w][a * 16 + b];
        }
        out[j] = v;
    }
}

// Z[j][i] = (X[j][i] - mean[j]) * inv_scale[j], planar FP64 (run_pipeline standardization)
__global__ void k_standardize(const double* __restrict__ X, int64_t n, int64_t ld, int D,
                              const double* __restrict__ mean, const double* __restrict__ inv_scale,
                              double* __restrict__ Z, int64_t zld) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int j = blockIdx.y; j < D; j += gridDim.y) {
        const double m = mean[j], s = inv_scale[j];
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
            Z[(int64_t)j * zld + i] = (X[(int64_t)j * ld + i] - m) * s;
    }
}

void launch_standardize(const double* X, int64_t n, int64_t ld, int D, const double* mean, const double* inv_scale,
                        double* Z, int64_t zld, int num_sms, cudaStream_t s, LaunchStats& ls) {
    if (n <= 0) return;
    k_standardize<<<dim3(num_sms * 4, D), 256, 0, s>>>(X, n, ld, D, mean, inv_scale, Z, zld);
    ++ls.launches;
}

void launch_unit_stats(const double* X, int64_t n, int64_t ld, int D, const double* center, double* partial,
                       int num_sms, int* nblk, cudaStream_t s, LaunchStats& ls) {
    if (D <= 16) {
        const int grid = num_sms * 4;
        *nblk = grid;
        k_unit_gram<<<grid, 256, 0, s>>>(X, n, ld, D, center, partial);
        ++ls.launches;
        return;
    }
    const int grid = num_sms * 2;
    *nblk = grid;
    const int T = generic_tile(D, 1);
    const size_t smem = (size_t)(D + 1) * (T + 1) * sizeof(double);
    static bool attr = false;
    if (!attr) {
        allow_max_smem(k_em_generic<true>);
        attr = true;
    }
    k_em_generic<true><<<grid, kBlock, smem, s>>>(X, n, ld, D, 1, nullptr, center, partial, T);
    ++ls.launches;
}

int score_grid(int D, int K, int num_sms) {
    (void)D;
    (void)K;
    return num_sms * 4;
}

template <int DM>
static void run_score_team(const double* X, int64_t n, int64_t ld, int D, int K, const double* model,
                           const ScoreOut& o, double* blocksum, int grid, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        allow_max_smem(k_score_team<DM>);
        attr = true;
    }
    k_score_team<DM><<<grid, kBlock, team_smem<DM, 1>(K, false), s>>>(X, n, ld, D, K, model, o, blocksum);
}

void launch_score(const double* X, int64_t n, int64_t ld, int D, int K, const double* model, const ScoreOut& o,
                  double* blocksum, int num_sms, int* nblk, cudaStream_t s, LaunchStats& ls) {
    const int grid = score_grid(D, K, num_sms);
    *nblk = grid;
    // the team kernels keep every component's W in shared memory: beyond the opt-in limit
    // (D = 32 with K > 26) the generic kernel reads the model from global memory
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (K <= 32 && D <= 4) run_score_team<4>(X, n, ld, D, K, model, o, blocksum, grid, s);
    else if (K <= 32 && D <= 8) run_score_team<8>(X, n, ld, D, K, model, o, blocksum, grid, s);
    else if (K <= 32 && D <= 16) run_score_team<16>(X, n, ld, D, K, model, o, blocksum, grid, s);
    else if (K <= 32 && D <= 32 && team_smem<32, 1>(K, false) <= (size_t)optin)
        run_score_team<32>(X, n, ld, D, K, model, o, blocksum, grid, s);
    else k_score_generic<<<grid, kBlock, 0, s>>>(X, n, ld, D, K, model, o, blocksum);
    ++ls.launches;
}

// ================================================== diagonal covariance
// Extension (not in the reference: SPEC.md:332).  Team of
// TS = next_pow2(K) lanes per event, lane k evaluates component k
// (q = sum_a (x_a - mu_ka)^2 / sigma2_ka) and accumulates its 2D+1 statistics
// about c_k = mu_k(old) in FP64 registers.  Statistics use the canonical
// packed layout with only the diagonal of s2 populated (finalize in diag mode).
constexpr int DTILE = kBlock;  // events per staged tile of k_em_diag (one per thread)

template <int DM>
__global__ void __launch_bounds__(kBlock, DM <= 16 ? 2 : 1) k_em_diag(const double* __restrict__ X, int64_t n, int64_t ld, int D, int K,
                                                   const double* __restrict__ model, double* __restrict__ partial) {
    extern __shared__ __align__(16) double sm[];
    const int MS = DM + 1;
    double* sMu = sm;                 // K * MS
    double* sP = sMu + K * MS;        // K * MS  (precisions 1/sigma^2)
    double* sC = sP + K * MS;         // 2K: logpi, lognorm
    double* sX = sC + 2 * K;          // [DM][DTILE] staged event tile (coalesced loads)
    const int TS = next_pow2(K);
    const int EPW = 32 / TS;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tl = lane % TS, slot = lane / TS;
    const int k = tl;
    const bool kact = k < K;
    const int kk = kact ? k : 0;
    ModelView mv{K, D, const_cast<double*>(model)};
    for (int e = threadIdx.x; e < K * DM; e += blockDim.x) {
        const int c = e / DM, j = e % DM;
        sMu[c * MS + j] = j < D ? mv.mu()[c * D + j] : 0.0;
        sP[c * MS + j] = j < D ? 1.0 / mv.cov()[(int64_t)c * D * D + j * D + j] : 0.0;
    }
    for (int c = threadIdx.x; c < K; c += blockDim.x) {
        sC[2 * c] = mv.logpi()[c];
        sC[2 * c + 1] = mv.lognorm()[c];
    }
    __syncthreads();
    const double* muk = sMu + kk * MS;
    const double* pk = sP + kk * MS;
    const double logpi = kact ? sC[2 * kk] : -INFINITY;
    const double lognorm = sC[2 * kk + 1];
    constexpr int NA = 1 + 2 * DM;
    double acc[NA];
#pragma unroll
    for (int j = 0; j < NA; ++j) acc[j] = 0.0;
    double ll_acc = 0.0;
    // tiles of DTILE events: staged into shared memory with coalesced loads (thread t loads
    // event t of the tile, every feature), the next tile prefetched into registers while
    // this one is evaluated; inside a tile, warp w / slot s take events (r * 8 + w) * EPW + s
    constexpr bool PF = DM <= 16;
    double pf[PF ? DM : 1];
    const int64_t ntl = (n + DTILE - 1) / DTILE;
    auto fetch = [&](int64_t tl_idx, double* dst) {
        const int64_t i = tl_idx * DTILE + threadIdx.x;
#pragma unroll
        for (int j = 0; j < DM; ++j) dst[j] = (i < n && j < D) ? __ldg(X + (int64_t)j * ld + i) : 0.0;
    };
    if (PF && blockIdx.x < ntl) fetch(blockIdx.x, pf);
    for (int64_t tt = blockIdx.x; tt < ntl; tt += gridDim.x) {
        __syncthreads();  // the previous tile is consumed
        if (PF) {
#pragma unroll
            for (int j = 0; j < DM; ++j) sX[j * DTILE + threadIdx.x] = pf[j];
        } else {
            double tmp[DM];
            fetch(tt, tmp);
#pragma unroll
            for (int j = 0; j < DM; ++j) sX[j * DTILE + threadIdx.x] = tmp[j];
        }
        __syncthreads();
        if (PF && tt + gridDim.x < ntl) fetch(tt + gridDim.x, pf);
      for (int rr = 0; rr < DTILE / (8 * EPW); ++rr) {
        const int le = (rr * 8 + warp) * EPW + slot;
        const int64_t i = tt * DTILE + le;
        const bool valid = i < n;
        double d[DM];
        double q = 0.0;
#pragma unroll
        for (int j = 0; j < DM; ++j) {
            const double x = sX[j * DTILE + le];
            d[j] = (j < D) ? x - muk[j] : 0.0;
            q = fma(d[j] * d[j], pk[j], q);
        }
        const double ln = lognorm - 0.5 * q;
        const double w = kact ? logpi + ln : -INFINITY;
        // team log-sum-exp; gamma = exp(w - m) / sum (one FP64 exp per lane)
        double m = w;
        for (int off = 1; off < TS; off <<= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
        const double e = kact ? exp(w - m) : 0.0;
        double ssum = e;
        for (int off = 1; off < TS; off <<= 1) ssum += __shfl_xor_sync(0xffffffffu, ssum, off);
        const double g = (valid && kact) ? e / ssum : 0.0;
        if (valid && tl == 0) ll_acc += m + log(ssum);
        acc[0] += g;
#pragma unroll
        for (int j = 0; j < DM; ++j) {
            const double gd = g * d[j];
            acc[1 + j] += gd;
            acc[1 + DM + j] = fma(gd, d[j], acc[1 + DM + j]);
        }
      }
    }
    // slots within the warp, then warps in order (fixed-order reduction)
#pragma unroll
    for (int j = 0; j < NA; ++j)
        for (int off = TS; off < 32; off <<= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], off);
    for (int off = TS; off < 32; off <<= 1) ll_acc += __shfl_xor_sync(0xffffffffu, ll_acc, off);
    __syncthreads();
    double* sRed = sm;  // reuse: 8 warps x TS lanes x NA
    if (slot == 0) {
#pragma unroll
        for (int j = 0; j < NA; ++j) sRed[((int64_t)warp * TS + tl) * NA + j] = acc[j];
    }
    __shared__ double sLL[8];
    if (lane == 0) sLL[warp] = ll_acc;
    __syncthreads();
    const int SK = stat_k(D), NE = K * SK;
    double* myp = partial + (int64_t)blockIdx.x * (NE + 1);
    for (int e = threadIdx.x; e < NE; e += blockDim.x) {
        const int c = e / SK, rr = e % SK;
        int j = -1;
        if (rr <= D) {
            j = rr;  // N, s1
        } else {
            int p2 = rr - 1 - D, a = 0;
            while (p2 >= D - a) {
                p2 -= D - a;
                ++a;
            }
            if (p2 == 0) j = 1 + DM + a;  // diagonal entry (a, a)
        }
        double v = 0.0;
        if (j >= 0)
            for (int wv = 0; wv < 8; ++wv) v += sRed[((int64_t)wv * TS + c) * NA + j];
        myp[e] = v;
    }
    if (threadIdx.x == 0) {
        double v = 0.0;
        for (int wv = 0; wv < 8; ++wv) v += sLL[wv];
        myp[NE] = v;
    }
}

void launch_em_diag(const double* X, int64_t n, int64_t ld, int D, int K, const double* model, double* partial,
                    int num_sms, int* nblk, cudaStream_t s, LaunchStats& ls) {
    const int grid = num_sms * 2;
    *nblk = grid;
    const int TS = next_pow2(K);
    auto smem_for = [&](int DM) {
        const size_t a = (size_t)(2 * K * (DM + 1) + 2 * K + DM * DTILE) * sizeof(double);
        const size_t b = (size_t)8 * TS * (1 + 2 * DM) * sizeof(double);
        return a > b ? a : b;
    };
    if (D <= 8) {
        static bool at = false;
        if (!at) { allow_max_smem(k_em_diag<8>); at = true; }
        k_em_diag<8><<<grid, kBlock, smem_for(8), s>>>(X, n, ld, D, K, model, partial);
    } else if (D <= 16) {
        static bool at = false;
        if (!at) { allow_max_smem(k_em_diag<16>); at = true; }
        k_em_diag<16><<<grid, kBlock, smem_for(16), s>>>(X, n, ld, D, K, model, partial);
    } else {
        static bool at = false;
        if (!at) { allow_max_smem(k_em_diag<32>); at = true; }
        k_em_diag<32><<<grid, kBlock, smem_for(32), s>>>(X, n, ld, D, K, model, partial);
    }
    ++ls.launches;
}

// ======================================================= finalize / derive
// Warp-cooperative Cholesky + inverse of the D x D matrix in A (smem).
// Writes L, W = L^-1 (smem) and returns logdet in lane 0; false if not PD.
// Cholesky A = L L^T and W = L^-1 of a D x D SPD matrix by one warp.  A, L, W in shared
// memory with row stride ld >= D + 1 (an odd stride in doubles keeps the lanes' rows on
// distinct banks); column D of L is scratch (1 / L_jj).  Returns false on a numerically
// singular pivot (the oracle's rule).

// Per-component derive from pi, mu, cov (block per component, warp 0 works).
__device__ void derive_component(ModelView mv, int k, double* sA, double* sL, double* sW, IterStatus* st) {
    const int D = mv.D, ld = D + 1;
    for (int e = threadIdx.x; e < D * D; e += blockDim.x) sA[(e / D) * ld + e % D] = mv.cov()[(int64_t)k * D * D + e];
    __syncthreads();
    {
        __shared__ double csc[2];
        double logdet = 0.0;
        const bool ok = chol_inv_any(sA, sL, sW, D, ld, &logdet, csc);
        if (threadIdx.x == 0) {
            if (!ok) atomicAdd(&st->not_pd, 1);
            mv.lognorm()[k] = -0.5 * logdet - 0.5 * D * kLog2Pi;
            mv.logpi()[k] = log(mv.pi()[k]);
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < D * D; e += blockDim.x) {
        mv.L()[(int64_t)k * D * D + e] = sL[(e / D) * ld + e % D];
        mv.W()[(int64_t)k * D * D + e] = sW[(e / D) * ld + e % D];
    }
}

__global__ void k_derive(double* model, int D, int K, IterStatus* st) {
    extern __shared__ double sm[];
    ModelView mv{K, D, model};
    const int m = D * (D + 1);
    derive_component(mv, blockIdx.x, sm, sm + m, sm + 2 * m, st);
}

void launch_derive(double* model, int D, int K, IterStatus* st, cudaStream_t s, LaunchStats& ls) {
    static bool attr = false;  // 3 D^2 doubles: 96 KB at D = 64 (opt-in above 48 KB)
    if (!attr) {
        allow_max_smem(k_derive);
        attr = true;
    }
    k_derive<<<K, 128, 3 * D * (D + 1) * sizeof(double), s>>>(model, D, K, st);
    ++ls.launches;
}

// M-step from the shifted statistics about c_k = mu_k(old):
//   mu_new = c + T zbar,  Sigma_new = T (S2/N_k - zbar zbar^T) T^T + reg I
// with T = L_k (whitened statistics) or I (raw), zbar = s1 / N_k.
// whitened == 3: raw statistics about the centre c + fp32((mu_k - c) xs) / xs
// (k_em_mma's record centre), given `center` = c and `xs`.
// `model_in` is the model the EM pass used, `model_out` receives the new one (may alias
// model_in; distinct buffers let the host keep theta_t while iteration t + 1 is in flight).
// G > 0: G rank blocks of statistics, summed in rank order (grid K x 1).  G < 0: -G per-CTA
// partial blocks of one rank (world 1), summed in k_reduce_blocks' fixed order (one warp per
// entry, lanes over blocks, xor tree) by the gridDim.y CTAs of component k into `red`; the
// last of them to finish (ticket in tick[k], reset for the next launch) does the M-step.
constexpr int k_fin_warps = 8 * 2;  // partial-sum entries per finalize CTA (two per warp)
#ifdef ES_FIN_TRACE
// debug timeline (scripts/fin_trace.py): %globaltimer per (CTA, phase), thread 0
__device__ unsigned long long g_fin_tr[256][8];
#define FTR(i)                                                                                          \
    do {                                                                                                \
        if (threadIdx.x == 0) {                                                                         \
            unsigned long long v;                                                                       \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));                                        \
            g_fin_tr[(blockIdx.y * gridDim.x + blockIdx.x) & 255][i] = v;                               \
        }                                                                                               \
    } while (0)
#else
#define FTR(i) \
    do {       \
    } while (0)
#endif
__global__ void k_finalize(const double* __restrict__ stats, int G, int D, int K, int64_t n_global, double reg,
                           int whitened, const double* __restrict__ model_in, double* model_out,
                           IterRecord* st, double* record, int t, const double* __restrict__ center, double xs,
                           double* red, int* tick) {
    extern __shared__ double sm[];
    __shared__ int last;
    const int k = blockIdx.x;
    const int SK = stat_k(D), NE = K * SK, P = packed_size(D), LD = D + 1;
    ModelView mv{K, D, const_cast<double*>(model_in)};
    ModelView mo{K, D, model_out};
    FTR(0);
    double* sS = sm;                 // SK   (summed statistics of component k)
    double* sM = sS + SK;            // D*D
    double* sT = sM + D * D;         // D*D  (T M)
    double* sA = sT + D * D;         // D*LD (new Sigma)
    double* sL = sA + D * LD;        // D*LD
    double* sW = sL + D * LD;        // D*LD
    double* sMu = sW + D * LD;       // D
    if (G > 0) {
        for (int e = threadIdx.x; e < SK; e += blockDim.x) {
            double v = 0.0;
            for (int g = 0; g < G; ++g) v += stats[(int64_t)g * (NE + 1) + k * SK + e];
            sS[e] = v;
        }
        if (k == 0 && threadIdx.x == 0) {
            double L = 0.0;
            for (int g = 0; g < G; ++g) L += stats[(int64_t)g * (NE + 1) + NE];
            st->logL = L;
            if (record) record[t] = L;
        }
    } else {
        const int nb = -G, lane = threadIdx.x & 31, nw = blockDim.x >> 5, R = gridDim.y;
        const int cnt = SK + (k == 0 ? 1 : 0);  // component 0 also sums logL (entry NE)
        for (int i = blockIdx.y * nw + (threadIdx.x >> 5); i < cnt; i += R * nw) {
            const int64_t col = i < SK ? (int64_t)k * SK + i : NE;
            double v = 0.0;
#pragma unroll 4
            for (int b = lane; b < nb; b += 32) v += stats[(int64_t)b * (NE + 1) + col];
            v = warp_sum(v);
            if (lane == 0) red[col] = v;
        }
        FTR(1);
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) {
            const int tk = atomicAdd(&tick[k], 1);
            last = tk == R - 1;
            if (last) tick[k] = 0;
        }
        __syncthreads();
        if (!last) return;
        FTR(2);
        __threadfence();
        for (int e = threadIdx.x; e < SK; e += blockDim.x) sS[e] = __ldcg(red + (int64_t)k * SK + e);
        if (k == 0 && threadIdx.x == 0) {
            const double L = __ldcg(red + NE);
            st->logL = L;
            if (record) record[t] = L;
        }
    }
    __syncthreads();
    const double Nk = sS[0];
    if (threadIdx.x == 0) st->nk[k] = Nk;
    if (!(Nk >= 1.0)) {  // collapse: N * pi_k < 1; host reseeds
        if (threadIdx.x == 0) st->flags[k] = 1;
        if (model_out != model_in) {  // carry component k over unchanged (the host reseeds it)
            if (threadIdx.x == 0) {
                mo.pi()[k] = mv.pi()[k];
                mo.logpi()[k] = mv.logpi()[k];
                mo.lognorm()[k] = mv.lognorm()[k];
            }
            for (int a = threadIdx.x; a < D; a += blockDim.x) mo.mu()[(int64_t)k * D + a] = mv.mu()[(int64_t)k * D + a];
            for (int e = threadIdx.x; e < D * D; e += blockDim.x) {
                const int64_t o = (int64_t)k * D * D + e;
                mo.cov()[o] = mv.cov()[o];
                mo.L()[o] = mv.L()[o];
                mo.W()[o] = mv.W()[o];
            }
        }
        return;
    }
    const double inv = 1.0 / Nk;
    const double* s1 = sS + 1;
    const double* s2 = sS + 1 + D;
    for (int e = threadIdx.x; e < D * D; e += blockDim.x) {
        const int a = e / D, b = e % D;
        const int x = min(a, b), y = max(a, b);
        sM[e] = s2[packed_index(x, y, D)] * inv - (s1[a] * inv) * (s1[b] * inv);
    }
    (void)P;
    __syncthreads();
    FTR(3);
    const double* Lold = mv.L() + (int64_t)k * D * D;
    const double* cold = mv.mu() + (int64_t)k * D;
    if (whitened == 1) {
        for (int e = threadIdx.x; e < D * D; e += blockDim.x) {
            const int a = e / D, b = e % D;
            double v = 0.0;
            for (int p = 0; p <= a; ++p) v = fma(Lold[a * D + p], sM[p * D + b], v);
            sT[e] = v;
        }
        for (int a = threadIdx.x; a < D; a += blockDim.x) {
            double v = 0.0;
            for (int p = 0; p <= a; ++p) v = fma(Lold[a * D + p], s1[p] * inv, v);
            sMu[a] = cold[a] + v;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < D * D; e += blockDim.x) {
            const int a = e / D, b = e % D;
            if (a > b) continue;
            double v = 0.0;
            for (int p = 0; p <= b; ++p) v = fma(sT[a * D + p], Lold[b * D + p], v);
            if (a == b) v += reg;
            sA[a * LD + b] = v;
            sA[b * LD + a] = v;
        }
    } else {
        for (int e = threadIdx.x; e < D * D; e += blockDim.x) {
            const int a = e / D, b = e % D;
            if (a > b) continue;
            const double v = ((whitened == 2 || whitened == 4) && a != b) ? 0.0 : sM[a * D + b] + (a == b ? reg : 0.0);
            sA[a * LD + b] = v;
            sA[b * LD + a] = v;
        }
        for (int a = threadIdx.x; a < D; a += blockDim.x) {
            double c0 = cold[a];
            if (whitened == 3 || whitened == 4) c0 = center[a] + (double)(float)((cold[a] - center[a]) * xs) / xs;
            sMu[a] = c0 + s1[a] * inv;
        }
    }
    __syncthreads();
    // write pi, mu, cov then derive L, W, lognorm, logpi
    __syncthreads();  // every read of model_in done (it may alias model_out)
    if (threadIdx.x == 0) mo.pi()[k] = Nk / (double)n_global;
    for (int a = threadIdx.x; a < D; a += blockDim.x) mo.mu()[(int64_t)k * D + a] = sMu[a];
    for (int e = threadIdx.x; e < D * D; e += blockDim.x) mo.cov()[(int64_t)k * D * D + e] = sA[(e / D) * LD + e % D];
    FTR(4);
    {
        __shared__ double csc[2];
        double logdet = 0.0;
        const bool ok = chol_inv_any(sA, sL, sW, D, LD, &logdet, csc);
        FTR(5);
        if (threadIdx.x == 0) {
            st->flags[k] = ok ? 0 : 2;
            mo.lognorm()[k] = -0.5 * logdet - 0.5 * D * kLog2Pi;
            mo.logpi()[k] = log(Nk / (double)n_global);
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < D * D; e += blockDim.x) {
        mo.L()[(int64_t)k * D * D + e] = sL[(e / D) * LD + e % D];
        mo.W()[(int64_t)k * D * D + e] = sW[(e / D) * LD + e % D];
    }
    FTR(6);
}

#ifdef ES_FIN_TRACE
extern "C" int es_debug_fin_trace(unsigned long long* out) {
    return (int)cudaMemcpyFromSymbol(out, g_fin_tr, sizeof(g_fin_tr));
}
#endif

void launch_finalize(const double* stats, int G, int D, int K, int64_t n_global, double reg, int whitened,
                     const double* model_in, double* model_out, IterRecord* st, double* record, int t,
                     cudaStream_t s, LaunchStats& ls, const double* center, double xs, double* red, int* tick) {
    const size_t smem = (size_t)(stat_k(D) + 2 * D * D + 3 * D * (D + 1) + D) * sizeof(double);
    static bool attr = false;
    if (!attr) {
        allow_max_smem(k_finalize);
        attr = true;
    }
    // per-CTA partials (G < 0): R CTAs of 8 warps per component, one entry per warp at a time
    const int R = G < 0 ? std::max(1, std::min(16, (stat_k(D) + (k_fin_warps - 1)) / k_fin_warps)) : 1;
    k_finalize<<<dim3(K, R), 256, smem, s>>>(stats, G, D, K, n_global, reg, whitened, model_in, model_out, st, record,
                                             t, center, xs, red, tick);
    ++ls.launches;
}

// ============================================================ radix select
__device__ __forceinline__ uint64_t ordkey(double v) {
    uint64_t u = (uint64_t)__double_as_longlong(v);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

__global__ void k_hist8(const double* __restrict__ keys, int64_t n, int shift, uint64_t pmask, uint64_t pval,
                        unsigned long long* __restrict__ hist) {
    __shared__ unsigned int h[256];
    for (int b = threadIdx.x; b < 256; b += blockDim.x) h[b] = 0;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t u = ordkey(keys[i]);
        if ((u & pmask) == pval) atomicAdd(&h[(u >> shift) & 0xFF], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < 256; b += blockDim.x)
        if (h[b]) atomicAdd(&hist[b], (unsigned long long)h[b]);
}

void launch_hist8(const double* keys, int64_t n, int shift, uint64_t prefix_mask, uint64_t prefix_val,
                  unsigned long long* hist, int num_sms, cudaStream_t s, LaunchStats& ls) {
    cudaMemsetAsync(hist, 0, 256 * sizeof(unsigned long long), s);
    if (n > 0) {
        k_hist8<<<num_sms * 4, kBlock, 0, s>>>(keys, n, shift, prefix_mask, prefix_val, hist);
        ++ls.launches;
    }
}

// ============================================================== compaction
constexpr int kChunkC = 4096;
static_assert(kChunkC == 16 * kBlock, "compaction: 16 flags per thread");

// Flags are 0 / 1 bytes; a thread takes 16 consecutive ones (one 16-byte load when the chunk is
// whole and the buffer 16-byte aligned) and counts them with popc; the per-chunk and per-block
// scans are warp-shuffle scans (integer, so any order is exact).
__device__ __forceinline__ int flags16(const uint8_t* __restrict__ flags, int64_t i0, int64_t n, bool vec,
                                       uint32_t (&w)[4]) {
    if (vec && i0 + 16 <= n) {
        const uint4 v = *reinterpret_cast<const uint4*>(flags + i0);
        w[0] = v.x, w[1] = v.y, w[2] = v.z, w[3] = v.w;
    } else {
        for (int q = 0; q < 4; ++q) {
            uint32_t x = 0;
            for (int b = 0; b < 4; ++b) {
                const int64_t i = i0 + 4 * q + b;
                if (i < n && flags[i]) x |= 1u << (8 * b);
            }
            w[q] = x;
        }
    }
    return __popc(w[0] & 0x01010101u) + __popc(w[1] & 0x01010101u) + __popc(w[2] & 0x01010101u) +
           __popc(w[3] & 0x01010101u);
}

// exclusive block scan of one int per thread (blockDim.x = kBlock); returns the block total in *tot
__device__ __forceinline__ int block_excl_scan(int v, int* wsum, int* tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int s = lane < nw ? wsum[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, s, d);
            if (lane >= d) s += y;
        }
        if (lane < nw) wsum[lane] = s;  // inclusive warp prefix
    }
    __syncthreads();
    const int before = (warp > 0 ? wsum[warp - 1] : 0) + x - v;
    *tot = wsum[nw - 1];
    return before;
}

__global__ void k_flag_count(const uint8_t* __restrict__ flags, int64_t n, int64_t* __restrict__ cnt) {
    __shared__ int wsum[32];
    const bool vec = ((uintptr_t)flags & 15) == 0;
    uint32_t w[4];
    const int c = flags16(flags, (int64_t)blockIdx.x * kChunkC + threadIdx.x * 16, n, vec, w);
    int tot;
    block_excl_scan(c, wsum, &tot);
    if (threadIdx.x == 0) cnt[blockIdx.x] = tot;
}

__global__ void k_scan_counts(int64_t* cnt, int64_t nc, int64_t* total) {
    // single block: each thread a contiguous segment, block-wide shuffle scan of the segment sums
    __shared__ long long wsum[32];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = blockDim.x >> 5;
    const int64_t per = (nc + blockDim.x - 1) / blockDim.x;
    const int64_t b = t * per, e = min(nc, b + per);
    long long s = 0;
    for (int64_t i = b; i < e; ++i) s += cnt[i];
    long long x = s;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
        long long v = lane < nw ? wsum[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, v, d);
            if (lane >= d) v += y;
        }
        if (lane < nw) wsum[lane] = v;
    }
    __syncthreads();
    long long a = (warp > 0 ? wsum[warp - 1] : 0) + x - s;
    if (t == blockDim.x - 1) *total = a + s;
    for (int64_t i = b; i < e; ++i) {
        const int64_t v = cnt[i];
        cnt[i] = a;
        a += v;
    }
}

__global__ void k_write_indices(const uint8_t* __restrict__ flags, int64_t n, const int64_t* __restrict__ offs,
                                int64_t base, int64_t* __restrict__ out) {
    __shared__ int wsum[32];
    const bool vec = ((uintptr_t)flags & 15) == 0;
    const int64_t c0 = (int64_t)blockIdx.x * kChunkC + threadIdx.x * 16;
    uint32_t w[4];
    const int c = flags16(flags, c0, n, vec, w);
    int tot;
    const int before = block_excl_scan(c, wsum, &tot);
    if (!c) return;
    int64_t o = offs[blockIdx.x] + before;
#pragma unroll
    for (int q = 0; q < 4; ++q)
        for (uint32_t x = w[q] & 0x01010101u; x; x &= x - 1) out[o++] = base + c0 + 4 * q + (__ffs(x) - 1) / 8;
}

void launch_compact(const uint8_t* flags, int64_t n, int64_t index_base, int64_t* counts_scratch, int64_t* out_idx,
                    int64_t* out_count, cudaStream_t s, LaunchStats& ls) {
    const int64_t nc = (n + kChunkC - 1) / kChunkC;
    if (nc == 0) {
        cudaMemsetAsync(out_count, 0, sizeof(int64_t), s);
        return;
    }
    k_flag_count<<<(unsigned)nc, kBlock, 0, s>>>(flags, n, counts_scratch);
    k_scan_counts<<<1, 1024, 0, s>>>(counts_scratch, nc, out_count);
    if (out_idx) k_write_indices<<<(unsigned)nc, kBlock, 0, s>>>(flags, n, counts_scratch, index_base, out_idx);
    ls.launches += out_idx ? 3 : 2;
}

// ================================================================ k-means++
__global__ void k_kpp_update(const double* __restrict__ X, int64_t n, int64_t ld, int D,
                             const double* __restrict__ c, double* __restrict__ d2, double* __restrict__ parts,
                             int first) {
    __shared__ double red[kBlock];
    constexpr int PER = kChunkC / kBlock;
    const int64_t c0 = (int64_t)blockIdx.x * kChunkC;
    double s = 0.0;
    // thread t covers rows c0 + t + j*kBlock (coalesced); the per-chunk sum is
    // a fixed-order tree, so it is deterministic.
    for (int j = 0; j < PER; ++j) {
        const int64_t i = c0 + threadIdx.x + (int64_t)j * kBlock;
        if (i >= n) break;
        double t = 0.0;
        for (int a = 0; a < D; ++a) {
            const double e = X[(int64_t)a * ld + i] - c[a];
            t = fma(e, e, t);
        }
        const double v = first ? t : fmin(d2[i], t);
        d2[i] = v;
        s += v;
    }
    const double b = block_sum(s, red);
    if (threadIdx.x == 0) parts[blockIdx.x] = b;
}

void launch_kpp_update(const double* X, int64_t n, int64_t ld, int D, const double* center, double* d2,
                       double* parts, bool first, cudaStream_t s, LaunchStats& ls) {
    const int64_t nc = (n + kChunkC - 1) / kChunkC;
    if (nc == 0) return;
    k_kpp_update<<<(unsigned)nc, kBlock, 0, s>>>(X, n, ld, D, center, d2, parts, first ? 1 : 0);
    ++ls.launches;
}


// ------------------------------------------------------------------ k-means baseline
// (eval-bench kmeans_baseline).  Rows in fixed order: CTA b, warp w,
// lane l take row (b + gridDim.x * it) * (32 * nwarps) + 32 w + l.  Nearest centroid by
// squared Euclidean distance as an FMA chain over the features in order (the oracle
// uses the same chain), ties -> lowest k.  Mode 0 (Lloyd step): per centroid the sum of
// its rows and their count, and the number of changed assignments, reduced per warp with
// xor shuffles and per CTA in warp order -> partial[blk][K (D + 1) + 1]; mode 1: the
// distance to the nearest centroid of every row.
__device__ __forceinline__ double warp_allsum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int DM>
__global__ void __launch_bounds__(kBlock) k_lloyd(const double* __restrict__ X, int64_t n, int64_t ld, int D, int K,
                                                  const double* __restrict__ cen, int32_t* __restrict__ assign,
                                                  double* __restrict__ partial, double* __restrict__ score, int mode) {
    extern __shared__ double sm[];
    const int L = K * (D + 1) + 1, nw = kBlock / 32;
    double* sc = sm;           // centroids [K][D]
    double* acc = sm + K * D;  // [nw][L]
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    for (int e = t; e < K * D; e += kBlock) sc[e] = cen[e];
    if (mode == 0)
        for (int e = t; e < nw * L; e += kBlock) acc[e] = 0.0;
    __syncthreads();
    double* wa = acc + warp * L;
    const int64_t step = (int64_t)gridDim.x * kBlock;
    for (int64_t base = (int64_t)blockIdx.x * kBlock; base < n; base += step) {
        const int64_t i = base + warp * 32 + lane;
        const bool valid = i < n;
        double x[DM];
#pragma unroll
        for (int a = 0; a < DM; ++a) x[a] = (valid && a < D) ? X[(int64_t)a * ld + i] : 0.0;
        double best = INFINITY;
        int bk = 0;
        for (int k = 0; k < K; ++k) {
            double d2 = 0.0;
#pragma unroll
            for (int a = 0; a < DM; ++a) {
                if (a < D) {
                    const double e = x[a] - sc[k * D + a];
                    d2 = fma(e, e, d2);
                }
            }
            if (d2 < best) {
                best = d2;
                bk = k;
            }
        }
        if (mode == 1) {
            if (valid) score[i] = sqrt(best);
            continue;
        }
        const bool ch = valid && assign[i] != bk;
        if (valid) assign[i] = bk;
        const unsigned chb = __ballot_sync(0xffffffffu, ch);
        for (int k = 0; k < K; ++k) {
            const bool m = valid && bk == k;
            const unsigned mb = __ballot_sync(0xffffffffu, m);
            if (!mb) continue;
#pragma unroll
            for (int a = 0; a < DM; ++a) {
                if (a < D) {
                    const double v = warp_allsum(m ? x[a] : 0.0);
                    if (lane == 0) wa[k * (D + 1) + a] += v;
                }
            }
            if (lane == 0) wa[k * (D + 1) + D] += (double)__popc(mb);
        }
        if (lane == 0) wa[L - 1] += (double)__popc(chb);
    }
    if (mode == 0) {
        __syncthreads();
        for (int e = t; e < L; e += kBlock) {
            double v = 0.0;
            for (int w = 0; w < nw; ++w) v += acc[w * L + e];
            partial[(int64_t)blockIdx.x * L + e] = v;
        }
    }
}

template <int DM>
static void lloyd_dm(const double* X, int64_t n, int64_t ld, int D, int K, const double* cen, int32_t* assign,
                     double* partial, double* score, int mode, int grid, cudaStream_t s) {
    const size_t smem = (size_t)(K * D + (kBlock / 32) * (K * (D + 1) + 1)) * sizeof(double);
    static size_t set = 0;
    if (smem > 48 * 1024 && smem > set) {
        cudaFuncSetAttribute(k_lloyd<DM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        set = smem;
    }
    k_lloyd<DM><<<grid, kBlock, smem, s>>>(X, n, ld, D, K, cen, assign, partial, score, mode);
}

int lloyd_grid(int64_t n, int num_sms) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(num_sms, (n + kBlock - 1) / kBlock));
}

void launch_lloyd(const double* X, int64_t n, int64_t ld, int D, int K, const double* cen, int32_t* assign,
                  double* partial, double* score, int mode, int grid, cudaStream_t s, LaunchStats& ls) {
    if (n <= 0) return;
    if (D <= 8)
        lloyd_dm<8>(X, n, ld, D, K, cen, assign, partial, score, mode, grid, s);
    else if (D <= 16)
        lloyd_dm<16>(X, n, ld, D, K, cen, assign, partial, score, mode, grid, s);
    else if (D <= 32)
        lloyd_dm<32>(X, n, ld, D, K, cen, assign, partial, score, mode, grid, s);
    else
        lloyd_dm<64>(X, n, ld, D, K, cen, assign, partial, score, mode, grid, s);
    ++ls.launches;
}

// flag_i = score_i > threshold; per-CTA flag counts
__global__ void k_flag_gt(const double* __restrict__ score, int64_t n, double thr, uint8_t* __restrict__ flags,
                          unsigned long long* __restrict__ count) {
    __shared__ unsigned long long c;
    if (threadIdx.x == 0) c = 0;
    __syncthreads();
    unsigned long long mine = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t f = score[i] > thr ? 1 : 0;
        flags[i] = f;
        mine += f;
    }
    atomicAdd(&c, mine);
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(count, c);
}

void launch_flag_gt(const double* score, int64_t n, double thr, uint8_t* flags, unsigned long long* count,
                    int num_sms, cudaStream_t s, LaunchStats& ls) {
    cudaMemsetAsync(count, 0, sizeof(unsigned long long), s);
    if (n <= 0) return;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(4 * num_sms, (n + kBlock - 1) / kBlock));
    k_flag_gt<<<grid, kBlock, 0, s>>>(score, n, thr, flags, count);
    ++ls.launches;
}

// confusion counts (anomaly = positive): out[0..3] = tp, fp, tn, fn
__global__ void k_confusion(const uint8_t* __restrict__ labels, const uint8_t* __restrict__ flags, int64_t n,
                            unsigned long long* __restrict__ out) {
    __shared__ unsigned long long c[4];
    if (threadIdx.x < 4) c[threadIdx.x] = 0;
    __syncthreads();
    unsigned long long m[4] = {0, 0, 0, 0};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int l = labels[i] != 0, f = flags[i] != 0;
        m[l ? (f ? 0 : 3) : (f ? 1 : 2)] += 1;
    }
    for (int j = 0; j < 4; ++j) atomicAdd(&c[j], m[j]);
    __syncthreads();
    if (threadIdx.x < 4) atomicAdd(&out[threadIdx.x], c[threadIdx.x]);
}

void launch_confusion(const uint8_t* labels, const uint8_t* flags, int64_t n, unsigned long long* out, int num_sms,
                      cudaStream_t s, LaunchStats& ls) {
    cudaMemsetAsync(out, 0, 4 * sizeof(unsigned long long), s);
    if (n <= 0) return;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(4 * num_sms, (n + kBlock - 1) / kBlock));
    k_confusion<<<grid, kBlock, 0, s>>>(labels, flags, n, out);
    ++ls.launches;
}


// ------------------------------------------------------------------ event features
// (event-model extract_features, with validate_event's invariants,
// SPEC.md:32-38,52-60).  Pass 1: keep_i = (layer_i == L); the first row violating an
// invariant (min row index, then its field code) via atomicMin on (row << 8 | field).
// Pass 2 (over the order-preserving compacted indices): the layer's default features,
// Cuda/Python/Torch: log10(duration_ns + 1); Nccl: log10(duration_ns + 1),
// log10(message_bytes + 1); GpuSample: util_pct, mem_used_mb, temp_c.
__global__ void k_event_keep(const uint8_t* __restrict__ layer, const int64_t* __restrict__ ts,
                             const int64_t* __restrict__ dur, const double* __restrict__ mb,
                             const double* __restrict__ util, const double* __restrict__ mem,
                             const double* __restrict__ temp, int64_t n, int L, uint8_t* __restrict__ keep,
                             unsigned long long* __restrict__ bad) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int l = layer[i];
        int f = 0;
        // field code (1 layer, 2 ts_start, 3 duration_ns, 4 message_bytes, 5 util_pct,
        // 6 mem_used_mb, 7 temp_c) | 0x10 when the attribute is absent (NULL column / NaN)
        auto miss = [&](const double* col) { return !col || isnan(col[i]); };
        if (l > 4) f = 1;
        else if (!(ts[i] > 0)) f = 2;
        else if (!(dur[i] >= 0)) f = 3;
        else if (l == 3 && miss(mb)) f = 0x14;
        else if (l == 3 && !(mb[i] >= 0.0)) f = 4;
        else if (l == 4 && miss(util)) f = 0x15;
        else if (l == 4 && !(util[i] >= 0.0 && util[i] <= 100.0)) f = 5;
        else if (l == 4 && miss(mem)) f = 0x16;
        else if (l == 4 && !(mem[i] >= 0.0)) f = 6;
        else if (l == 4 && miss(temp)) f = 0x17;
        else if (l == 4 && !(temp[i] > -50.0 && temp[i] < 150.0)) f = 7;
        if (f) atomicMin(bad, ((unsigned long long)i << 8) | (unsigned long long)f);
        keep[i] = (l == L) ? 1 : 0;
    }
}

__global__ void k_event_features(const int64_t* __restrict__ idx, int64_t m, const int64_t* __restrict__ dur,
                                 const double* __restrict__ mb, const double* __restrict__ util,
                                 const double* __restrict__ mem, const double* __restrict__ temp, int L,
                                 double* __restrict__ X, int64_t ld) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = idx[r];
        if (L == 4) {
            X[r] = util[i];
            X[ld + r] = mem[i];
            X[2 * ld + r] = temp[i];
        } else {
            X[r] = log10((double)dur[i] + 1.0);
            if (L == 3) X[ld + r] = log10(mb[i] + 1.0);
        }
    }
}

void launch_event_keep(const uint8_t* layer, const int64_t* ts, const int64_t* dur, const double* mb,
                       const double* util, const double* mem, const double* temp, int64_t n, int L, uint8_t* keep,
                       unsigned long long* bad, int num_sms, cudaStream_t s, LaunchStats& ls) {
    cudaMemsetAsync(bad, 0xFF, sizeof(unsigned long long), s);
    if (n <= 0) return;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(8 * num_sms, (n + kBlock - 1) / kBlock));
    k_event_keep<<<grid, kBlock, 0, s>>>(layer, ts, dur, mb, util, mem, temp, n, L, keep, bad);
    ++ls.launches;
}

void launch_event_features(const int64_t* idx, int64_t m, const int64_t* dur, const double* mb, const double* util,
                           const double* mem, const double* temp, int L, double* X, int64_t ld, int num_sms,
                           cudaStream_t s, LaunchStats& ls) {
    if (m <= 0) return;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(8 * num_sms, (m + kBlock - 1) / kBlock));
    k_event_features<<<grid, kBlock, 0, s>>>(idx, m, dur, mb, util, mem, temp, L, X, ld);
    ++ls.launches;
}

}  // namespace es
