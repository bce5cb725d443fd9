// es_fast.cu — mixed-precision fast path of the EM pass and the scoring pass.
//
// The FP64 team kernels (es_kernels.cu) are the strict path.  On B200 FP64
// SIMT caps a full-covariance E+M pass at ~13% of the HBM roofline (DESIGN.md
// "Roofline"), so the production path computes the whitening in FP32 and
// keeps every accumulation that the parity contract names in FP64:
//
//   k_em_fast<DM>   thread-per-event E-step: x' = x - c (FP64 subtract, then
//                   FP32), z = W_k (x' - mu'_k) with 16 independent FP32 row
//                   chains, in-thread log-sum-exp, logL accumulated in FP64.
//                   Responsibilities >= 1e-20 are compacted (deterministic
//                   ballot order) into per-component lists; warp k then
//                   accumulates component k's sufficient statistics about
//                   c_k = mu_k(old) from its list in FP32 registers, flushed
//                   every 32 batches into FP64 shared accumulators.
//                   Pruning is certified: a skipped pair has gamma < 1e-20, so
//                   all skipped pairs move N_k by < N*1e-20 (< 1e-12 at 2^26
//                   events) — far inside the 1e-5 parameter tolerance, and any
//                   component that small has N_k < 1 and is reseeded anyway
//                   (SPEC.md:294).
//   k_score_fast<DM> FP32 E-step for all components, then the components that
//                   can matter at 1e-6 (within 20 nats of the best, or within
//                   rounding of the best-component / posterior argmax) are
//                   recomputed in FP64 by per-lane "refine slots", so ll,
//                   best_logdens, best_k, predict and flags carry FP64
//                   accuracy; the rest enter ll only through exp(w - m) < 2e-9.
#include <cfloat>
#include <cmath>
#include <cstdlib>

#include "es_kernels.h"
#include "es_tc.cuh"

namespace es {

namespace {

template <class F>
void allow_smem(F* f, size_t bytes) {
    cudaFuncSetAttribute(reinterpret_cast<const void*>(f), cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)bytes);
}

__device__ double block_sum_d(double v, double* red) {
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

constexpr int kT = 256;     // events per tile (thread per event)
constexpr int kKmax = 8;    // components handled by the fast path
constexpr float kGammaMin = 1e-20f;

template <int DM>
struct FastCfg {
    static constexpr int XS = kT + 4;                    // FP32 x' plane stride
    static constexpr int NS = 1 + DM + DM * (DM + 1) / 2;  // statistics per component
    static constexpr int W64S = DM * DM + 2;             // FP64 W stride (bank skew)
};

// FP32 whitening against component k: q = ||W_k (x' - mu'_k)||^2 with all DM
// rows as independent FMA chains.
template <int DM>
__device__ __forceinline__ float whiten32(const float* __restrict__ Wk, const float* __restrict__ mk,
                                          const float (&xp)[DM]) {
    float d[DM];
#pragma unroll
    for (int j = 0; j < DM; j += 4) {
        const float4 m = *reinterpret_cast<const float4*>(mk + j);
        d[j] = xp[j] - m.x;
        d[j + 1] = xp[j + 1] - m.y;
        d[j + 2] = xp[j + 2] - m.z;
        d[j + 3] = xp[j + 3] - m.w;
    }
    float q = 0.f;
#pragma unroll
    for (int r = 0; r < DM; ++r) {
        const float* Wr = Wk + r * DM;
        float a = 0.f;
#pragma unroll
        for (int j = 0; j <= r; j += 4) {
            const float4 w = *reinterpret_cast<const float4*>(Wr + j);
            a = fmaf(w.x, d[j], a);
            if (j + 1 <= r) a = fmaf(w.y, d[j + 1], a);
            if (j + 2 <= r) a = fmaf(w.z, d[j + 2], a);
            if (j + 3 <= r) a = fmaf(w.w, d[j + 3], a);
        }
        q = fmaf(a, a, q);
    }
    return q;
}

// Stage FP32 W (rows padded to DM), mu' = mu - c and constants into smem.
template <int DM>
__device__ void stage32(const ModelView& mv, const double* __restrict__ c, float* sW, float* sMu, float* sCst) {
    const int K = mv.K, D = mv.D;
    for (int e = threadIdx.x; e < kKmax * DM * DM; e += blockDim.x) {
        const int k = e / (DM * DM), rc = e % (DM * DM), r = rc / DM, cc = rc % DM;
        sW[e] = (k < K && r < D && cc < D) ? (float)mv.W()[(int64_t)k * D * D + r * D + cc] : 0.f;
    }
    for (int e = threadIdx.x; e < kKmax * DM; e += blockDim.x) {
        const int k = e / DM, j = e % DM;
        sMu[e] = (k < K && j < D) ? (float)(mv.mu()[k * D + j] - c[j]) : 0.f;
    }
    for (int k = threadIdx.x; k < kKmax; k += blockDim.x)
        sCst[k] = k < K ? (float)(mv.logpi()[k] + mv.lognorm()[k]) : -INFINITY;
}

}  // namespace

// ======================================================== fused E + M pass
template <int DM>
__global__ void __launch_bounds__(kT, 1) k_em_fast(const double* __restrict__ X, int64_t n, int64_t ld, int D, int K,
                                                    const double* __restrict__ model,
                                                    const double* __restrict__ center,
                                                    double* __restrict__ partial) {
    using C = FastCfg<DM>;
    extern __shared__ __align__(16) unsigned char smraw[];
    float* sW = reinterpret_cast<float*>(smraw);           // 8*DM*DM
    float* sMu = sW + kKmax * DM * DM;                     // 8*DM
    float* sCst = sMu + kKmax * DM;                        // 8
    float* sX = sCst + kKmax;                              // DM*XS
    float* lstG = sX + DM * C::XS;                         // 8*T
    uint16_t* lstT = reinterpret_cast<uint16_t*>(lstG + kKmax * kT);  // 8*T
    int* cnt = reinterpret_cast<int*>(lstT + kKmax * kT);  // 8 warps x 8 comps
    int* off = cnt + 64;                                   // 8 x 8
    int* tot = off + 64;                                   // 8
    double* sAcc = reinterpret_cast<double*>(tot + 8);     // 8*NS (8-byte aligned: offsets above are even)
    double* sRed = sAcc + kKmax * C::NS;                   // T
    double* sC = sRed + kT;                                // DM (center)

    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    ModelView mv{K, D, const_cast<double*>(model)};
    stage32<DM>(mv, center, sW, sMu, sCst);
    for (int e = t; e < kKmax * C::NS; e += kT) sAcc[e] = 0.0;
    for (int j = t; j < DM; j += kT) sC[j] = j < D ? center[j] : 0.0;
    __syncthreads();

    const int kw = warp;           // component owned by this warp in the M-phase
    const bool mact = kw < K;
    float acc[C::NS];
#pragma unroll
    for (int j = 0; j < C::NS; ++j) acc[j] = 0.f;
    int since_flush = 0;
    double ll_acc = 0.0;
    const unsigned lt_mask = (1u << lane) - 1u;

    auto flush = [&]() {
        if (!mact) return;
#pragma unroll
        for (int j = 0; j < C::NS; ++j) {
            float v = acc[j];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if ((j & 31) == lane) sAcc[kw * C::NS + j] += (double)v;
            acc[j] = 0.f;
        }
    };

    for (int64_t tile = blockIdx.x;; tile += gridDim.x) {
        const int64_t t0 = tile * kT;
        if (t0 >= n) break;
        const int64_t i = t0 + t;
        const bool valid = i < n;
        // ---------------- E-phase: thread per event
        float xp[DM];
#pragma unroll
        for (int j = 0; j < DM; ++j) {
            xp[j] = (valid && j < D) ? (float)(__ldg(X + (int64_t)j * ld + i) - sC[j]) : 0.f;
            sX[j * C::XS + t] = xp[j];
        }
        float w[kKmax];
        float m = -INFINITY;
#pragma unroll
        for (int k = 0; k < kKmax; ++k) {
            w[k] = -INFINITY;
            if (k < K) {
                const float q = whiten32<DM>(sW + k * DM * DM, sMu + k * DM, xp);
                w[k] = sCst[k] - 0.5f * q;
                m = fmaxf(m, w[k]);
            }
        }
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < kKmax; ++k) s += __expf(w[k] - m);
        const float ll = m + __logf(s);
        if (valid) ll_acc += (double)ll;
        // ---------------- deterministic compaction of significant (event, k)
        float g[kKmax];
        unsigned rank[kKmax];
#pragma unroll
        for (int k = 0; k < kKmax; ++k) {
            g[k] = __expf(w[k] - ll);
            const bool sig = valid && k < K && g[k] >= kGammaMin;
            const unsigned b = __ballot_sync(0xffffffffu, sig);
            rank[k] = sig ? __popc(b & lt_mask) : 0xffffffffu;
            if (lane == 0) cnt[warp * 8 + k] = __popc(b);
        }
        __syncthreads();
        if (t < kKmax) {
            int a = 0;
            for (int wv = 0; wv < 8; ++wv) {
                off[wv * 8 + t] = a;
                a += cnt[wv * 8 + t];
            }
            tot[t] = a;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kKmax; ++k)
            if (rank[k] != 0xffffffffu) {
                const int p = off[warp * 8 + k] + (int)rank[k];
                lstT[k * kT + p] = (uint16_t)t;
                lstG[k * kT + p] = g[k];
            }
        __syncthreads();
        // ---------------- M-phase: warp kw accumulates component kw
        if (mact) {
            const int nk = tot[kw];
            const float* muk = sMu + kw * DM;
            for (int e0 = 0; e0 < nk; e0 += 32) {
                const int e = e0 + lane;
                const bool ve = e < nk;
                const int tt = ve ? lstT[kw * kT + e] : 0;
                const float gg = ve ? lstG[kw * kT + e] : 0.f;
                float d[DM];
#pragma unroll
                for (int a = 0; a < DM; ++a) d[a] = sX[a * C::XS + tt] - muk[a];
                acc[0] += gg;
                int p = 1 + DM;
#pragma unroll
                for (int a = 0; a < DM; ++a) {
                    const float ga = gg * d[a];
                    acc[1 + a] += ga;
#pragma unroll
                    for (int b = a; b < DM; ++b) {
                        acc[p] = fmaf(ga, d[b], acc[p]);
                        ++p;
                    }
                }
                if (++since_flush == 32) {
                    flush();
                    since_flush = 0;
                }
            }
        }
        __syncthreads();
    }
    flush();
    const double bl = block_sum_d(ll_acc, sRed);  // syncs: sAcc complete
    // ---------------- partial block in the canonical raw layout (about mu_k)
    const int SK = stat_k(D), NE = K * SK;
    double* myp = partial + (int64_t)blockIdx.x * (NE + 1);
    for (int e = t; e < NE; e += kT) {
        const int k = e / SK, r = e % SK;
        int j;
        if (r <= D) {
            j = r;
        } else {
            int p = r - 1 - D, a = 0;
            while (p >= D - a) {
                p -= D - a;
                ++a;
            }
            const int b = a + p;
            j = 1 + DM + (a * DM - (a * (a - 1)) / 2 + (b - a));
        }
        myp[e] = sAcc[k * C::NS + j];
    }
    if (t == 0) myp[NE] = bl;
}

template <int DM>
static size_t em_fast_smem() {
    using C = FastCfg<DM>;
    size_t b = (size_t)(kKmax * DM * DM + kKmax * DM + kKmax + DM * C::XS + kKmax * kT) * 4;  // floats
    b += (size_t)kKmax * kT * 2;                                                          // u16 list
    b += (64 + 64 + 8) * 4;                                                               // ints
    b = (b + 15) / 16 * 16;
    b += (size_t)(kKmax * C::NS + kT + DM) * 8;
    return b;
}

bool em_fast_supported(int D, int K) { return D <= 16 && K <= kKmax; }

void launch_em_fast(const double* X, int64_t n, int64_t ld, int D, int K, const double* model, const double* center,
                    double* partial, int num_sms, int* nblk, cudaStream_t s, LaunchStats& ls) {
    *nblk = num_sms;
    if (D <= 8) {
        static bool a = false;
        if (!a) { allow_smem(k_em_fast<8>, em_fast_smem<8>()); a = true; }
        k_em_fast<8><<<num_sms, kT, em_fast_smem<8>(), s>>>(X, n, ld, D, K, model, center, partial);
    } else {
        static bool a = false;
        if (!a) { allow_smem(k_em_fast<16>, em_fast_smem<16>()); a = true; }
        k_em_fast<16><<<num_sms, kT, em_fast_smem<16>(), s>>>(X, n, ld, D, K, model, center, partial);
    }
    ++ls.launches;
}

// ============================================ tcgen05 E-step (3xTF32 UMMA)
// Whitening of a 256-event tile as two M=128 x N=128 x K=24 tcgen05 GEMMs:
//   U[i, (k,r)] = sum_j A[i, j] B[(k,r), j],  A = [x'_i | 1 | 0...],
//   B = [W_k[r, :] | -(W_k mu'_k)_r | 0...]  =>  U[i,(k,r)] = (W_k (x'_i - mu'_k))_r.
// Operands are split hi/lo in TF32 (D = AhBh + AhBl + AlBh, FP32 accumulate in
// TMEM): FP32-level whitening on the tensor cores.  SMEM operands use the
// canonical K-major SWIZZLE_NONE layout (8-row x 16-byte core matrices,
// LBO = 128 B between K chunks, SBO = 768 B between 8-row groups).
using namespace tc;

// Gram accumulator layout for DM = 16 in FP32 pairs: row a covers b >= a as
// (odd a: one single (a,a)) + pairs (2m, 2m+1) for 2m >= a.
struct GramPairs {
    static constexpr int NP = 64;   // pairs
    static constexpr int NSG = 8;   // singles (odd diagonal entries)
};

constexpr int kXR = 20;  // row-major FP32 x' stride (16 + 4 pad floats = 80 B)

// Software pipeline per CTA (one tile = 256 events = 2 UMMA M-tiles):
//   [wait MMA(j)] [epilogue(j): TMEM -> w, LSE, gamma lists] [A-prep(j+1) from
//   the bulk-prefetched X tile] [issue MMA(j+1), prefetch X(j+2)] [M-phase(j)]
// so the tensor cores and the copy engine work under the FP32 M-phase.
__global__ void __launch_bounds__(kT, 1) k_em_tc(const double* __restrict__ X, int64_t n, int64_t ld, int D, int K,
                                                  const double* __restrict__ model,
                                                  const double* __restrict__ center, double* __restrict__ partial) {
    constexpr int DM = 16;
    using C = FastCfg<DM>;
    extern __shared__ __align__(1024) unsigned char smraw[];
    unsigned char* sAh = smraw;                         // 2 sub-tiles x 12 KB
    unsigned char* sAl = sAh + 2 * kOpBytes;            // 2 x 12 KB
    unsigned char* sBh = sAl + 2 * kOpBytes;            // 12 KB
    unsigned char* sBl = sBh + kOpBytes;                // 12 KB
    double* sXd = reinterpret_cast<double*>(sBl + kOpBytes);   // 2 x DM x T FP64 (bulk-prefetched tiles)
    float* sXr = reinterpret_cast<float*>(sXd + 2 * DM * kT);  // 2 x T x kXR FP32 rows (x' - for the M-phase)
    float* sNMu = sXr + 2 * kT * kXR;                   // 8 x DM: -mu'
    float* sCst = sNMu + kKmax * DM;                    // 8
    float* sThr = sCst + kKmax;                         // 8 pruning thresholds
    float* lstG = sThr + kKmax;                         // 8*T
    float* sG = lstG + kKmax * kT;                      // 8*T responsibilities of the tile
    uint16_t* lstT = reinterpret_cast<uint16_t*>(sG + kKmax * kT);
    unsigned* bal = reinterpret_cast<unsigned*>(lstT + kKmax * kT);  // 8 warps x 8 comps ballots
    int* off = reinterpret_cast<int*>(bal + 64);
    int* tot = off + 64;
    double* sAcc = reinterpret_cast<double*>(tot + 8);
    double* sRed = sAcc + kKmax * C::NS;
    double* sC = sRed + kT;
    __shared__ uint64_t mbar_mma, mbar_x[2];
    __shared__ uint32_t tmem_slot;

    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    ModelView mv{K, D, const_cast<double*>(model)};
    for (int j = t; j < DM; j += kT) sC[j] = j < D ? center[j] : 0.0;
    __syncthreads();
    for (int e = t; e < kTileRows * kKA; e += kT) {
        const int row = e / kKA, kk = e % kKA, k = row / DM, r = row % DM;
        double v = 0.0;
        if (k < K && r < D) {
            const double* Wr = mv.W() + (int64_t)k * D * D + (int64_t)r * D;
            if (kk < D) {
                v = Wr[kk];
            } else if (kk == DM) {
                double b = 0.0;
                for (int j = 0; j <= r; ++j) b = fma(Wr[j], mv.mu()[k * D + j] - sC[j], b);
                v = -b;
            }
        }
        const uint32_t h = tf32((float)v);
        const uint32_t l = tf32((float)(v - (double)__uint_as_float(h)));
        *reinterpret_cast<uint32_t*>(sBh + op_off(row, kk)) = h;
        *reinterpret_cast<uint32_t*>(sBl + op_off(row, kk)) = l;
    }
    for (int e = t; e < kKmax * DM; e += kT) {
        const int k = e / DM, j = e % DM;
        sNMu[e] = (k < K && j < D) ? -(float)(mv.mu()[k * D + j] - sC[j]) : 0.f;
    }
    for (int k = t; k < kKmax; k += kT) {
        sCst[k] = k < K ? (float)(mv.logpi()[k] + mv.lognorm()[k]) : -INFINITY;
        // certified pruning: skipped responsibility mass <= N * 1e-9 * pi_k = 1e-9 N_k
        sThr[k] = k < K ? fmaxf((float)(1e-9 * mv.pi()[k]), 1e-30f) : INFINITY;
    }
    for (int e = t; e < kKmax * C::NS; e += kT) sAcc[e] = 0.0;
    for (int e = t; e < 2 * kTileRows * (kKA - DM); e += kT) {
        const int s2 = e / (kTileRows * (kKA - DM)), rr = e % (kTileRows * (kKA - DM));
        const int row = rr / (kKA - DM), kk = DM + rr % (kKA - DM);
        *reinterpret_cast<uint32_t*>(sAh + s2 * kOpBytes + op_off(row, kk)) = kk == DM ? 0x3F800000u : 0u;
        *reinterpret_cast<uint32_t*>(sAl + s2 * kOpBytes + op_off(row, kk)) = 0u;
    }
    for (int e = t; e < 2 * DM * kT; e += kT) sXd[e] = 0.0;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar_mma)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar_x[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar_x[1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;
    const uint32_t bar = su32(&mbar_mma);
    uint32_t phase = 0, xphase[2] = {0, 0};
    const uint64_t dBh = umma_desc(su32(sBh)), dBl = umma_desc(su32(sBl));
    const int64_t ntiles = (n + kT - 1) / kT;
    auto prefetch = [&](int64_t tile, int buf) {
        if (tile >= ntiles || (tile + 1) * kT > n) return;
        const uint32_t b = su32(&mbar_x[buf]);
        mbar_expect_tx(b, (uint32_t)(D * kT * 8));
        for (int j = 0; j < D; ++j)
            bulk_g2s(su32(sXd + (buf * DM + j) * kT), X + (int64_t)j * ld + tile * kT, kT * 8, b);
    };
    const int sub = t >> 7, row = t & 127;
    // A-prep of `tile` from X buffer xb into the A operands and FP32 rows buffer xb
    auto aprep = [&](int64_t tile, int xb) {
        const int64_t i = tile * kT + t;
        const bool valid = i < n;
        const bool full = (tile + 1) * kT <= n;
        if (full) {
            mbar_wait(su32(&mbar_x[xb]), xphase[xb]);
            xphase[xb] ^= 1;
        }
        unsigned char* ah = sAh + sub * kOpBytes;
        unsigned char* al = sAl + sub * kOpBytes;
        const double* xs = sXd + xb * DM * kT;
        float* xr = sXr + (xb * kT + t) * kXR;
#pragma unroll
        for (int j = 0; j < DM; j += 4) {
            float f[4];
            uint32_t h[4], l[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                double xv;
                if (full) xv = xs[(j + q) * kT + t];
                else xv = (valid && j + q < D) ? __ldg(X + (int64_t)(j + q) * ld + i) : 0.0;
                f[q] = (valid && j + q < D) ? (float)(xv - sC[j + q]) : 0.f;
                h[q] = tf32(f[q]);
                l[q] = tf32(f[q] - __uint_as_float(h[q]));
            }
            *reinterpret_cast<float4*>(xr + j) = make_float4(f[0], f[1], f[2], f[3]);
            *reinterpret_cast<uint4*>(ah + op_off(row, j)) = make_uint4(h[0], h[1], h[2], h[3]);
            *reinterpret_cast<uint4*>(al + op_off(row, j)) = make_uint4(l[0], l[1], l[2], l[3]);
        }
        proxy_fence();
    };
    auto issue_mma = [&]() {
        tc_fence_after();
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
            const uint32_t d = tmem + 128 * s2;
            const uint64_t dAh = umma_desc(su32(sAh + s2 * kOpBytes)), dAl = umma_desc(su32(sAl + s2 * kOpBytes));
#pragma unroll
            for (int ks = 0; ks < kKA / 8; ++ks) {
                const uint64_t ko = (uint64_t)((2 * ks * kLBO) >> 4);
                mma_tf32(d, dAh + ko, dBh + ko, ks > 0 ? 1u : 0u);
                mma_tf32(d, dAh + ko, dBl + ko, 1u);
                mma_tf32(d, dAl + ko, dBh + ko, 1u);
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                     : "memory");
    };

    const int kw = warp;
    const bool mact = kw < K;
    uint64_t accp[GramPairs::NP];
    float accs[GramPairs::NSG];
    uint64_t acc1[DM / 2];
    float accn = 0.f;
#pragma unroll
    for (int j = 0; j < GramPairs::NP; ++j) accp[j] = 0;
#pragma unroll
    for (int j = 0; j < GramPairs::NSG; ++j) accs[j] = 0.f;
#pragma unroll
    for (int j = 0; j < DM / 2; ++j) acc1[j] = 0;
    double ll_acc = 0.0;
    const unsigned lt_mask = (1u << lane) - 1u;
    auto flush1 = [&](float v, int idx) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((idx & 31) == lane) sAcc[kw * C::NS + idx] += (double)v;
    };
    auto flush = [&]() {
        __syncwarp();
        if (!mact) return;
        flush1(accn, 0);
        accn = 0.f;
#pragma unroll
        for (int m = 0; m < DM / 2; ++m) {
            float lo, hi;
            unpack2(acc1[m], lo, hi);
            flush1(lo, 1 + 2 * m);
            flush1(hi, 2 + 2 * m);
            acc1[m] = 0;
        }
        int ip = 0, is = 0;
#pragma unroll
        for (int a = 0; a < DM; ++a) {
            const int base = 1 + DM + a * DM - (a * (a - 1)) / 2;
            if (a & 1) {
                flush1(accs[is], base);
                accs[is++] = 0.f;
            }
#pragma unroll
            for (int m = (a + 1) / 2; m < DM / 2; ++m) {
                float lo, hi;
                unpack2(accp[ip], lo, hi);
                flush1(lo, base + (2 * m - a));
                flush1(hi, base + (2 * m + 1 - a));
                accp[ip++] = 0;
            }
        }
    };
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;

    int64_t cur = blockIdx.x;
    int xb = 0;
    if (cur < ntiles) {
        if (t == 0) {
            prefetch(cur, 0);
            prefetch(cur + gridDim.x, 1);
        }
        aprep(cur, 0);
        tc_fence_before();
        __syncthreads();
        if (t == 0) issue_mma();
    }
    while (cur < ntiles) {
      // one flush site per super-tile of up to 64 tiles keeps the FP32
      // partials short (<= 64*8 batches per lane) and the code compact
      for (int st = 0; st < 64 && cur < ntiles; ++st) {
        const int64_t next = cur + gridDim.x;
        const bool valid = cur * kT + t < n;
        mbar_wait(bar, phase);
        phase ^= 1;
        tc_fence_after();
        // ---------------- epilogue(cur)
        float w[kKmax];
        float m = -INFINITY;
#pragma unroll
        for (int k = 0; k < kKmax; ++k) {
            float u[16];
            tmem_ld16(tmem + lane_base + 128 * sub + 16 * k, u);
            tmem_wait_ld();
            uint64_t q2 = 0;
#pragma unroll
            for (int r = 0; r < 16; r += 2) {
                const uint64_t uu = pack2(u[r], u[r + 1]);
                ffma2(q2, uu, uu);
            }
            float qa, qb;
            unpack2(q2, qa, qb);
            w[k] = sCst[k] - 0.5f * (qa + qb);
            m = fmaxf(m, w[k]);
        }
        tc_fence_before();
        float ssum = 0.f;
#pragma unroll
        for (int k = 0; k < kKmax; ++k) ssum += __expf(w[k] - m);
        const float ll = m + __logf(ssum);
        if (valid) ll_acc += (double)ll;
#pragma unroll
        for (int k = 0; k < kKmax; ++k) {
            const float gk = __expf(w[k] - ll);
            sG[k * kT + t] = gk;
            const unsigned b = __ballot_sync(0xffffffffu, valid && gk >= sThr[k]);
            if (lane == 0) bal[warp * 8 + k] = b;
        }
        __syncthreads();
        if (t < kKmax) {
            int a2 = 0;
            for (int wv = 0; wv < 8; ++wv) {
                off[wv * 8 + t] = a2;
                a2 += __popc(bal[wv * 8 + t]);
            }
            tot[t] = a2;
        }
        __syncthreads();
#pragma unroll 1
        for (int k = 0; k < kKmax; ++k) {
            const unsigned b = bal[warp * 8 + k];
            if ((b >> lane) & 1u) {
                const int p = off[warp * 8 + k] + __popc(b & lt_mask);
                lstT[k * kT + p] = (uint16_t)t;
                lstG[k * kT + p] = sG[k * kT + t];
            }
        }
        // ---------------- A-prep(next) overlaps nothing yet; MMA(next) then runs under M(cur)
        if (next < ntiles) aprep(next, xb ^ 1);
        tc_fence_before();
        __syncthreads();
        if (t == 0 && next < ntiles) {
            prefetch(next + gridDim.x, xb);  // buffer xb was consumed by aprep(cur)
            issue_mma();
        }
        // ---------------- M-phase(cur)
        if (mact) {
            const int nk = tot[kw];
            const float* nmu = sNMu + kw * DM;
            uint64_t nm2[DM / 2];
#pragma unroll
            for (int mm = 0; mm < DM / 2; ++mm) nm2[mm] = pack2(nmu[2 * mm], nmu[2 * mm + 1]);
            for (int e0 = 0; e0 < nk; e0 += 32) {
                const int e = e0 + lane;
                const bool ve = e < nk;
                const int tt = ve ? lstT[kw * kT + e] : 0;
                const float gg = ve ? lstG[kw * kT + e] : 0.f;
                const float4* xr4 = reinterpret_cast<const float4*>(sXr + (xb * kT + tt) * kXR);
                uint64_t d2[DM / 2], gd2[DM / 2];
#pragma unroll
                for (int q = 0; q < DM / 4; ++q) {
                    const float4 v = xr4[q];
                    d2[2 * q] = add2(pack2(v.x, v.y), nm2[2 * q]);
                    d2[2 * q + 1] = add2(pack2(v.z, v.w), nm2[2 * q + 1]);
                }
                accn += gg;
                const uint64_t g2 = pack2(gg, gg);
#pragma unroll
                for (int mm = 0; mm < DM / 2; ++mm) {
                    gd2[mm] = mul2(g2, d2[mm]);
                    acc1[mm] = add2(acc1[mm], gd2[mm]);
                }
                int ip = 0, is = 0;
#pragma unroll
                for (int a2 = 0; a2 < DM; ++a2) {
                    float gl, gh, dl, dh;
                    unpack2(gd2[a2 / 2], gl, gh);
                    unpack2(d2[a2 / 2], dl, dh);
                    const float ga = (a2 & 1) ? gh : gl;
                    const uint64_t ga2 = pack2(ga, ga);
                    if (a2 & 1) {
                        accs[is] = fmaf(ga, dh, accs[is]);
                        ++is;
                    }
#pragma unroll
                    for (int mm = (a2 + 1) / 2; mm < DM / 2; ++mm) {
                        ffma2(accp[ip], ga2, d2[mm]);
                        ++ip;
                    }
                }
            }
        }
        __syncthreads();
        cur = next;
        xb ^= 1;
      }
      flush();
    }
    const double bl = block_sum_d(ll_acc, sRed);
    const int SK = stat_k(D), NE = K * SK;
    double* myp = partial + (int64_t)blockIdx.x * (NE + 1);
    for (int e = t; e < NE; e += kT) {
        const int k = e / SK, r = e % SK;
        int j;
        if (r <= D) {
            j = r;
        } else {
            int p = r - 1 - D, a2 = 0;
            while (p >= D - a2) {
                p -= D - a2;
                ++a2;
            }
            const int b2 = a2 + p;
            j = 1 + DM + (a2 * DM - (a2 * (a2 - 1)) / 2 + (b2 - a2));
        }
        myp[e] = sAcc[k * C::NS + j];
    }
    if (t == 0) myp[NE] = bl;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

static size_t em_tc_smem() {
    using C = FastCfg<16>;
    size_t b = (size_t)6 * kOpBytes + (size_t)2 * 16 * kT * 8;
    b += (size_t)(2 * kT * kXR + kKmax * 16 + 2 * kKmax + 2 * kKmax * kT) * 4;
    b += (size_t)kKmax * kT * 2;
    b += (64 + 64 + 8) * 4;
    b = (b + 15) / 16 * 16;
    b += (size_t)(kKmax * C::NS + kT + 16) * 8;
    return b + 1024;
}

bool em_tc_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("ES_EM_KERNEL");
        v = (e && e[0] == 's') ? 0 : 1;  // "simt" selects k_em_fast (and "ws" is handled first)
    }
    return v == 1;
}

void launch_em_tc(const double* X, int64_t n, int64_t ld, int D, int K, const double* model, const double* center,
                  double* partial, int num_sms, int* nblk, cudaStream_t s, LaunchStats& ls) {
    *nblk = num_sms;
    static bool a = false;
    if (!a) { allow_smem(k_em_tc, em_tc_smem()); a = true; }
    k_em_tc<<<num_sms, kT, em_tc_smem(), s>>>(X, n, ld, D, K, model, center, partial);
    ++ls.launches;
}

// ============================================================ scoring pass
// Per-lane refine slots: each lane recomputes, in FP64, the components its
// event needs (candidate mask); the warp loops max-count times.
template <int DM>
__global__ void __launch_bounds__(kT) k_score_fast(const double* __restrict__ X, int64_t n, int64_t ld, int D, int K,
                                                   const double* __restrict__ model,
                                                   const double* __restrict__ center, ScoreOut o,
                                                   double* __restrict__ blocksum) {
    using C = FastCfg<DM>;
    extern __shared__ __align__(16) unsigned char smraw[];
    double* sW64 = reinterpret_cast<double*>(smraw);        // 8 * W64S
    double* sMu64 = sW64 + kKmax * C::W64S;                 // 8 * (DM+2)
    double* sLn = sMu64 + kKmax * (DM + 2);                 // 8 lognorm
    double* sLp = sLn + kKmax;                              // 8 logpi
    double* sRed = sLp + kKmax;                             // T
    double* sC = sRed + kT;                                 // DM
    float* sW = reinterpret_cast<float*>(sC + DM);          // 8*DM*DM
    float* sMu = sW + kKmax * DM * DM;
    float* sCst = sMu + kKmax * DM;
    const int t = threadIdx.x;
    ModelView mv{K, D, const_cast<double*>(model)};
    stage32<DM>(mv, center, sW, sMu, sCst);
    for (int e = t; e < kKmax * DM * DM; e += kT) {
        const int k = e / (DM * DM), rc = e % (DM * DM), r = rc / DM, cc = rc % DM;
        sW64[k * C::W64S + rc] = (k < K && r < D && cc < D) ? mv.W()[(int64_t)k * D * D + r * D + cc] : 0.0;
    }
    for (int e = t; e < kKmax * DM; e += kT) {
        const int k = e / DM, j = e % DM;
        sMu64[k * (DM + 2) + j] = (k < K && j < D) ? mv.mu()[k * D + j] : 0.0;
    }
    for (int k = t; k < kKmax; k += kT) {
        sLn[k] = k < K ? mv.lognorm()[k] : 0.0;
        sLp[k] = k < K ? mv.logpi()[k] : -INFINITY;
    }
    for (int j = t; j < DM; j += kT) sC[j] = j < D ? center[j] : 0.0;
    __syncthreads();
    double ll_acc = 0.0, nflag = 0.0;
    for (int64_t tile = blockIdx.x;; tile += gridDim.x) {
        const int64_t t0 = tile * kT;
        if (t0 >= n) break;
        const int64_t i = t0 + t;
        const bool valid = i < n;
        double x[DM];
        float xp[DM];
#pragma unroll
        for (int j = 0; j < DM; ++j) {
            x[j] = (valid && j < D) ? __ldg(X + (int64_t)j * ld + i) : 0.0;
            xp[j] = (float)(x[j] - sC[j]);
        }
        float w[kKmax], ln[kKmax];
        float m = -INFINITY, bl = -INFINITY;
#pragma unroll
        for (int k = 0; k < kKmax; ++k) {
            w[k] = -INFINITY;
            ln[k] = -INFINITY;
            if (k < K) {
                const float q = whiten32<DM>(sW + k * DM * DM, sMu + k * DM, xp);
                ln[k] = (float)sLn[k] - 0.5f * q;
                w[k] = sCst[k] - 0.5f * q;
                m = fmaxf(m, w[k]);
                bl = fmaxf(bl, ln[k]);
            }
        }
        // candidates: anything that can move ll by >= 2e-9 relative, or be the
        // weighted / unweighted argmax within FP32 rounding
        unsigned cand = 0;
#pragma unroll
        for (int k = 0; k < kKmax; ++k) {
            const float tol = 1e-3f * (1.f + fabsf(w[k]));
            if (k < K && (w[k] >= m - 20.f || ln[k] >= bl - tol)) cand |= 1u << k;
        }
        if (!valid) cand = 0;
        const int nc = __popc(cand);
        int maxc = nc;
#pragma unroll
        for (int o2 = 16; o2 > 0; o2 >>= 1) maxc = max(maxc, __shfl_xor_sync(0xffffffffu, maxc, o2));
        double w64[kKmax], ln64[kKmax];
#pragma unroll
        for (int k = 0; k < kKmax; ++k) {
            ln64[k] = (double)ln[k];
            w64[k] = (double)w[k];
        }
        unsigned rem = cand;
        for (int sl = 0; sl < maxc; ++sl) {
            const int k = rem ? __ffs(rem) - 1 : 0;
            const bool act = rem != 0;
            rem &= rem - 1;
            const double* Wk = sW64 + k * C::W64S;
            const double* mk = sMu64 + k * (DM + 2);
            double dd[DM];
#pragma unroll
            for (int j = 0; j < DM; ++j) dd[j] = x[j] - mk[j];
            double q = 0.0;
#pragma unroll
            for (int r = 0; r < DM; ++r) {
                double a = 0.0;
#pragma unroll
                for (int j = 0; j <= r; ++j) a = fma(Wk[r * DM + j], dd[j], a);
                q = fma(a, a, q);
            }
            const double l = sLn[k] - 0.5 * q;
            if (act) {
#pragma unroll
                for (int kk = 0; kk < kKmax; ++kk)
                    if (kk == k) {
                        ln64[kk] = l;
                        w64[kk] = sLp[kk] + l;
                    }
            }
        }
        // exact argmax / LSE over the refined values (ties -> lowest k)
        double mm = -INFINITY, bb = -INFINITY;
        int am = 0, ab = 0;
#pragma unroll
        for (int k = 0; k < kKmax; ++k) {
            if (k >= K) continue;
            if (w64[k] > mm) { mm = w64[k]; am = k; }
            if (ln64[k] > bb) { bb = ln64[k]; ab = k; }
        }
        double ss = 0.0;
#pragma unroll
        for (int k = 0; k < kKmax; ++k)
            if (k < K) ss += exp(w64[k] - mm);
        const double lld = mm + log(ss);
        if (valid) {
            ll_acc += lld;
            const uint8_t f = ((o.mode == 1) ? lld : bb) < o.log_delta ? 1 : 0;
            nflag += f;
            if (o.ll) o.ll[i] = lld;
            if (o.predict) o.predict[i] = am;
            if (o.best_k) o.best_k[i] = ab;
            if (o.best_ld) o.best_ld[i] = bb;
            if (o.flags) o.flags[i] = f;
        }
    }
    const double a = block_sum_d(ll_acc, sRed);
    const double b = block_sum_d(nflag, sRed);
    if (t == 0) {
        blocksum[2 * blockIdx.x] = a;
        blocksum[2 * blockIdx.x + 1] = b;
    }
}

template <int DM>
static size_t score_fast_smem() {
    using C = FastCfg<DM>;
    size_t b = (size_t)(kKmax * C::W64S + kKmax * (DM + 2) + 2 * kKmax + kT + DM) * 8;
    b += (size_t)(kKmax * DM * DM + kKmax * DM + kKmax) * 4;
    return b;
}

bool score_fast_supported(int D, int K, const ScoreOut& o) { return D <= 16 && K <= kKmax && !o.gamma && !o.lnk; }

void launch_score_fast(const double* X, int64_t n, int64_t ld, int D, int K, const double* model,
                       const double* center, const ScoreOut& o, double* blocksum, int num_sms, int* nblk,
                       cudaStream_t s, LaunchStats& ls) {
    const int grid = num_sms * 2;
    *nblk = grid;
    if (D <= 8) {
        static bool a = false;
        if (!a) { allow_smem(k_score_fast<8>, score_fast_smem<8>()); a = true; }
        k_score_fast<8><<<grid, kT, score_fast_smem<8>(), s>>>(X, n, ld, D, K, model, center, o, blocksum);
    } else {
        static bool a = false;
        if (!a) { allow_smem(k_score_fast<16>, score_fast_smem<16>()); a = true; }
        k_score_fast<16><<<grid, kT, score_fast_smem<16>(), s>>>(X, n, ld, D, K, model, center, o, blocksum);
    }
    ++ls.launches;
}

}  // namespace es
