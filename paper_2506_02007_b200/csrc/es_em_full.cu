// es_em_full.cu — mixed-precision fused E + M pass for FULL covariances beyond the
// tensor-core pass's shapes (BASELINE config c5: K = 32, D = 32; any D <= 32, K <= 32 that
// k_em_mma does not take).  FP32 arithmetic on the packed f32x2 pipe with per-component
// centring, FP64 statistics; the strict FP64 team / generic kernels remain the path for
// components with fewer than kMixedMinNk events.
//
// One persistent CTA of 512 threads per SM, tiles of T = 32 events, three phases per tile:
//   E  lane = event, warp w takes components w, w + 16: d = x^ - mu^_k,
//      z = W'_k d (W' = W / xs, FP32, packed lower triangle by feature pair in shared memory),
//      w_k = log pi_k + lognorm_k - |z|^2 / 2 -> smem
//   LSE  thread = (event, component group): max / sum over the K components (4 shuffles
//      each), ll, gamma_k -> smem
//   M  thread = (component, 4 x 4 block of the upper-triangular Gram | 4-vector of s1):
//      sum over the tile's 32 events of gamma d_a d_b in FP32 registers, then added to the
//      CTA's FP64 statistics in shared memory.
// x^ = (x - c) xs (c the data mean, xs a power of two), mu^_k = fp32((mu_k - c) xs): the
// statistics are about c + mu^_k / xs in x^ units, scaled back by xs^-1, xs^-2 (exact) --
// finalize mode 3, the format of k_em_mma.
#include <algorithm>
#include <cmath>

#include "es_kernels.h"

namespace es {

namespace {

constexpr int FD = 32;                      // features (padded)
constexpr int FK = 32;                      // components (padded)
constexpr int FT = 32;                      // events per tile
constexpr int FNT = 512;                    // threads
constexpr int FXS = FD + 4;                 // x^ tile row stride (floats): 16-byte rows, conflict-free LDS.128
constexpr int NPAIR = (FD / 2) * (FD / 2 + 1);  // 272 (row, feature-pair) entries of the lower triangle
constexpr int FP = FD * (FD + 1) / 2;       // packed upper triangle
constexpr int FSK = 1 + FD + FP;            // per-component statistics (padded shape)
constexpr int NGB = (FD / 4) * (FD / 4 + 1) / 2;  // 36 upper-triangular 4 x 4 Gram blocks
constexpr int NITEM = NGB + FD / 4;         // + 8 first-moment blocks per component

__device__ __forceinline__ uint64_t pk2(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void up2(uint64_t v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t sub2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ float ex2f(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__host__ __device__ constexpr int pair_off(int j) {  // feature pair j: rows 2j .. FD-1 from here
    return j * (FD + 1 - j);
}

struct FullSmem {
    double acc[FK][FSK];         // FP64 statistics: N_k | s1[32] | s2 packed upper (x^ units)
    float w2[FK][NPAIR][2];      // W'_k: for feature pair j, rows 2j .. 31 of (W'_rf, W'_r,f+1)
    float mu[FK][FD];            // mu^_k
    float xt[FT][FXS];           // x^ tile, event-major
    float gw[FK][FT + 1];        // w_k, then gamma_k, per (component, event)
    float cst[FK];
    double ll[FNT / 32];
};

// packed upper index of (a, b), a <= b < FD
__device__ __forceinline__ int pidx(int a, int b) { return a * FD - (a * (a - 1)) / 2 + (b - a); }

}  // namespace

__global__ void __launch_bounds__(FNT, 1) k_em_full_mixed(const double* __restrict__ X, int64_t n, int64_t ld, int D,
                                                          int K, const double* __restrict__ model,
                                                          const double* __restrict__ center, double xs,
                                                          double* __restrict__ partial) {
    extern __shared__ __align__(16) unsigned char smraw[];
    FullSmem& S = *reinterpret_cast<FullSmem*>(smraw);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    ModelView mv{K, D, const_cast<double*>(model)};
    // ---- staging: W' = W / xs as row pairs, mu^ = fp32((mu - c) xs), constants, zeroed stats
    for (int e = t; e < FK * FSK; e += FNT) (&S.acc[0][0])[e] = 0.0;
    for (int e = t; e < FK * NPAIR; e += FNT) {
        const int k = e / NPAIR, pr = e % NPAIR;
        int j = 0;
        while (j + 1 < FD / 2 && pair_off(j + 1) <= pr) ++j;
        const int r = 2 * j + (pr - pair_off(j)), f = 2 * j;
        float a = 0.f, b = 0.f;
        if (k < K && r < D) {
            const double* Wr = mv.W() + (int64_t)k * D * D + (int64_t)r * D;
            if (f <= r && f < D) a = (float)(Wr[f] / xs);
            if (f + 1 <= r && f + 1 < D) b = (float)(Wr[f + 1] / xs);
        }
        S.w2[k][pr][0] = a;
        S.w2[k][pr][1] = b;
    }
    for (int e = t; e < FK * FD; e += FNT) {
        const int k = e / FD, f = e % FD;
        S.mu[k][f] = (k < K && f < D) ? (float)((mv.mu()[k * D + f] - center[f]) * xs) : 0.f;
    }
    for (int k = t; k < FK; k += FNT) S.cst[k] = k < K ? (float)(mv.logpi()[k] + mv.lognorm()[k]) : -INFINITY;
    // tile staging: thread t loads event t % 32 of planes 2 (t / 32), + 1 (coalesced by plane)
    const int se = t & (FT - 1), sp = (t >> 5) * 2;
    double pf[2];
    const int64_t ntiles = (n + FT - 1) / FT;
    auto fetch = [&](int64_t tile) {
        const int64_t i = tile * FT + se;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int f = sp + j;
            pf[j] = (i < n && f < D) ? __ldg(X + (int64_t)f * ld + i) : center[f < D ? f : 0];
        }
    };
    double llacc = 0.0;
    float llf = 0.f;
    int64_t jt = 0;
    if (blockIdx.x < ntiles) fetch(blockIdx.x);
    __syncthreads();
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++jt) {
        const int nt = (int)std::min<int64_t>(FT, n - tile * FT);
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int f = sp + j;
            S.xt[se][f] = f < D ? (float)((pf[j] - center[f]) * xs) : 0.f;
        }
        __syncthreads();  // tile staged; the previous tile's M phase is done
        if (tile + gridDim.x < ntiles) fetch(tile + gridDim.x);
        // ---------------------------------------------------------------- E phase
        // lane = event, warp w: components w, w + 16; z_r accumulated over feature pairs j
        // (rows r >= 2j) as f32x2 partial sums, W' read two rows per 16-byte load
        {
            const int e = lane;
            for (int k = warp; k < K; k += FNT / 32) {
                uint64_t a2[FD];
#pragma unroll
                for (int r = 0; r < FD; ++r) a2[r] = 0;
                const uint64_t* xr = reinterpret_cast<const uint64_t*>(&S.xt[e][0]);
                const uint64_t* m2 = reinterpret_cast<const uint64_t*>(&S.mu[k][0]);
                const ulonglong2* wk = reinterpret_cast<const ulonglong2*>(&S.w2[k][0][0]);
#pragma unroll
                for (int j = 0; j < FD / 2; ++j) {
                    const uint64_t d2 = sub2(xr[j], m2[j]);
#pragma unroll
                    for (int r = 2 * j; r < FD; r += 2) {
                        const ulonglong2 w = wk[(pair_off(j) + r - 2 * j) / 2];
                        a2[r] = fma2(w.x, d2, a2[r]);
                        a2[r + 1] = fma2(w.y, d2, a2[r + 1]);
                    }
                }
                float q = 0.f;
#pragma unroll
                for (int r = 0; r < FD; ++r) {
                    float za, zb;
                    up2(a2[r], za, zb);
                    const float z = za + zb;
                    q = fmaf(z, z, q);
                }
                S.gw[k][e] = S.cst[k] - 0.5f * q;
            }
        }
        __syncthreads();
        // --------------------------------------------------------------- LSE phase
        {
            const int e = t >> 4, g = t & 15;  // event, component group (k = g, g + 16)
            float wv[FK / 16];
            float m = -INFINITY;
#pragma unroll
            for (int i = 0; i < FK / 16; ++i) {
                const int k = g + 16 * i;
                wv[i] = k < K ? S.gw[k][e] : -INFINITY;
                m = fmaxf(m, wv[i]);
            }
#pragma unroll
            for (int o = 1; o < 16; o <<= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            float s = 0.f;
#pragma unroll
            for (int i = 0; i < FK / 16; ++i) {
                wv[i] = g + 16 * i < K ? ex2f((wv[i] - m) * 1.4426950408889634f) : 0.f;
                s += wv[i];
            }
#pragma unroll
            for (int o = 1; o < 16; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            const bool valid = e < nt;
            const float inv = 1.f / s;
#pragma unroll
            for (int i = 0; i < FK / 16; ++i) {
                const int k = g + 16 * i;
                if (k < K) S.gw[k][e] = valid ? wv[i] * inv : 0.f;
            }
            if (valid && g == 0) llf += m + __logf(s);
        }
        __syncthreads();
        // ----------------------------------------------------------------- M phase
        for (int it = t; it < K * NITEM; it += FNT) {
            const int k = it / NITEM, r = it % NITEM;
            const float* gk = &S.gw[k][0];
            if (r < NGB) {  // Gram block (ab, bb), ab <= bb, 4 x 4
                int ab = 0, rr = r;
                while (rr >= FD / 4 - ab) {
                    rr -= FD / 4 - ab;
                    ++ab;
                }
                const int bb = ab + rr;
                const float4 ma = *reinterpret_cast<const float4*>(&S.mu[k][4 * ab]);
                const float4 mb = *reinterpret_cast<const float4*>(&S.mu[k][4 * bb]);
                const uint64_t ma0 = pk2(ma.x, ma.y), ma1 = pk2(ma.z, ma.w);
                const uint64_t mb0 = pk2(mb.x, mb.y), mb1 = pk2(mb.z, mb.w);
                uint64_t acc[4][2] = {};
#pragma unroll 4
                for (int e = 0; e < nt; ++e) {
                    const float4 xa = *reinterpret_cast<const float4*>(&S.xt[e][4 * ab]);
                    const float4 xb = *reinterpret_cast<const float4*>(&S.xt[e][4 * bb]);
                    const float g = gk[e];
                    const uint64_t g2 = pk2(g, g);
                    const uint64_t da0 = mul2(sub2(pk2(xa.x, xa.y), ma0), g2);
                    const uint64_t da1 = mul2(sub2(pk2(xa.z, xa.w), ma1), g2);
                    const uint64_t db0 = sub2(pk2(xb.x, xb.y), mb0), db1 = sub2(pk2(xb.z, xb.w), mb1);
                    float a0, a1, a2, a3;
                    up2(da0, a0, a1);
                    up2(da1, a2, a3);
                    const float av[4] = {a0, a1, a2, a3};
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const uint64_t ai = pk2(av[i], av[i]);
                        acc[i][0] = fma2(ai, db0, acc[i][0]);
                        acc[i][1] = fma2(ai, db1, acc[i][1]);
                    }
                }
                double* ak = S.acc[k];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    float v[4];
                    up2(acc[i][0], v[0], v[1]);
                    up2(acc[i][1], v[2], v[3]);
                    const int a = 4 * ab + i;
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) {
                        const int b = 4 * bb + jj;
                        if (a <= b) ak[1 + FD + pidx(a, b)] += (double)v[jj];
                    }
                }
            } else {  // first-moment block ab (and N_k with ab == 0)
                const int ab = r - NGB;
                const float4 ma = *reinterpret_cast<const float4*>(&S.mu[k][4 * ab]);
                const uint64_t ma0 = pk2(ma.x, ma.y), ma1 = pk2(ma.z, ma.w);
                uint64_t s0 = 0, s1 = 0;
                float nk = 0.f;
#pragma unroll 4
                for (int e = 0; e < nt; ++e) {
                    const float4 xa = *reinterpret_cast<const float4*>(&S.xt[e][4 * ab]);
                    const float g = gk[e];
                    const uint64_t g2 = pk2(g, g);
                    s0 = fma2(sub2(pk2(xa.x, xa.y), ma0), g2, s0);
                    s1 = fma2(sub2(pk2(xa.z, xa.w), ma1), g2, s1);
                    nk += g;
                }
                double* ak = S.acc[k];
                float v[4];
                up2(s0, v[0], v[1]);
                up2(s1, v[2], v[3]);
#pragma unroll
                for (int i = 0; i < 4; ++i) ak[1 + 4 * ab + i] += (double)v[i];
                if (ab == 0) ak[0] += (double)nk;
            }
        }
        if ((jt & 7) == 7) {  // ll: FP32 over 8 tiles, then FP64
            llacc += (double)llf;
            llf = 0.f;
        }
        // the next iteration's __syncthreads (after staging) orders the M phase before reuse
        __syncthreads();
    }
    llacc += (double)llf;
    // per-warp ll (threads with g == 0 hold it), fixed order
    {
        double v = (t & 15) == 0 ? llacc : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) S.ll[warp] = v;
    }
    __syncthreads();
    // CTA partial block (canonical layout, real D): x^ units -> x units (xs^-1, xs^-2, exact)
    const int SK = stat_k(D), NE = K * SK;
    double* myp = partial + (int64_t)blockIdx.x * (NE + 1);
    const double i1 = 1.0 / xs, i2 = i1 * i1;
    for (int e = t; e < NE; e += FNT) {
        const int k = e / SK, r = e % SK;
        double v;
        if (r == 0) {
            v = S.acc[k][0];
        } else if (r <= D) {
            v = S.acc[k][r] * i1;
        } else {
            int p2 = r - 1 - D, a = 0;
            while (p2 >= D - a) {
                p2 -= D - a;
                ++a;
            }
            v = S.acc[k][1 + FD + pidx(a, a + p2)] * i2;
        }
        myp[e] = v;
    }
    if (t == 0) {
        double v = 0.0;
        for (int w = 0; w < FNT / 32; ++w) v += S.ll[w];
        myp[NE] = v;
    }
}

bool em_full_mixed_supported(int D, int K) { return D <= FD && K <= FK; }

void launch_em_full_mixed(const double* X, int64_t n, int64_t ld, int D, int K, const double* model,
                          const double* center, double xs, double* partial, int num_sms, int* nblk, cudaStream_t s,
                          LaunchStats& ls) {
    const int64_t ntiles = (n + FT - 1) / FT;
    const int grid = (int)std::min<int64_t>(num_sms, std::max<int64_t>(ntiles, 1));
    *nblk = grid;
    const size_t smem = sizeof(FullSmem);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_em_full_mixed, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    k_em_full_mixed<<<grid, FNT, smem, s>>>(X, n, ld, D, K, model, center, xs, partial);
    ++ls.launches;
}

}  // namespace es
