// es_em_diag.cu — mixed-precision fused E + M pass for DIAGONAL covariances (BASELINE
// config c3: K = 16, D = 16; an extension, the reference has no diagonal variant,
// SPEC.md:332).  Used when every component holds >= kOnePassMinNk events; smaller
// components keep the FP64 team kernel k_em_diag (es_kernels.cu).
//
// Layout: one persistent CTA of 512 threads per SM; a team of 16 lanes per event, lane
// k = component k (2 events per warp, 32 teams).  Event tiles of 256 rows are staged
// from the planar FP64 matrix with coalesced loads (the next tile held in registers
// while the current one is evaluated) as FP32 offsets x^ = x - c from the data mean c.
// Per (event, k), all on the FP32 pipe in packed f32x2 form, in scaled coordinates:
//   d' = x^ s_k - fp32(mu^_k s_k) (s_k = fp32(1 / sigma_k), mu^_k = fp32(mu_k - c); one FMA),
//   q = |d'|^2,  w = (log pi_k + lognorm_k) - q / 2;  team max / sum (shuffles) -> ll, gamma_k;
//   N_k += gamma, s1' += gamma d', s2' += gamma d'^2  (FP32 over 32 events per lane, then
// added to per-lane FP64 accumulators in shared memory), logL in FP64.  The output unscales
// (1 / s, 1 / s^2) and re-centres the moments from fp32(mu^ s) / s onto mu^ exactly in FP64:
// statistics about c + mu^_k (finalize mode 4: diagonal, fp32-rounded centre).
//
// Precision: per-event w error ~2^-24 (|x^| + |mu^|) |d| / sigma^2,
// random across events; the FP32 partial sums cover 32 events before the FP64 flush.
#include <algorithm>
#include <cmath>

#include "es_kernels.h"

namespace es {

namespace {

constexpr int DG = 16;        // features (padded)
constexpr int TSD = 16;       // team size = max components
constexpr int NTD = 512;      // threads per CTA
constexpr int ROWS = 256;     // events per staged tile
constexpr int NTEAM = NTD / TSD;
constexpr int NACC = 1 + 2 * DG;  // N | s1[16] | s2[16]
constexpr int FLUSH_TILES = 4;    // FP32 partial sums over FLUSH_TILES * ROWS / NTEAM = 32 events

__device__ __forceinline__ uint64_t pk2(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void up2(uint64_t v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
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

// 1 / sigma_kf (fp32) and mu^_kf = fp32(mu_kf - c_f): shared by the lanes' set-up and the output
// re-centring, so both use bit-identical values
__device__ __forceinline__ float diag_scale(const ModelView& mv, int k, int f) {
    return (float)sqrt(1.0 / mv.cov()[(int64_t)k * mv.D * mv.D + f * mv.D + f]);
}
__device__ __forceinline__ float diag_centre(const ModelView& mv, const double* center, int k, int f) {
    return (float)(mv.mu()[k * mv.D + f] - center[f]);
}

struct DiagSmem {
    float x[2][ROWS][DG];        // staged tiles, row-major x^ (FP32)
    double acc[NTD][NACC + 1];   // per-lane FP64 accumulators (+1: bank skew)
    double ll[NTD / 32];
    double c[DG];
};

}  // namespace

__global__ void __launch_bounds__(NTD, 1) k_em_diag_mixed(const double* __restrict__ X, int64_t n, int64_t ld,
                                                          int D, int K, const double* __restrict__ model,
                                                          const double* __restrict__ center,
                                                          double* __restrict__ partial) {
    extern __shared__ __align__(16) unsigned char smraw[];
    DiagSmem& S = *reinterpret_cast<DiagSmem*>(smraw);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int k = lane & (TSD - 1);  // component of this lane
    const int team = t / TSD;
    const bool kact = k < K;
    ModelView mv{K, D, const_cast<double*>(model)};
    for (int f = t; f < DG; f += NTD) S.c[f] = f < D ? center[f] : 0.0;
    for (int e = t; e < NTD * (NACC + 1); e += NTD) (&S.acc[0][0])[e] = 0.0;
    // this lane's component, in scaled coordinates d' = x^ s - mu^ s (s = 1 / sigma, fp32): one
    // f32x2 FMA forms d', another accumulates |d'|^2 (0 on padded features)
    uint64_t s2v[DG / 2], nms2[DG / 2];
    float cst = -INFINITY;
    {
        float sc[DG], nms[DG];
#pragma unroll
        for (int f = 0; f < DG; ++f) {
            const bool on = kact && f < D;
            sc[f] = on ? diag_scale(mv, k, f) : 0.f;
            nms[f] = on ? -(diag_centre(mv, center, k, f) * sc[f]) : 0.f;
        }
#pragma unroll
        for (int f = 0; f < DG; f += 2) {
            s2v[f / 2] = pk2(sc[f], sc[f + 1]);
            nms2[f / 2] = pk2(nms[f], nms[f + 1]);
        }
        if (kact) cst = (float)(mv.logpi()[k] + mv.lognorm()[k]);
    }
    __syncthreads();
    // staging: thread t loads event t % 256 of a tile, planes 8 (t / 256) .. + 7
    const int se = t & (ROWS - 1), sp = (t >> 8) * 8;
    const int64_t ntiles = (n + ROWS - 1) / ROWS;
    double pf[8];
    auto fetch = [&](int64_t tile) {
        const int64_t i = tile * ROWS + se;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int f = sp + j;
            pf[j] = (i < n && f < D) ? __ldg(X + (int64_t)f * ld + i) : S.c[f];  // centred at stage time
        }
    };
    auto stage = [&](int b) {
        float4* dst = reinterpret_cast<float4*>(&S.x[b][se][sp]);
        const double* cc = S.c + sp;
        dst[0] = make_float4((float)(pf[0] - cc[0]), (float)(pf[1] - cc[1]), (float)(pf[2] - cc[2]),
                             (float)(pf[3] - cc[3]));
        dst[1] = make_float4((float)(pf[4] - cc[4]), (float)(pf[5] - cc[5]), (float)(pf[6] - cc[6]),
                             (float)(pf[7] - cc[7]));
    };
    uint64_t s1[DG / 2], s2[DG / 2];
    float nk = 0.f, llf = 0.f;  // llf: sum of ll over the flush window (used from lane k = 0)
    double llacc = 0.0;
#pragma unroll
    for (int f = 0; f < DG / 2; ++f) s1[f] = s2[f] = 0;
    auto flush = [&]() {  // FP32 partial sums -> this lane's FP64 accumulators
        double* a = S.acc[t];
        a[0] += (double)nk;
#pragma unroll
        for (int f = 0; f < DG / 2; ++f) {
            float u0, u1, v0, v1;
            up2(s1[f], u0, u1);
            up2(s2[f], v0, v1);
            a[1 + 2 * f] += (double)u0;
            a[2 + 2 * f] += (double)u1;
            a[1 + DG + 2 * f] += (double)v0;
            a[2 + DG + 2 * f] += (double)v1;
            s1[f] = s2[f] = 0;
        }
        nk = 0.f;
        llacc += (double)llf;
        llf = 0.f;
    };
    int64_t jt = 0;
    if (blockIdx.x < ntiles) fetch(blockIdx.x);
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++jt) {
        const int b = (int)(jt & 1);
        stage(b);
        __syncthreads();  // tile b staged (and tile b of two rounds ago consumed)
        if (tile + gridDim.x < ntiles) fetch(tile + gridDim.x);
#pragma unroll 2
        for (int r = 0; r < ROWS / NTEAM; ++r) {
            const int e = team + NTEAM * r;
            const bool valid = tile * ROWS + e < n;
            const float4* xr = reinterpret_cast<const float4*>(&S.x[b][e][0]);
            uint64_t d2[DG / 2];
            uint64_t qa = 0, qb = 0;
#pragma unroll
            for (int v = 0; v < DG / 4; ++v) {
                const float4 xv = xr[v];
                d2[2 * v] = fma2(pk2(xv.x, xv.y), s2v[2 * v], nms2[2 * v]);
                d2[2 * v + 1] = fma2(pk2(xv.z, xv.w), s2v[2 * v + 1], nms2[2 * v + 1]);
                qa = fma2(d2[2 * v], d2[2 * v], qa);
                qb = fma2(d2[2 * v + 1], d2[2 * v + 1], qb);
            }
            float q0, q1, q2, q3;
            up2(qa, q0, q1);
            up2(qb, q2, q3);
            const float w = cst - 0.5f * ((q0 + q1) + (q2 + q3));
            float m = w;
#pragma unroll
            for (int o = 1; o < TSD; o <<= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            const float ex = kact ? ex2f((w - m) * 1.4426950408889634f) : 0.f;
            float sum = ex;
#pragma unroll
            for (int o = 1; o < TSD; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
            const float g = valid ? __fdividef(ex, sum) : 0.f;
            if (valid) llf += m + __logf(sum);  // kept by lane k = 0 of the team
            nk += g;
            const uint64_t g2 = pk2(g, g);
#pragma unroll
            for (int f = 0; f < DG / 2; ++f) {
                const uint64_t gd = mul2(g2, d2[f]);
                s1[f] = add2(s1[f], gd);
                s2[f] = fma2(gd, d2[f], s2[f]);
            }
        }
        if ((jt + 1) % FLUSH_TILES == 0) flush();
    }
    flush();
    {  // the 2 teams of this warp (their k = 0 lanes 0, 16 hold logL), fixed order
        const double o = __shfl_down_sync(0xffffffffu, llacc, 16);
        if (lane == 0) S.ll[warp] = llacc + o;
    }
    __syncthreads();
    // CTA partial block: component kc, entry j summed over the 32 teams in order
    const int SK = stat_k(D), NE = K * SK;
    double* myp = partial + (int64_t)blockIdx.x * (NE + 1);
    for (int e = t; e < NE; e += NTD) {
        const int kc = e / SK, rr = e % SK;
        int j = -1;
        if (rr <= D) {
            j = rr;  // N, s1
        } else {
            int p2i = rr - 1 - D, a = 0;
            while (p2i >= D - a) {
                p2i -= D - a;
                ++a;
            }
            if (p2i == 0) j = 1 + DG + a;  // diagonal entry (a, a)
        }
        double v = 0.0;
        if (j >= 0) {
            auto tsum = [&](int jj) {
                double a = 0.0;
                for (int tm = 0; tm < NTEAM; ++tm) a += S.acc[tm * TSD + kc][jj];
                return a;
            };
            // scaled moments about m = (mu^ s)_fp32 / s -> moments about mu^ (finalize mode 4), FP64
            v = tsum(j);
            if (j > 0) {
                const int f = j <= DG ? j - 1 : j - 1 - DG;
                const double sf = (double)diag_scale(mv, kc, f);
                const double mf = (double)diag_centre(mv, center, kc, f);
                const double dl = (double)(float)(mf * sf) / sf - mf;  // centre of the scaled moments - mu^
                const double Nk = tsum(0), s1 = tsum(1 + f) / sf;
                v = j <= DG ? s1 + Nk * dl : v / (sf * sf) + 2.0 * dl * s1 + Nk * dl * dl;
            }
        }
        myp[e] = v;
    }
    if (t == 0) {
        double v = 0.0;
        for (int wv = 0; wv < NTD / 32; ++wv) v += S.ll[wv];
        myp[NE] = v;
    }
}

bool em_diag_mixed_supported(int D, int K) { return D <= DG && K <= TSD; }

void launch_em_diag_mixed(const double* X, int64_t n, int64_t ld, int D, int K, const double* model,
                          const double* center, double* partial, int num_sms, int* nblk, cudaStream_t s,
                          LaunchStats& ls) {
    const int64_t ntiles = (n + ROWS - 1) / ROWS;
    const int grid = (int)std::min<int64_t>(num_sms, std::max<int64_t>(ntiles, 1));
    *nblk = grid;
    const size_t smem = sizeof(DiagSmem);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_em_diag_mixed, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    k_em_diag_mixed<<<grid, NTD, smem, s>>>(X, n, ld, D, K, model, center, partial);
    ++ls.launches;
}

}  // namespace es
