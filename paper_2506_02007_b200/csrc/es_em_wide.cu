// es_em_wide.cu — fused EM pass on the 5th-gen tensor cores for full covariances up to
// D = 32, K = 32 (BASELINE config c5: D = K = 32, the shape where the whitening work
// K * D^2 per event is largest).  The reference op is SPEC.md:291-299 (fit_em, E + M);
// the numerics follow k_em_mma (es_em_mma.cu) with one-fp16 records.
//
// Components are processed in groups of CG = 4 (E-step N = M-step M = 4 * 32 = 128).
// Per 128-event tile, one persistent CTA per SM:
//   TMA warp      the group images of the E-step operand (W'/t_k as fp16 hi + lo for the
//                 two 16-feature K-steps, and fp32(b'/t_k) as three fp16 parts), prepared
//                 once per pass in global memory by k_wide_stage, streamed group by group
//                 into a 3-slot ring (the whole set, 8 x 20 KB, does not fit next to the
//                 accumulators; it stays L2-resident).
//   MMA warp      E:  U = b' + W' x^ per group, over KS = ceil(D / 13) K-steps of 13 features
//                     plus three bias columns each (see k_wide_stage): 3 * KS kind::f16
//                     dispatches M128 N128 K16 with A (x^ hi / lo and ones) in TMEM, into one
//                     of two TMEM E regions;
//                 M:  per group the Gram of the tile's records R = s_k (x^ - m_k) over its
//                     128 events (8 K-steps of 16), M = 128 rows (k, a): NPASS = 1 one fp16
//                     record per value, R_h^T [R_h | s_h]; NPASS = 2 (fewer than 2^20 events
//                     in some component) records R_h + R_l and the symmetric three-product
//                     Gram R_h^T [R_h | s_h | s_l] + R_l^T [R_h | s_h] + R_h^T R_l.
//   epilogue WG   thread = event = TMEM lane: loads its FP64 row (coalesced, the next tile
//                 prefetched to L2), x^ = (x - c) xs -> FP32 + fp16 hi/lo A operands;
//                 |U_k|^2 -> w_k for the K components; log-sum-exp; s_k = sqrt(gamma_k);
//                 N_k by a warp transpose-reduce; the records of each group;
//                 thread = Gram row (k, a): adds the upper part of the group's Gram row (its
//                 4-column chunks from column 4 floor(a / 4) on) and the first moment into
//                 FP32 shared-memory accumulators (144 chunks per component).
//   Every 16 tiles (and after local tiles 1, 2, 4, 8) the FP32 accumulators are added into
//   the CTA's FP64 partial block in global memory; after tiles 1, 2, 4, ... the record
//   centres m_k move to the CTA's running estimate of the new means with the exact FP64
//   re-expression P' = P - s1 d^T - d s1^T + N d d^T (as k_em_mma), and at the end the
//   statistics are re-expressed about the starting centre c + fp32((mu_k - c) xs) / xs and
//   scaled to x units: finalize mode 3.
#include <cmath>
#include <cstdlib>
#include <cuda_fp16.h>

#include "es_kernels.h"
#include "es_mma.cuh"

namespace es {

namespace {

using namespace mma;

constexpr int WD = 32;                     // features (padded)
constexpr int WK = 32;                     // components (padded)
constexpr int CG = 4;                      // components per group
constexpr uint32_t WOP = 4096;             // 128 rows x 16 K fp16 operand, K-major, SWIZZLE_NONE
constexpr int FKS = 13;                    // features per E-step K-step (+ 3 bias columns)
constexpr int KSMAX = (WD + FKS - 1) / FKS;  // 3
constexpr uint32_t WIMG = 2 * KSMAX * WOP; // group image: (hi, lo) per K-step
constexpr uint32_t RG = (TM / 8) * 128;    // 2048 B: one MN-major 8-column group of records
constexpr int RHG = 18, RLG = 16;          // record groups: R_h (16) | s_h | s_l, then R_l (NPASS = 2)
// NPASS = 1: two R_h buffers (the records of group m are written while the Gram of group m - 1
// runs); NPASS = 2: one R_h + R_l buffer
constexpr uint32_t RECB = (2 * RHG > RHG + RLG ? 2 * RHG : RHG + RLG) * RG;
constexpr int NSLOT = 3;                   // group-image ring slots
constexpr int WNT = 128 + 64;              // epilogue WG, TMA warp, MMA warp
constexpr int TE = 0, TGR = 256, TAX = 400;  // TMEM columns: E x 2, Gram (144), A (hi, lo) x KSMAX
constexpr int FLUSH = 16;                  // FP32 accumulation window (tiles)
constexpr int ACH = 144;                   // FP32 accumulator chunks (4 floats) per component

struct WSmem {
    unsigned char w[NSLOT][WIMG];          // 72 KB group-image ring
    unsigned char rec[RECB];               // 68 KB records (FP64 recentring scratch between tiles)
    float4 acc[WK * ACH];                  // 72 KB upper Gram chunks: row a holds chunks floor(a/4) .. 7
    float mom[WK * WD];                    // first moments
    float nmu[WK * WD];                    // -(record centre), x^ units, FP32
    float cst[WK], hq[WK];                 // log pi_k + lognorm_k, t_k^2 / 2
    double nkw[4][WK];
    double llw[4];
    uint64_t wfull[NSLOT], wfree[NSLOT], aready, edone[2], efree[2], mready, mdone, gfree;
    uint32_t tmem;
};

// first chunk of accumulator row a, minus floor(a / 4): chunk c (>= floor(a / 4)) at row_base(a) + c
__device__ __forceinline__ int row_base(int a) {
    const int i = a >> 2, j = a & 3;
    return 4 * (8 * i - i * (i - 1) / 2) + j * (8 - i) - i;
}

__device__ __forceinline__ void tmem_ld32w(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr)
        : "memory");
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
}

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

}  // namespace

// E-step operand images of the groups (block g = components 4g .. 4g+3) and the per-component
// constants cst = log pi + lognorm, hq = t_k^2 / 2 (consts[0..31], consts[32..63]).
// Rows (k_local, a) = 32 k_local + a of W'/t_k (W' = W / xs, lower triangular).  K-step s
// holds features F_s = [13 s, 13 s + 13) in K columns 0-12 and, in columns 13-15, its own part
// of the bias b_s = -sum_{f in F_s} W'_af mu^_f / t_k (mu^ = (mu - c) xs) rounded to FP32 and
// split exactly into three fp16 parts (the A operand has ones there).  Every dispatch then adds
// W'_{F_s} (x^ - mu^)_{F_s}: the accumulator's running sums stay of the size of the whitened
// residual for the events that matter to component k (near mu_k), instead of passing through
// |W' x^| ~ |b'|, where the FP32 truncation of each dispatch would bias U.  W' hi + lo fp16.
// t_k (a power of two) puts each component's largest |entry| into (2^12, 2^13] (as stage_estep).
__global__ void k_wide_stage(const double* __restrict__ model, int K, int D, const double* __restrict__ center,
                             double xs, unsigned char* __restrict__ wimg, float* __restrict__ consts) {
    ModelView mv{K, D, const_cast<double*>(model)};
    const int g = blockIdx.x, t = threadIdx.x;
    __shared__ double tks[CG];
    __shared__ double bias[TM][KSMAX];
    for (int e = t; e < TM * KSMAX; e += blockDim.x) {  // partial biases (unscaled)
        const int row = e / KSMAX, sidx = e % KSMAX, kl = row / WD, a = row % WD, k = CG * g + kl;
        double b = 0.0;
        if (k < K && a < D) {
            const double* Wr = mv.W() + (int64_t)k * D * D + (int64_t)a * D;
            for (int f = FKS * sidx; f < FKS * sidx + FKS && f <= a; ++f)
                b = fma(Wr[f], mv.mu()[k * D + f] - center[f], b);
        }
        bias[row][sidx] = -b;
    }
    __syncthreads();
    if (t < CG) {
        const int k = CG * g + t;
        double tk = 1.0;
        float cst = -INFINITY;
        if (k < K) {
            cst = (float)(mv.logpi()[k] + mv.lognorm()[k]);
            double m = 0.0;
            const double* W = mv.W() + (int64_t)k * D * D;
            for (int a = 0; a < D; ++a) {
                for (int f = 0; f <= a; ++f) m = fmax(m, fabs(W[a * D + f] / xs));
                for (int sidx = 0; sidx < KSMAX; ++sidx) m = fmax(m, fabs(bias[t * WD + a][sidx]));
            }
            if (m > 0.0) tk = exp2(ceil(log2(m)) - 13.0);
        }
        tks[t] = tk;
        consts[k] = cst;
        consts[WK + k] = (float)(0.5 * tk * tk);
    }
    __syncthreads();
    unsigned char* img = wimg + (size_t)g * WIMG;
    for (int e = t; e < TM * 16 * KSMAX; e += blockDim.x) {
        const int row = e / (16 * KSMAX), cs = e % (16 * KSMAX), sidx = cs / 16, col = cs % 16;
        const int kl = row / WD, a = row % WD, k = CG * g + kl, f = FKS * sidx + col;
        __half wh = __half(0.f), wl = __half(0.f);
        if (col < FKS) {
            double w = 0.0;
            if (k < K && a < D && f <= a) w = mv.W()[(int64_t)k * D * D + a * D + f] / xs / tks[kl];
            wh = __double2half(w);
            wl = __double2half(w - (double)__half2float(wh));
        } else {  // fp32(b_s / t_k) in three exact fp16 parts (hi image); the lo image holds zeros
            const float b32 = (float)(bias[row][sidx] / tks[kl]);
            const __half bh = __float2half_rn(b32);
            const float r1 = b32 - __half2float(bh);
            const __half bm = __float2half_rn(r1);
            const __half bl = __float2half_rn(r1 - __half2float(bm));
            wh = col == FKS ? bh : (col == FKS + 1 ? bm : bl);
        }
        *reinterpret_cast<__half*>(img + (2 * sidx) * WOP + kmaj(row, col)) = wh;
        *reinterpret_cast<__half*>(img + (2 * sidx + 1) * WOP + kmaj(row, col)) = wl;
    }
}

struct NegCxW {
    double v[WD];
};
struct NegCxWF {
    float v[WD];
};

template <int NPASS, bool F32>
__global__ void __launch_bounds__(WNT, 1)
    k_em_wide(const double* __restrict__ X, int64_t n, int64_t ld, int D, int K, const double* __restrict__ model,
              const double* __restrict__ center, double xs, const __grid_constant__ NegCxW ncx,
              const __grid_constant__ NegCxWF ncxf, float xsf, const unsigned char* __restrict__ wimg,
              const float* __restrict__ consts, double* __restrict__ partial, float qscale) {
    extern __shared__ __align__(128) unsigned char smraw[];
    WSmem& S = *reinterpret_cast<WSmem*>(smraw + ((128u - (su32(smraw) & 127u)) & 127u));
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    ModelView mv{K, D, const_cast<double*>(model)};
    const int NG = (K + CG - 1) / CG, KS = (D + FKS - 1) / FKS;
    const int SK = stat_k(D), NE = K * SK;
    double* part = partial + (int64_t)blockIdx.x * (NE + 1);
    const int64_t ntiles = (n + TM - 1) / TM;
    const int64_t J = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    // ------------------------------------------------------------------ staging
    for (int e = t; e < NE + 1; e += WNT) part[e] = 0.0;
    for (int e = t; e < WK * ACH; e += WNT) S.acc[e] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int e = t; e < WK * WD; e += WNT) {
        const int k = e / WD, a = e % WD;
        S.mom[e] = 0.f;
        S.nmu[e] = (k < K && a < D) ? -(float)((mv.mu()[k * D + a] - center[a]) * xs) : 0.f;
    }
    for (int k = t; k < WK; k += WNT) {
        S.cst[k] = consts[k];
        S.hq[k] = consts[WK + k] * qscale;
    }
    if (warp == 5) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&S.tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        for (int i = 0; i < NSLOT; ++i) {
            mbar_init(&S.wfull[i], 1);
            mbar_init(&S.wfree[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&S.edone[i], 1);
            mbar_init(&S.efree[i], 4);
        }
        mbar_init(&S.aready, 4);
        mbar_init(&S.mready, 4);
        mbar_init(&S.mdone, 1);
        mbar_init(&S.gfree, 4);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    proxy_fence();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = S.tmem;

    auto tile_of = [&](int64_t j) { return (int64_t)blockIdx.x + j * gridDim.x; };

    if (warp < 4) {
        // ========================================================= epilogue warpgroup
        const int p = t;                            // event of the tile / Gram row (kl, a)
        const uint32_t lq = (uint32_t)(32 * warp) << 16;
        double ll_acc = 0.0, nkp = 0.0;             // nkp: N_k partial of component `lane` (this warp)

        // FP32 window -> FP64 partial block (fixed order; N_k from the warps' partials)
        auto flush64 = [&]() {
            S.nkw[warp][lane] = nkp;
            nkp = 0.0;
            named_sync(1, 128);
            for (int r = p; r < K * WD; r += 128) {
                const int k = r / WD, a = r % WD;
                if (a >= D) continue;
                double* __restrict__ blk = part + (int64_t)k * SK;
                if (a == 0) blk[0] += ((S.nkw[0][k] + S.nkw[1][k]) + S.nkw[2][k]) + S.nkw[3][k];
                blk[1 + a] += (double)S.mom[k * WD + a];
                double* __restrict__ s2 = blk + 1 + D + packed_index(a, a, D);
                const float4* rowp = S.acc + k * ACH + row_base(a);
#pragma unroll
                for (int c = 0; c < WD / 4; ++c) {  // a chunk of FP64 entries loaded together
                    if (4 * c + 3 < a || 4 * c >= D) continue;
                    const float4 q = rowp[c];
                    const float qv[4] = {q.x, q.y, q.z, q.w};
                    double v[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (4 * c + j >= a && 4 * c + j < D) v[j] = s2[4 * c + j - a];
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (4 * c + j >= a && 4 * c + j < D) s2[4 * c + j - a] = v[j] + (double)qv[j];
                }
            }
            named_sync(1, 128);
            for (int e = p; e < K * ACH; e += 128) S.acc[e] = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int e = p; e < K * WD; e += 128) S.mom[e] = 0.f;
            named_sync(1, 128);
        };
        // Move the record centre of every component to this CTA's running estimate of its new
        // mean (x^ units, FP32-representable) and re-express the FP64 statistics exactly:
        //   P' = P - s1 d^T - d s1^T + N d d^T,  s1' = s1 - N d.
        // back: re-express about the starting centre -fp32((mu_k - c) xs) instead.
        auto recentre = [&](bool back) {
            double* sN = reinterpret_cast<double*>(S.rec);
            double* sS1 = sN + WK;
            double* sD = sS1 + WK * WD;
            for (int r = p; r < K * WD; r += 128) {
                const int k = r / WD, a = r % WD;
                const double* blk = part + (int64_t)k * SK;
                const double N = blk[0];
                if (a == 0) sN[k] = N;
                double d = 0.0, s1 = 0.0;
                if (a < D) {
                    s1 = blk[1 + a];
                    const double cur = -(double)S.nmu[k * WD + a];
                    if (back)
                        d = (double)(float)((mv.mu()[k * D + a] - center[a]) * xs) - cur;
                    else if (N > 0.5)
                        d = (double)(float)(cur + s1 / N) - cur;
                }
                sS1[r] = s1;
                sD[r] = d;
            }
            named_sync(1, 128);
            for (int r = p; r < K * WD; r += 128) {
                const int k = r / WD, a = r % WD;
                if (a >= D) continue;
                double* __restrict__ blk = part + (int64_t)k * SK;
                const double N = sN[k], da = sD[r], ga = sS1[r];
                double* __restrict__ s2 = blk + 1 + D + packed_index(a, a, D);
#pragma unroll
                for (int c = 0; c < WD / 4; ++c) {
                    if (4 * c + 3 < a || 4 * c >= D) continue;
                    double v[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (4 * c + j >= a && 4 * c + j < D) v[j] = s2[4 * c + j - a];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int b = 4 * c + j;
                        if (b < a || b >= D) continue;
                        const double db = sD[k * WD + b], sb = sS1[k * WD + b];
                        s2[b - a] = v[j] + fma(N * da, db, -fma(ga, db, da * sb));
                    }
                }
                blk[1 + a] = fma(-N, da, ga);
                if (!back) S.nmu[r] = -(float)(-(double)S.nmu[r] + da);
            }
            named_sync(1, 128);
        };

        for (int64_t jj = 0; jj < J; ++jj) {
            const int64_t tile = tile_of(jj);
            const int64_t i = tile * TM + p;
            const bool valid = i < n;
            if (p == 0 && jj + 1 < J) {  // next tile's planes into L2
                const int64_t r0 = tile_of(jj + 1) * TM;
                const uint32_t bytes = (uint32_t)(min((int64_t)TM, n - r0) * 8 + 15) & ~15u;
                for (int f = 0; f < D; ++f) prefetch_l2(X + (int64_t)f * ld + r0, bytes);
            }
            // ---- x^ = (x - c) xs: FP32 row (registers) + fp16 hi / lo A operands (TMEM)
            uint64_t x2[WD / 2];
            {
                double xv[WD];
#pragma unroll
                for (int f = 0; f < WD; ++f) xv[f] = (valid && f < D) ? __ldg(X + (int64_t)f * ld + i) : 0.0;
                float xf[WD];
#pragma unroll
                for (int f = 0; f < WD; f += 2) {
                    float v0 = 0.f, v1 = 0.f;
                    if (f < D) v0 = F32 ? fmaf(__double2float_rn(xv[f]), xsf, ncxf.v[f]) : (float)fma(xv[f], xs, ncx.v[f]);
                    if (f + 1 < D)
                        v1 = F32 ? fmaf(__double2float_rn(xv[f + 1]), xsf, ncxf.v[f + 1])
                                 : (float)fma(xv[f + 1], xs, ncx.v[f + 1]);
                    if (!valid) v0 = v1 = 0.f;
                    x2[f / 2] = pack2(v0, v1);
                    xf[f] = v0;
                    xf[f + 1] = v1;
                }
                // K-step s: features 13 s .. 13 s + 12 in columns 0-12, ones (hi) / zeros (lo) in 13-15
#pragma unroll
                for (int sidx = 0; sidx < KSMAX; ++sidx) {
                    if (sidx >= KS) break;
                    uint32_t hw[8], lw[8];
#pragma unroll
                    for (int c = 0; c < 16; c += 2) {
                        float a0, a1;
                        if (c + 1 < FKS) {
                            const int f = FKS * sidx + c;
                            a0 = f < WD ? xf[f] : 0.f;
                            a1 = f + 1 < WD ? xf[f + 1] : 0.f;
                        } else if (c < FKS) {  // c = 12: feature 12 of the step, then the first one
                            const int f = FKS * sidx + c;
                            a0 = f < WD ? xf[f] : 0.f;
                            a1 = 1.f;
                        } else {
                            a0 = a1 = 1.f;
                        }
                        const uint32_t h = pack_h2(a0, a1);
                        const float2 hf = __half22float2(u2h(h));
                        hw[c / 2] = h;
                        lw[c / 2] = pack_h2(a0 - hf.x, a1 - hf.y);
                    }
                    tmem_st8(tmem + lq + TAX + 16 * sidx, hw);
                    tmem_st8(tmem + lq + TAX + 16 * sidx + 8, lw);
                }
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                tc_fence_before();
                __syncwarp();
                if (lane == 0) arrive(&S.aready);
            }
            // ---- E: w_k = cst_k - hq_k |U^_k|^2 for every component
            float w[WK];
#pragma unroll
            for (int k = 0; k < WK; ++k) w[k] = -INFINITY;
#pragma unroll
            for (int g = 0; g < WK / CG; ++g) {
                if (g < NG) {
                    const int64_t e = jj * NG + g;
                    const int r = (int)(e & 1);
                    mbar_wait(su32(&S.edone[r]), (uint32_t)((e >> 1) & 1));
                    tc_fence_after();
#pragma unroll
                    for (int h = 0; h < CG; h += 2) {
                        float u0[32], u1[32];
                        tmem_ld32w(tmem + lq + TE + 128 * r + 32 * h, u0);
                        tmem_ld32w(tmem + lq + TE + 128 * r + 32 * (h + 1), u1);
                        tmem_wait_ld();
                        if (h + 2 == CG) {
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) arrive(&S.efree[r]);
                        }
                        uint64_t qa = 0, qb = 0, qc = 0, qd = 0;
#pragma unroll
                        for (int c = 0; c < 32; c += 4) {
                            const uint64_t a0 = pack2(u0[c], u0[c + 1]), a1 = pack2(u0[c + 2], u0[c + 3]);
                            const uint64_t b0 = pack2(u1[c], u1[c + 1]), b1 = pack2(u1[c + 2], u1[c + 3]);
                            ffma2(qa, a0, a0);
                            ffma2(qb, a1, a1);
                            ffma2(qc, b0, b0);
                            ffma2(qd, b1, b1);
                        }
                        float q0, q1, q2, q3;
                        unpack2(add2(qa, qb), q0, q1);
                        unpack2(add2(qc, qd), q2, q3);
                        const int k0 = CG * g + h;
                        w[k0] = S.cst[k0] - S.hq[k0] * (q0 + q1);
                        w[k0 + 1] = S.cst[k0 + 1] - S.hq[k0 + 1] * (q2 + q3);
                    }
                }
            }
            // ---- log-sum-exp, s_k = sqrt(gamma_k)
            float mx = -INFINITY;
#pragma unroll
            for (int k = 0; k < WK; ++k) mx = fmaxf(mx, w[k]);
            float ssum = 0.f;
#pragma unroll
            for (int k = 0; k < WK; ++k) ssum += ex2((w[k] - mx) * 1.4426950408889634f);
            const float ll = mx + lg2(ssum) * 0.6931471805599453f;
            if (valid) ll_acc += (double)ll;
#pragma unroll
            for (int k = 0; k < WK; ++k) w[k] = valid ? ex2((w[k] - ll) * 0.7213475204444817f) : 0.f;  // s_k
            {  // N_k += sum over the warp's events of gamma_k: transpose-reduce, lane l <- component l
                float v[WK];
#pragma unroll
                for (int k = 0; k < WK; ++k) v[k] = w[k] * w[k];
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1) {
                    const bool up = (lane & o) != 0;
#pragma unroll
                    for (int q = 0; q < o; ++q) {
                        const float send = up ? v[q] : v[q + o];
                        const float keep = up ? v[q + o] : v[q];
                        v[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                    }
                }
                nkp += (double)v[0];
            }
            // ---- M: per group, records -> Gram (MMA warp) -> flush of the Gram rows
            auto flush = [&](int64_t m) {  // Gram m (group m % NG of its tile) -> FP32 accumulators
                mbar_wait(su32(&S.mdone), (uint32_t)(m & 1));
                tc_fence_after();
                const int k = CG * (int)(m % NG) + warp;  // row (kl = warp, a = lane)
                if (k < K) {
                    float v[32], f0, f1, m1;
                    tmem_ld32w(tmem + lq + TGR + 32 * warp, v);
                    tmem_ld2(tmem + lq + TGR + 128 + 2 * (warp >> 1), f0, f1);
                    if (NPASS == 2) {  // + R_h^T s_l
                        float e0, e1;
                        tmem_ld2(tmem + lq + TGR + 136 + 2 * (warp >> 1), e0, e1);
                        tmem_wait_ld();
                        m1 = (warp & 1) ? f1 + e1 : f0 + e0;
                    } else {
                        tmem_wait_ld();
                        m1 = (warp & 1) ? f1 : f0;
                    }
                    float4* row = S.acc + k * ACH + row_base(lane);
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        if (c < (lane >> 2)) continue;
                        float4* a4 = row + c;
                        float4 o = *a4;
                        uint64_t lo = add2(pack2(o.x, o.y), pack2(v[4 * c], v[4 * c + 1]));
                        uint64_t hi = add2(pack2(o.z, o.w), pack2(v[4 * c + 2], v[4 * c + 3]));
                        unpack2(lo, o.x, o.y);
                        unpack2(hi, o.z, o.w);
                        *a4 = o;
                    }
                    S.mom[k * WD + lane] += m1;
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) arrive(&S.gfree);
            };
            unsigned char* const rp0 = S.rec + (p >> 3) * 128 + (p & 7) * 16;  // R_h groups, then R_l at RHG
#pragma unroll
            for (int g = 0; g < WK / CG; ++g) {
                if (g >= NG) break;
                const int64_t m = jj * NG + g;
                // NPASS = 2: one records buffer, free once Gram m - 1 completed; NPASS = 1: buffer
                // m & 1 (Gram m - 2 was flushed in the previous group), Gram m - 1 flushed after
                if (NPASS == 2 && g >= 1) flush(m - 1);
                unsigned char* const rp = rp0 + (NPASS == 1 ? (uint32_t)(m & 1) * RHG * RG : 0u);
#pragma unroll
                for (int kl = 0; kl < CG; ++kl) {
                    const float sk = w[CG * g + kl];
                    const uint64_t s2 = pack2(sk, sk);
                    const ulonglong2* nm = reinterpret_cast<const ulonglong2*>(S.nmu + (CG * g + kl) * WD);
                    uint32_t oh[16], ol[16];
#pragma unroll
                    for (int r = 0; r < 16; r += 2) {
                        const ulonglong2 m2 = nm[r / 2];
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const uint64_t rr = mul2(add2(x2[r + h], h ? m2.y : m2.x), s2);
                            float a0, a1;
                            unpack2(rr, a0, a1);
                            oh[r + h] = pack_h2(a0, a1);
                            if (NPASS == 2) {  // R_l = fp16(r - R_h), R_h rounded to nearest
                                const float2 hf = __half22float2(u2h(oh[r + h]));
                                unpack2(sub2(rr, pack2(hf.x, hf.y)), a0, a1);
                                ol[r + h] = pack_h2(a0, a1);
                            }
                        }
                    }
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        *reinterpret_cast<uint4*>(rp + (4 * kl + c) * RG) =
                            make_uint4(oh[4 * c], oh[4 * c + 1], oh[4 * c + 2], oh[4 * c + 3]);
                        if (NPASS == 2)
                            *reinterpret_cast<uint4*>(rp + (RHG + 4 * kl + c) * RG) =
                                make_uint4(ol[4 * c], ol[4 * c + 1], ol[4 * c + 2], ol[4 * c + 3]);
                    }
                }
                {
                    const uint32_t h01 = pack_h2(w[CG * g], w[CG * g + 1]), h23 = pack_h2(w[CG * g + 2], w[CG * g + 3]);
                    *reinterpret_cast<uint4*>(rp + 16 * RG) = make_uint4(h01, h23, 0u, 0u);
                    if (NPASS == 2) {
                        const float2 a = __half22float2(u2h(h01)), b = __half22float2(u2h(h23));
                        *reinterpret_cast<uint4*>(rp + 17 * RG) =
                            make_uint4(pack_h2(w[CG * g] - a.x, w[CG * g + 1] - a.y),
                                       pack_h2(w[CG * g + 2] - b.x, w[CG * g + 3] - b.y), 0u, 0u);
                    }
                }
                proxy_fence();
                if (NPASS == 1 && g >= 1) flush(m - 1);
                __syncwarp();
                if (lane == 0) arrive(&S.mready);
            }
            flush(jj * NG + NG - 1);
            // ---- FP64 window and recentring
            const bool pow2 = ((jj + 1) & jj) == 0;
            if (pow2 || (jj + 1) % FLUSH == 0 || jj + 1 == J) {
                flush64();
                if (pow2 && jj + 1 < J) recentre(false);
            }
        }
        if (J == 0) flush64();
        recentre(true);
        // ---- output: logL, and the statistics scaled to x units (xs^-1, xs^-2: exact)
        {
            const double v = warp_sum(ll_acc);
            if (lane == 0) S.llw[warp] = v;
        }
        named_sync(1, 128);
        const double i1 = 1.0 / xs, i2 = i1 * i1;
        for (int e = p; e < NE; e += 128) {
            const int r = e % SK;
            if (r == 0) continue;
            part[e] *= r <= D ? i1 : i2;
        }
        if (p == 0) part[NE] = ((S.llw[0] + S.llw[1]) + S.llw[2]) + S.llw[3];
    } else if (warp == 4) {
        // ========================================================== group images (TMA)
        if (lane == 0) {
            for (int64_t jj = 0; jj < J; ++jj) {
                for (int g = 0; g < NG; ++g) {
                    const int64_t q = jj * NG + g;
                    const int sl = (int)(q % NSLOT);
                    if (q >= NSLOT) mbar_wait_sleep(su32(&S.wfree[sl]), (uint32_t)(((q - NSLOT) / NSLOT) & 1));
                    mbar_expect_tx(su32(&S.wfull[sl]), WIMG);
                    bulk_g2s(su32(S.w[sl]), wimg + (size_t)g * WIMG, WIMG, su32(&S.wfull[sl]));
                }
            }
        }
    } else {
        // ================================================================ MMA issuer
        if (lane == 0) {
            const uint64_t dh = sdesc(su32(S.rec), 128, RG), dl = sdesc(su32(S.rec) + RHG * RG, 128, RG);
            for (int64_t jj = 0; jj < J; ++jj) {
                mbar_wait_sleep(su32(&S.aready), (uint32_t)(jj & 1));
                for (int g = 0; g < NG; ++g) {
                    const int64_t e = jj * NG + g;
                    const int sl = (int)(e % NSLOT), r = (int)(e & 1);
                    mbar_wait_sleep(su32(&S.wfull[sl]), (uint32_t)((e / NSLOT) & 1));
                    if (e >= 2) mbar_wait_sleep(su32(&S.efree[r]), (uint32_t)(((e - 2) >> 1) & 1));
                    tc_fence_after();
                    const uint32_t base = su32(S.w[sl]);
                    const uint32_t dt = tmem + TE + 128 * r;
                    // the hi x hi products of every K-step first (each adds a centred partial
                    // whitening), then the hi x lo and lo x hi corrections
                    for (int ks = 0; ks < KS; ++ks)
                        mma_f16_ta(dt, tmem + TAX + 16 * ks, sdesc(base + (2 * ks) * WOP, 128, 256), kIdescE,
                                   ks > 0 ? 1u : 0u);
                    for (int ks = 0; ks < KS; ++ks) {
                        const uint64_t bh = sdesc(base + (2 * ks) * WOP, 128, 256);
                        const uint64_t bl = sdesc(base + (2 * ks + 1) * WOP, 128, 256);
                        const uint32_t ah = tmem + TAX + 16 * ks, al = ah + 8;
                        mma_f16_ta(dt, ah, bl, kIdescE, 1u);
                        mma_f16_ta(dt, al, bh, kIdescE, 1u);
                    }
                    commit(&S.edone[r]);
                    commit(&S.wfree[sl]);
                }
                for (int g = 0; g < NG; ++g) {
                    const int64_t m = jj * NG + g;
                    mbar_wait_sleep(su32(&S.mready), (uint32_t)(m & 1));
                    if (m >= 1) mbar_wait_sleep(su32(&S.gfree), (uint32_t)((m - 1) & 1));
                    tc_fence_after();
                    if (NPASS == 1) {
                        const uint64_t dhm = sdesc(su32(S.rec) + (uint32_t)(m & 1) * RHG * RG, 128, RG);
#pragma unroll
                        for (int ks = 0; ks < TM / 16; ++ks)
                            mma_f16(tmem + TGR, dhm + 16 * ks, dhm + 16 * ks, idesc_f16(128, 136, 1), ks > 0 ? 1u : 0u);
                    } else {
                        // the small lo products first: the FP32 accumulator truncates ~1 ulp of its
                        // running sum per dispatch, so the 16 lo dispatches issued after the 8 big
                        // R_h^T R_h ones tripled the Gram's same-sign truncation bias
#pragma unroll
                        for (int ks = 0; ks < TM / 16; ++ks)  // R_l^T [R_h | s_h | s_l] (+ the lo*lo term)
                            mma_f16(tmem + TGR, dl + 16 * ks, dh + 16 * ks, idesc_f16(128, 144, 1), ks > 0 ? 1u : 0u);
#pragma unroll
                        for (int ks = 0; ks < TM / 16; ++ks)  // + R_h^T R_l
                            mma_f16(tmem + TGR, dh + 16 * ks, dl + 16 * ks, idesc_f16(128, 128, 1), 1u);
#pragma unroll
                        for (int ks = 0; ks < TM / 16; ++ks)  // + R_h^T [R_h | s_h | s_l]
                            mma_f16(tmem + TGR, dh + 16 * ks, dh + 16 * ks, idesc_f16(128, 144, 1), 1u);
                    }
                    commit(&S.mdone);
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 5) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// Shapes of the wide tensor-core pass: full covariances with D <= 32, K <= 32 outside k_em_mma's.
bool em_wide_supported(int D, int K) { return D >= 1 && D <= WD && K >= 1 && K <= WK; }

size_t em_wide_workspace_bytes() { return (size_t)(WK / CG) * WIMG + 2 * WK * sizeof(float); }

template <int NPASS, bool F32>
static void launch_wide_t(const double* X, int64_t n, int64_t ld, int D, int K, const double* model,
                          const double* center, double xs, const NegCxW& ncx, const NegCxWF& ncxf,
                          const unsigned char* wimg, const float* consts, double* partial, int grid, cudaStream_t s,
                          float qscale) {
    const size_t smem = sizeof(WSmem) + 128;
    static bool a = false;
    if (!a) {
        cudaFuncSetAttribute(k_em_wide<NPASS, F32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        a = true;
    }
    k_em_wide<NPASS, F32><<<grid, WNT, smem, s>>>(X, n, ld, D, K, model, center, xs, ncx, ncxf, (float)xs, wimg,
                                                   consts, partial, qscale);
}

void launch_em_wide(const double* X, int64_t n, int64_t ld, int D, int K, const double* model, const double* center,
                    const double* center_host, double xs, bool f32conv, int npass, void* workspace, double* partial,
                    int num_sms, int* nblk, cudaStream_t s, LaunchStats& ls) {
    unsigned char* wimg = static_cast<unsigned char*>(workspace);
    float* consts = reinterpret_cast<float*>(wimg + (size_t)(WK / CG) * WIMG);
    const int NG = (K + CG - 1) / CG;
    k_wide_stage<<<NG, 256, 0, s>>>(model, K, D, center, xs, wimg, consts);
    NegCxW ncx{};
    NegCxWF ncxf{};
    for (int j = 0; j < D; ++j) {
        ncx.v[j] = -center_host[j] * xs;
        ncxf.v[j] = (float)ncx.v[j];
    }
    const int64_t ntiles = (n + TM - 1) / TM;
    const int grid = (int)std::min<int64_t>(num_sms, std::max<int64_t>(ntiles, 1));
    *nblk = grid;
    // ES_WIDE_TRUNC (diagnostic): assumed mean truncation per E dispatch in ulps of the result;
    // |U|^2 is scaled up by 2 n_d tau E[ulp(u) / |u|] (E = 0.7213 2^-23 for Benford mantissas)
    const char* tr = getenv("ES_WIDE_TRUNC");
    const double tau = tr ? atof(tr) : 0.0;
    const int KS = (D + FKS - 1) / FKS;
    const float qs = (float)(1.0 + 2.0 * 3 * KS * tau * 0.7213475204444817 * 0x1p-23);
    if (npass == 1 && f32conv)
        launch_wide_t<1, true>(X, n, ld, D, K, model, center, xs, ncx, ncxf, wimg, consts, partial, grid, s, qs);
    else if (npass == 1)
        launch_wide_t<1, false>(X, n, ld, D, K, model, center, xs, ncx, ncxf, wimg, consts, partial, grid, s, qs);
    else if (f32conv)
        launch_wide_t<2, true>(X, n, ld, D, K, model, center, xs, ncx, ncxf, wimg, consts, partial, grid, s, qs);
    else
        launch_wide_t<2, false>(X, n, ld, D, K, model, center, xs, ncx, ncxf, wimg, consts, partial, grid, s, qs);
    ls.launches += 2;
}

}  // namespace es
