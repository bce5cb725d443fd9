// es_score_mma.cu — scoring pass (score_samples / predict / detect) on the fused
// pipeline of es_em_mma.cu.
//
// Per 128-event tile (one CTA per SM, persistent), 10 warps:
//   TMA warp      2-D tensor copy of the FP64 tile into a 4-stage ring; a stage is
//                 released only after the FP64 refinement of its tile.
//   2 epilogue warpgroups (alternate tiles), thread = event = TMEM lane:
//                 convert x^ = (x - c) xs -> fp16 hi/lo E-step A operand (tcgen05.st);
//                 FP32 log densities of all K from U = W' x^ + b' (TMEM); candidates
//                 needing FP64 (responsibility above 1e-6, or within FP32 rounding of
//                 either argmax), compacted component-major inside the warpgroup;
//                 FP64 recomputation of the candidates from the FP64 tile (two events
//                 of one component per thread and W-row load); ll (log-sum-exp about
//                 the FP64 maximum), predict, best_k, best_logdens, flag.
//   MMA warp      E-step dispatches (4 x kind::f16 M128 N128 K16, A from TMEM) as
//                 soon as a warpgroup's operand is staged and the accumulator is free.
// The warpgroups synchronise on named barriers only, so one refines its tile while
// the other's E-step and conversion run.
#include <cmath>
#include <cstdlib>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include "es_kernels.h"
#include "es_mma.cuh"

namespace es {

#ifdef ES_SCORE_COUNT
__device__ unsigned long long g_score_pairs;
#endif

namespace {

using namespace mma;

// MUFU square root (relative error ~2^-22): feeds only the error bounds
__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

#ifndef ES_SCORE_NWG  // 3: 7.3 ms per 2^26-event pass; 2 (168 registers): 8.0 ms
#define ES_SCORE_NWG 3
#endif
constexpr int NWG = ES_SCORE_NWG;  // epilogue warpgroups (tiles j = w mod NWG)
constexpr int NTHR = 128 * NWG + 64;  // + TMA warp + MMA warp
constexpr int WTMA = 4 * NWG, WMMA = 4 * NWG + 1;
constexpr int XS = 2 * NWG;        // FP64 tile stages: each WG holds its tile and the next one
constexpr int W64S = DM * DM + 2;  // FP64 W^T stride (bank skew between components)
constexpr int TA0 = 128, TONE = 128 + 16 * NWG;  // TMEM: E accumulator [0,128), A operands, ones

struct SmemS {
    double xd[XS][DM * TM];                  // 64 KB  FP64 tiles (planar, TMA destination)
    double lnv[NWG][KMAX * TM];              // FP64 log densities of the refined pairs
    alignas(16) double W64[KMAX * W64S];
    double mu64[KMAX * (DM + 2)];
    double ln64[KMAX], lp64[KMAX];
    double c[DM];
    double wred[4 * NWG][2];
    unsigned char bw[2][OPB];
    unsigned char bb[OPB];
    uint16_t plist[NWG][4 * 256];                // extra (event << 4 | component) pairs per warp
    float cst[KMAX], lnf[KMAX], hq[KMAX], tk[KMAX];
    float ec1[KMAX], ec0[KMAX];  // error-bound constants: eps1 ||B_k||_F, eps2 ||b^_k||_2 (U / t_k units)
    float lpf[KMAX];             // log pi_k (FP32)
    uint64_t xfull[XS], xfree[XS], aeready[NWG], edone[NWG], efree;
    uint32_t tmem;
};

}  // namespace

__global__ void __launch_bounds__(NTHR, 1) k_score_mma(const __grid_constant__ CUtensorMap xmap, int64_t n, int D,
                                                        int K, const double* __restrict__ model,
                                                        const double* __restrict__ center, double xs,
                                                        const __grid_constant__ NegCx ncx, ScoreOut o,
                                                        double* __restrict__ blocksum, int refine_all) {
    extern __shared__ __align__(128) unsigned char smraw[];
    SmemS& S = *reinterpret_cast<SmemS*>(smraw + ((128u - (su32(smraw) & 127u)) & 127u));
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    ModelView mv{K, D, const_cast<double*>(model)};
    const int64_t ntiles = (n + TM - 1) / TM;
    const int64_t J = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    // ------------------------------------------------------------------ staging
    for (int j = t; j < DM; j += NTHR) S.c[j] = j < D ? center[j] : 0.0;
    for (int e = t; e < XS * DM * TM; e += NTHR) (&S.xd[0][0])[e] = 0.0;  // planes >= D stay zero
    stage_estep(mv, K, D, center, S.c, xs, S.bw[0], S.bw[1], S.bb, S.cst, S.lnf, S.hq, S.tk, t, NTHR);
    __syncthreads();
    if (t < KMAX) {  // error-bound constants of the 3 x fp16 whitening (see the candidate selection)
        double nB = 0.0, nb = 0.0;
        if (t < K) {
            const double* W = mv.W() + (int64_t)t * D * D;
            const double it = 1.0 / (double)S.tk[t];
            for (int a = 0; a < D; ++a) {
                double b = 0.0;
                for (int f = 0; f <= a; ++f) {
                    const double w = W[a * D + f] / xs * it;
                    nB += w * w;
                    b = fma(W[a * D + f], mv.mu()[t * D + f] - S.c[f], b);
                }
                nb += (b * it) * (b * it);
            }
        }
        S.ec1[t] = (float)(0x1p-19 * sqrt(nB));
        S.ec0[t] = (float)(0x1p-22 * sqrt(nb));
        S.lpf[t] = t < K ? (float)mv.logpi()[t] : 0.f;
    }
    for (int e = t; e < KMAX * DM * DM; e += NTHR) {  // transposed: WT[k][f][r] = W_k[r][f]
        const int k = e / (DM * DM), fr = e % (DM * DM), f = fr / DM, r = fr % DM;
        S.W64[k * W64S + fr] = (k < K && r < D && f < D) ? mv.W()[(int64_t)k * D * D + r * D + f] : 0.0;
    }
    for (int e = t; e < KMAX * DM; e += NTHR) {
        const int k = e / DM, j = e % DM;
        S.mu64[k * (DM + 2) + j] = (k < K && j < D) ? mv.mu()[k * D + j] : 0.0;
    }
    for (int k = t; k < KMAX; k += NTHR) {
        S.ln64[k] = k < K ? mv.lognorm()[k] : 0.0;
        S.lp64[k] = k < K ? mv.logpi()[k] : -INFINITY;
    }
    if (warp == WMMA) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&S.tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        for (int i = 0; i < XS; ++i) {
            mbar_init(&S.xfull[i], 1);
            mbar_init(&S.xfree[i], 4);  // one arrival per warp of the warpgroup that refines the tile
        }
        for (int i = 0; i < NWG; ++i) {
            mbar_init(&S.aeready[i], 4);
            mbar_init(&S.edone[i], 1);
        }
        mbar_init(&S.efree, 4);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    proxy_fence();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = S.tmem;
    auto tile_of = [&](int64_t j) { return (int64_t)blockIdx.x + j * gridDim.x; };
    if (warp < 4) {  // ones in K columns 0-2 of every row: the bias dispatch's A operand
        const uint32_t one[8] = {0x3C003C00u, 0x00003C00u, 0u, 0u, 0u, 0u, 0u, 0u};  // K columns 0, 1, 2
        tmem_st8(tmem + ((uint32_t)(32 * warp) << 16) + TONE, one);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    if (warp < 4 * NWG) {
        // ====================================================== epilogue warpgroups
        const int w = warp >> 2;
        const int p = t & 127;
        const int q = warp & 3;
        const uint32_t lq = (uint32_t)(32 * q) << 16;
        // per-component constants are read from shared memory (broadcast) where used: kept in
        // registers they would be live across the FP64 refinement (register spills)
        const float* lnf = S.lnf;
        const float* hq = S.hq;
        float xnorm = 0.f, xnorm_next = 0.f;  // ||x^||_2 of this thread's event (error bound)
        double ll_acc = 0.0, nflag = 0.0;
        // convert tile j; returns whether this event left the fp16-safe range of x^ (then
        // every component of the event is refined in FP64: its FP32 densities are not used)
        auto convert = [&](int64_t j, float& xn) -> bool {
            const int s = (int)(j % XS);
            mbar_wait(su32(&S.xfull[s]), (uint32_t)((j / XS) & 1));
            uint32_t hw[DM / 2], lw[DM / 2];
            float vmax = 0.f, n2 = 0.f;
#pragma unroll
            for (int f = 0; f < DM; f += 2) {
                const float v0 = (float)fma(S.xd[s][f * TM + p], xs, ncx.v[f]);
                const float v1 = (float)fma(S.xd[s][(f + 1) * TM + p], xs, ncx.v[f + 1]);
                vmax = fmaxf(vmax, fmaxf(fabsf(v0), fabsf(v1)));
                n2 = fmaf(v0, v0, fmaf(v1, v1, n2));
                const uint32_t h = pack_h2(v0, v1);
                const float2 hf = __half22float2(u2h(h));
                hw[f / 2] = h;
                lw[f / 2] = pack_h2(v0 - hf.x, v1 - hf.y);
            }
            tmem_st8(tmem + lq + TA0 + 16 * w, hw);
            tmem_st8(tmem + lq + TA0 + 16 * w + 8, lw);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            tc_fence_before();
            __syncwarp();
            if (lane == 0) arrive(&S.aeready[w]);  // per warp: its 32 events are staged
            xn = sqrt_approx(n2);
            return !(vmax <= 16384.f);
        };
        bool ovf = w < J ? convert(w, xnorm) : false, ovf_next = false;
        // weighted quantities (ll, predict, mixture flags) are needed only when requested:
        // detect (best component, its density, the flag) refines the unweighted argmax alone
        const bool need_w = o.ll != nullptr || o.predict != nullptr || o.mode == 1 || o.sum_ll;
        // FP64 log N(x_e | k) of an event of this warpgroup's tile (planar FP64 tile, stage s):
        // z = W_k (x - mu_k) as a sum of columns (16 independent accumulators)
        auto refine = [&](int s, int e, int k) -> double {
            const double* WTk = S.W64 + k * W64S;  // column f of W_k at WTk[f * DM + r]
            const double* mk = S.mu64 + k * (DM + 2);
            double z[DM];
#pragma unroll
            for (int r = 0; r < DM; ++r) z[r] = 0.0;
#pragma unroll
            for (int f = 0; f < DM; ++f) {
                const double df = S.xd[s][f * TM + e] - mk[f];
                // W is lower triangular: rows r >= f.  Odd f: the diagonal entry alone (8 B), then
                // aligned pairs (the zero above the diagonal is not loaded: these loads are the
                // pass's binding shared-memory traffic)
                if (f & 1) z[f] = fma(WTk[f * DM + f], df, z[f]);
#pragma unroll
                for (int r = (f & 1) ? f + 1 : f; r < DM; r += 2) {
                    const double2 wv = *reinterpret_cast<const double2*>(WTk + f * DM + r);
                    z[r] = fma(wv.x, df, z[r]);
                    z[r + 1] = fma(wv.y, df, z[r + 1]);
                }
            }
            double q0 = 0.0, q1 = 0.0;
#pragma unroll
            for (int r = 0; r < DM; r += 2) {
                q0 = fma(z[r], z[r], q0);
                q1 = fma(z[r + 1], z[r + 1], q1);
            }
            return S.ln64[k] - 0.5 * (q0 + q1);
        };
        int64_t jj = 0;
        for (int64_t j = w; j < J; j += NWG, ++jj) {
            const int s = (int)(j % XS);
            const int64_t i = tile_of(j) * TM + p;
            const bool valid = i < n;
            mbar_wait(su32(&S.edone[w]), (uint32_t)(jj & 1));
            tc_fence_after();
            // FP32 densities of all K and a per-(event, component) bound dw on their error.
            // U^ = U / t_k from 4 kind::f16 dispatches: b^ (fp32, exact in the accumulator), then
            // x_hi B_hi, x_hi B_lo, x_lo B_hi with x^ = x_hi + x_lo, B = B_hi + B_lo (fp16).  Per
            // entry a:  |U^_a - U_a| <= eps1' sum_f |B_af| |x^_f| + eps2' |b^_a| + eps3 |U^_a|,
            // eps1' <= 2^-24 (x^ rounding) + 3 2^-22 (split residuals, dropped lo*lo) + 2^-23
            // (accumulator truncation against the products), eps2' <= 2^-24 (fp32(b^)) + 2^-23
            // (truncation against the accumulator input), eps3 = 3 2^-23 (truncation of the three
            // later dispatches, measured ~1 ulp of the running sum, scripts/umma_probe.cu); doubled
            // here: eps1 = 2^-19, eps2 = 2^-22, eps3 = 2^-21.  Cauchy-Schwarz over a gives
            //   ||dU|| <= e = eps1 ||B_k||_F ||x^|| + eps2 ||b^_k|| + eps3 ||U^||,
            //   |q^ - q| <= 2 ||U^|| e + e^2 + 2^-20 q^ (FP32 sum of 16 squares),
            //   |ln^ - ln| <= hq (|q^ - q|) + 2^-21 (|ln^| + |lognorm| + 1)   (hq = t_k^2 / 2),
            // and for w = ln + log pi_k (FP32 add) 2^-20 |log pi_k| more.
            // ln_k (FP32, unweighted) and its bound dw_k; the weighted w_k = ln_k + log pi_k is
            // formed only when weighted outputs are requested (bound + 2^-20 |log pi_k|)
            float ln[KMAX], dw[KMAX];
            float bl = -INFINITY;
            int kb = 0;
#pragma unroll
            for (int k0 = 0; k0 < KMAX; k0 += 2) {  // two components per TMEM wait
                float u[2][16];
                tmem_ld16(tmem + lq + 16 * k0, u[0]);
                tmem_ld16(tmem + lq + 16 * (k0 + 1), u[1]);
                tmem_wait_ld();
                if (k0 + 2 == KMAX) {  // the accumulator is free for the next E-step
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) arrive(&S.efree);
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int k = k0 + h;
                    uint64_t qa2 = 0, qb2 = 0;  // two independent FFMA2 chains
#pragma unroll
                    for (int r = 0; r < 16; r += 4) {
                        const uint64_t ua = pack2(u[h][r], u[h][r + 1]), ub = pack2(u[h][r + 2], u[h][r + 3]);
                        ffma2(qa2, ua, ua);
                        ffma2(qb2, ub, ub);
                    }
                    float a0, a1, b0, b1;
                    unpack2(qa2, a0, a1);
                    unpack2(qb2, b0, b1);
                    const float q = (a0 + a1) + (b0 + b1);
                    const float lf = lnf[k];
                    ln[k] = fmaf(-hq[k], q, lf);
                    const float rr = sqrt_approx(q);
                    const float e = fmaf(S.ec1[k], xnorm, fmaf(0x1p-21f, rr, S.ec0[k]));
                    const float dq = fmaf(rr, fmaf(2.f, e, 0x1p-20f * rr), e * e);
                    dw[k] = fmaf(hq[k], dq, 0x1p-21f * (fabsf(ln[k]) + fabsf(lf) + 1.f));
                    if (k < K && ln[k] > bl) {  // ties -> lowest k
                        bl = ln[k];
                        kb = k;
                    }
                }
            }
            // E(j) has consumed this WG's A operand: stage the next tile now
            if (j + NWG < J) ovf_next = convert(j + NWG, xnorm_next);
            // FP64 recomputation: the unweighted argmax kb (best_k, best_logdens, the flag) by
            // every thread for its own event; as "extra" pairs every component whose bound
            // interval reaches kb's, and, when weighted outputs are requested, the weighted
            // argmax, its contenders and every component with gamma_k dw_k > tau / 8 (the
            // others enter ll = LSE_k w_k with their FP32 value: ll error <= tau + the FP32 LSE
            // rounding).  ovf: every component.
            const float db = dw[kb];
            unsigned extra = 0;
#pragma unroll
            for (int k = 0; k < KMAX; ++k)
                if (ln[k] + dw[k] >= bl - db) extra |= 1u << k;
            float wk[KMAX];  // weighted FP32 densities (need_w only)
            float m = -INFINITY;
            int km = 0;
            if (need_w) {
#pragma unroll
                for (int k = 0; k < KMAX; ++k) {
                    wk[k] = ln[k] + S.lpf[k];
                    dw[k] = fmaf(0x1p-20f, fabsf(S.lpf[k]), dw[k]);
                    if (k < K && wk[k] > m) {
                        m = wk[k];
                        km = k;
                    }
                }
                const float tau8 = 2.5e-8f * fmaxf(1.f, fabsf(m) - 2.1f);
                const float dm = dw[km];
#pragma unroll
                for (int k = 0; k < KMAX; ++k) {
                    bool c;
                    if (refine_all == 1)  // ES_SCORE_REFINE=all: every component with gamma > 1e-6
                        c = wk[k] >= m - 13.9f;
                    else
                        c = k == km || wk[k] + dw[k] >= m - dm ||
                            ex2((wk[k] - m) * 1.4426950408889634f) * dw[k] > tau8;
                    if (c) extra |= 1u << k;
                }
            }
            extra = (ovf ? 0xFFu : extra) & ~(1u << kb) & ((1u << K) - 1u);
            if (!valid || refine_all == 3) extra = 0;  // refine_all 3: diagnostics, no FP64 pass at all
#ifdef ES_SCORE_COUNT
            if (valid) atomicAdd(&g_score_pairs, (unsigned long long)(1 + __popc(extra)));
#endif
#ifdef ES_SCORE_KB0  // diagnostic (wrong answers): every lane recomputes component 0, i.e. W loads all broadcast
            const double lp = (valid && refine_all != 3) ? refine(s, p, 0) : (double)ln[kb];
#else
            const double lp = (valid && refine_all != 3) ? refine(s, p, kb) : (double)ln[kb];
#endif
            // extra pairs: compacted per warp (lane order, then component), one pair per lane
            double* lnv = S.lnv[w];
            const unsigned any = __ballot_sync(0xffffffffu, extra != 0);
            if (any) {
                const int cnt = __popc(extra);
                int off = cnt;  // inclusive prefix over lanes
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, off, d);
                    if (lane >= d) off += v;
                }
                const int tot = __shfl_sync(0xffffffffu, off, 31);
                off -= cnt;
                uint16_t* lst = S.plist[w] + q * 256;
                for (unsigned b = extra; b; b &= b - 1) lst[off++] = (uint16_t)((p << 4) | (__ffs(b) - 1));
                __syncwarp();
                for (int pi = lane; pi < tot; pi += 32) {
                    const int pe = lst[pi];
                    lnv[(pe & 15) * TM + (pe >> 4)] = refine(s, pe >> 4, pe & 15);
                }
                __syncwarp();
            }
            if (lane == 0) arrive(&S.xfree[s]);  // this warp no longer reads the FP64 tile
            // best component (ties -> lowest k) among the refined ones; non-refined components
            // lie below kb's bound interval
            double bb = lp;
            int ab = kb;
            for (unsigned b = extra; b; b &= b - 1) {
                const int k = __ffs(b) - 1;
                const double l = lnv[k * TM + p];
                if (l > bb || (l == bb && k < ab)) {
                    bb = l;
                    ab = k;
                }
            }
            double lld = 0.0;
            int am = 0;
            if (need_w) {
                double mm = -INFINITY;
                double w64[KMAX];
#pragma unroll
                for (int k = 0; k < KMAX; ++k) {
                    double l;
                    if (k == kb)
                        l = lp;
                    else if ((extra >> k) & 1u)
                        l = lnv[k * TM + p];
                    else
                        l = (double)ln[k];
                    w64[k] = S.lp64[k] + l;
                    if (k < K && w64[k] > mm) {
                        mm = w64[k];
                        am = k;
                    }
                }
                // log-sum-exp about the FP64 maximum: the max term is exactly 1, the others are
                // ex2.approx terms (relative error ~2^-22.5 each of a sum in [1, K]); logf is
                // correctly rounded to 1 ulp of a result in [0, log K]: ll error < 4e-7 absolute
                float ss = 0.f;
#pragma unroll
                for (int k = 0; k < KMAX; ++k)
                    if (k < K) ss += ex2((float)(w64[k] - mm) * 1.4426950408889634f);
                lld = mm + (double)logf(ss);
            }
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
            ovf = ovf_next;
            xnorm = xnorm_next;
        }
        // per-CTA [sum ll, flag count], fixed-order reduction over the 8 warps
        const double a1 = warp_sum(ll_acc), a2 = warp_sum(nflag);
        if (lane == 0) {
            S.wred[warp][0] = a1;
            S.wred[warp][1] = a2;
        }
        named_sync(1 + 2 * NWG, 128 * NWG);
        if (t == 0) {
            double s1 = 0.0, s2 = 0.0;
            for (int i = 0; i < 4 * NWG; ++i) {
                s1 += S.wred[i][0];
                s2 += S.wred[i][1];
            }
            blocksum[2 * blockIdx.x] = s1;
            blocksum[2 * blockIdx.x + 1] = s2;
        }
    } else if (warp == WTMA) {
        // ========================================================== TMA producer
        if (lane == 0) {
            for (int64_t j = 0; j < J; ++j) {
                const int s = (int)(j % XS);
                if (j >= XS) mbar_wait_sleep(su32(&S.xfree[s]), (uint32_t)(((j - XS) / XS) & 1));
                mbar_expect_tx(su32(&S.xfull[s]), (uint32_t)(D * TM * 8));
                tma_load_2d(su32(&S.xd[s][0]), &xmap, (int)(tile_of(j) * TM), 0, su32(&S.xfull[s]));
            }
        }
    } else {
        // ========================================================== MMA issuer
        if (lane == 0) {
            const uint64_t dbh = sdesc(su32(S.bw[0]), 128, 256), dbl = sdesc(su32(S.bw[1]), 128, 256);
            const uint64_t dbb = sdesc(su32(S.bb), 128, 256);
            for (int64_t je = 0; je < J; ++je) {
                const int w = (int)(je % NWG);
                mbar_wait_sleep(su32(&S.aeready[w]), (uint32_t)((je / NWG) & 1));
                if (je >= 1) mbar_wait_sleep(su32(&S.efree), (uint32_t)((je - 1) & 1));
                tc_fence_after();
                const uint32_t tah = tmem + TA0 + 16 * w, tal = tah + 8;
                mma_f16_ta(tmem, tmem + TONE, dbb, kIdescE, 0u);  // fp32(b') exactly, first
                mma_f16_ta(tmem, tah, dbh, kIdescE, 1u);
                mma_f16_ta(tmem, tah, dbl, kIdescE, 1u);
                mma_f16_ta(tmem, tal, dbh, kIdescE, 1u);
                commit(&S.edone[w]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == WMMA) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

// ES_SCORE_KERNEL=fp64 scores on the strict FP64 kernel instead.
bool score_mma_enabled(int D, int K, const ScoreOut& o) {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("ES_SCORE_KERNEL");
        v = (e && e[0] == 'f') ? 0 : 1;
    }
    return v == 1 && D <= DM && K <= KMAX && !o.gamma && !o.lnk;
}

void launch_score_mma(const CUtensorMap* xmap, int64_t n, int D, int K, const double* model, const double* center,
                      const double* center_host, double xs, const ScoreOut& o, double* blocksum, int num_sms,
                      int* nblk, cudaStream_t s, LaunchStats& ls) {
    const int64_t ntiles = (n + TM - 1) / TM;
    const int grid = (int)std::min<int64_t>(num_sms, std::max<int64_t>(ntiles, 1));
    *nblk = grid;
    NegCx ncx{};
    for (int j = 0; j < D && j < DM; ++j) ncx.v[j] = -center_host[j] * xs;
    const size_t smem = sizeof(SmemS) + 128;
    static bool a = false;
    if (!a) {
        cudaFuncSetAttribute(k_score_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        a = true;
    }
    static int refine_all = -1;
    if (refine_all < 0) {
        const char* e = getenv("ES_SCORE_REFINE");
        // ES_SCORE_REFINE=all: every component with gamma > 1e-6; =argmax / =none: diagnostics
        refine_all = !e ? 0 : e[0] == 'a' && e[1] == 'l' ? 1 : e[0] == 'a' ? 2 : e[0] == 'n' ? 3 : 0;
    }
    k_score_mma<<<grid, NTHR, smem, s>>>(*xmap, n, D, K, model, center, xs, ncx, o, blocksum, refine_all);
    ++ls.launches;
}

}  // namespace es

#ifdef ES_SCORE_COUNT
extern "C" unsigned long long es_debug_score_pairs(void) {
    unsigned long long v = 0;
    cudaMemcpyFromSymbol(&v, es::g_score_pairs, sizeof(v));
    unsigned long long z = 0;
    cudaMemcpyToSymbol(es::g_score_pairs, &z, sizeof(z));
    return v;
}
#endif
