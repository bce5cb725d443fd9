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

namespace {

using namespace mma;

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
    uint8_t cev[NWG][4 * (KMAX * 32 + KMAX)];    // compacted candidates per warp (component-major): event
    uint8_t ccomp[NWG][4 * (KMAX * 32 + KMAX)];  //                                                component
    float cst[KMAX], lnf[KMAX], hq[KMAX], tk[KMAX];
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
        const unsigned lt_mask = (1u << lane) - 1u;
        float cst[KMAX], lnf[KMAX], hq[KMAX];
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
            cst[k] = S.cst[k];
            lnf[k] = S.lnf[k];
            hq[k] = S.hq[k];
        }
        const float ldf = (float)o.log_delta;
        double ll_acc = 0.0, nflag = 0.0;
        // convert tile j; returns whether this event left the fp16-safe range of x^ (then
        // every component of the event is refined in FP64: its FP32 densities are not used)
        auto convert = [&](int64_t j) -> bool {
            const int s = (int)(j % XS);
            mbar_wait(su32(&S.xfull[s]), (uint32_t)((j / XS) & 1));
            uint32_t hw[DM / 2], lw[DM / 2];
            float vmax = 0.f;
#pragma unroll
            for (int f = 0; f < DM; f += 2) {
                const float v0 = (float)fma(S.xd[s][f * TM + p], xs, ncx.v[f]);
                const float v1 = (float)fma(S.xd[s][(f + 1) * TM + p], xs, ncx.v[f + 1]);
                vmax = fmaxf(vmax, fmaxf(fabsf(v0), fabsf(v1)));
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
            return !(vmax <= 16384.f);
        };
        bool ovf = w < J ? convert(w) : false, ovf_next = false;
        int64_t jj = 0;
        for (int64_t j = w; j < J; j += NWG, ++jj) {
            const int s = (int)(j % XS);
            const int64_t i = tile_of(j) * TM + p;
            const bool valid = i < n;
            mbar_wait(su32(&S.edone[w]), (uint32_t)(jj & 1));
            tc_fence_after();
            float wk[KMAX], ln[KMAX];
            float m = -INFINITY, bl = -INFINITY;
#pragma unroll
            for (int k = 0; k < KMAX; ++k) {
                float u[16];
                tmem_ld16(tmem + lq + 16 * k, u);
                tmem_wait_ld();
                uint64_t q2 = 0;
#pragma unroll
                for (int r = 0; r < 16; r += 2) {
                    const uint64_t uu = pack2(u[r], u[r + 1]);
                    ffma2(q2, uu, uu);
                }
                float qa, qb;
                unpack2(q2, qa, qb);
                const float hqq = hq[k] * (qa + qb);
                ln[k] = lnf[k] - hqq;
                wk[k] = cst[k] - hqq;
                m = fmaxf(m, wk[k]);
                bl = fmaxf(bl, ln[k]);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) arrive(&S.efree);
            // E(j) has consumed this WG's A operand: stage the next tile now
            if (j + NWG < J) ovf_next = convert(j + NWG);
            // candidates needing FP64: responsibility above 1e-6 (FP32 error then moves ll by
            // < 1e-6 * 1e-3 relative), or within FP32 rounding of either argmax / of log delta
            unsigned cand = 0;
#pragma unroll
            for (int k = 0; k < KMAX; ++k) {
                const float tol = 1e-3f * (1.f + fabsf(wk[k]));
                bool c;
                if (refine_all)
                    c = wk[k] >= m - 13.9f || ln[k] >= bl - tol;
                else
                    c = wk[k] >= m - tol || ln[k] >= bl - tol ||
                        (ln[k] == bl && fabsf(bl - ldf) <= 1e-3f * (1.f + fabsf(ldf)));
                if (valid && k < K && (c || ovf)) cand |= 1u << k;
            }
            // component-major compaction inside the warp (fixed order: component, lane); each
            // component segment padded to an even length (two events of one component per item).
            // Warp-local: no warpgroup barrier, each warp refines its own 32 events.
            uint8_t* cev = S.cev[w] + q * (KMAX * 32 + KMAX);
            uint8_t* ccomp = S.ccomp[w] + q * (KMAX * 32 + KMAX);
            int nc = 0;
#pragma unroll
            for (int k = 0; k < KMAX; ++k) {
                const unsigned kb = __ballot_sync(0xffffffffu, (cand >> k) & 1u);
                if ((cand >> k) & 1u) {
                    const int pos = nc + __popc(kb & lt_mask);
                    cev[pos] = (uint8_t)p;
                    ccomp[pos] = (uint8_t)k;
                }
                nc += __popc(kb);
                if (nc & 1) {
                    if (lane == 0) {
                        cev[nc] = 0xFFu;
                        ccomp[nc] = (uint8_t)k;
                    }
                    ++nc;
                }
            }
            __syncwarp();
            // FP64 refinement, two events of one component per lane (each W row load serves both)
            double* lnv = S.lnv[w];
            for (int pidx = 2 * lane; pidx < nc; pidx += 64) {
                const int k = ccomp[pidx];
                const int e0 = cev[pidx], e1r = cev[pidx + 1];
                const int e1 = e1r == 0xFF ? e0 : e1r;
                const double* WTk = S.W64 + k * W64S;  // column f of W_k at WTk[f * DM + r]
                const double* mk = S.mu64 + k * (DM + 2);
                // z = W_k (x - mu_k) as a sum of columns: 16 independent accumulators per event
                double z0[DM], z1[DM];
#pragma unroll
                for (int r = 0; r < DM; ++r) z0[r] = z1[r] = 0.0;
#pragma unroll
                for (int f = 0; f < DM; ++f) {
                    const double df0 = S.xd[s][f * TM + e0] - mk[f];
                    const double df1 = S.xd[s][f * TM + e1] - mk[f];
#pragma unroll
                    for (int r = f & ~1; r < DM; r += 2) {  // W is lower triangular: rows r >= f
                        const double2 wv = *reinterpret_cast<const double2*>(WTk + f * DM + r);
                        z0[r] = fma(wv.x, df0, z0[r]);
                        z1[r] = fma(wv.x, df1, z1[r]);
                        z0[r + 1] = fma(wv.y, df0, z0[r + 1]);
                        z1[r + 1] = fma(wv.y, df1, z1[r + 1]);
                    }
                }
                double q0 = 0.0, q1 = 0.0;
#pragma unroll
                for (int r = 0; r < DM; ++r) {
                    q0 = fma(z0[r], z0[r], q0);
                    q1 = fma(z1[r], z1[r], q1);
                }
                lnv[k * TM + e0] = S.ln64[k] - 0.5 * q0;
                if (e1r != 0xFF) lnv[k * TM + e1] = S.ln64[k] - 0.5 * q1;
            }
            __syncwarp();
            if (lane == 0) arrive(&S.xfree[s]);  // this warp no longer reads the FP64 tile
            double mm = -INFINITY, bb = -INFINITY;
            int am = 0, ab = 0;
            double w64[KMAX];
#pragma unroll
            for (int k = 0; k < KMAX; ++k) {
                const double l = ((cand >> k) & 1u) ? lnv[k * TM + p] : (double)ln[k];
                w64[k] = S.lp64[k] + l;
                if (k >= K) continue;
                if (w64[k] > mm) {
                    mm = w64[k];
                    am = k;
                }
                if (l > bb) {
                    bb = l;
                    ab = k;
                }
            }
            // log-sum-exp about the FP64 maximum: the max term is exactly 1, the others are
            // summed with FP32 exp (relative 1e-7 of a sum >= 1 -> ll error < 2e-7 absolute)
            float ss = 0.f;
#pragma unroll
            for (int k = 0; k < KMAX; ++k)
                if (k < K) ss += __expf((float)(w64[k] - mm));
            const double lld = mm + log((double)ss);
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

bool score_mma_enabled(int D, int K, const ScoreOut& o) {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("ES_SCORE_KERNEL");
        v = (!e || e[0] == 'm') ? 1 : 0;  // default; "tc" / "simt" select the older kernels
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
        refine_all = (e && e[0] == 'm') ? 0 : 1;  // ES_SCORE_REFINE=min: decisive components only
    }
    k_score_mma<<<grid, NTHR, smem, s>>>(*xmap, n, D, K, model, center, xs, ncx, o, blocksum, refine_all);
    ++ls.launches;
}

}  // namespace es
