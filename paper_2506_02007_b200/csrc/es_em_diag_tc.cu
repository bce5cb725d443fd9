// es_em_diag_tc.cu — fused EM pass for DIAGONAL covariances with the E-step quadratic form and
// the M-step moments on the 5th-gen tensor cores (BASELINE config c3: K = 16, D = 16; an
// extension, the reference has no diagonal variant).  Default diagonal pass when
// every component holds >= kOnePassMinNk events (as k_em_diag_mixed, which it replaces there).
//
// A diagonal Gaussian's log density is linear in the per-event statistics a = (x^2, x, 1):
//   w_k = log pi_k + lognorm_k - 1/2 sum_f p_kf (x_f - mu_kf)^2
//       = sum_f [-1/2 p_kf x_f^2 + p_kf mu_kf x_f] + (log pi_k + lognorm_k - 1/2 sum_f p_kf mu_kf^2),
// and the M-step needs sum_n gamma_nk a_n.  So one fp16 record of a per event serves as
//   E-step A operand (K-major: rows = events, K = statistics)  ->  w = A Theta   (N = 16 components)
//   M-step A operand (MN-major: M = statistics, K = events)    ->  S = A^T Gamma (N = 16 components)
// — the same shared-memory bytes read in the two orientations (a core matrix is 8 events x 8
// statistics in both).  The SIMT work per event is the record (x^ = (x - c) xs, its squares,
// fp16 hi + lo splits), one 16-column TMEM load, the log-sum-exp and the fp16 gamma record.
//
// Per 128-event tile (one persistent CTA per SM): TMA warp (FP64 tile ring), E-issuer warp,
// M-issuer warp, NWG epilogue warpgroups taking tiles round robin (thread = event = TMEM lane).
//
// Record (per event, 6 chunks of 16 fp16 statistics; group g holds features 7g .. 7g + 6):
//   chunk 2g     (hi): hi(x^_f^2) | hi(x^_f) | 1 | 0        slots 0-6 | 7-13 | 14 | 15
//   chunk 2g + 1 (lo): lo(x^_f^2) | lo(x^_f) | 0 | 0
// E-step per group: hi x [Theta_hi | Theta_lo] (M128 N32 K16) and lo x Theta_hi (M128 N16 K16):
// 6 dispatches (each tcgen05.mma costs ~60-90 cycles of the in-order tensor pipe however small),
// Theta = coefficients / t_k (t_k a power of two: largest |entry| in (2^12, 2^13]), the group's
// constant -1/2 sum_{f in g} p mu^2 (+ log pi + lognorm for g = 0) in its '1' slot, so every
// running sum of the FP32 accumulator (truncated ~1 ulp per dispatch, scripts/umma_probe.cu) is
// a partial log density (of the size of w) rather than of the size of the separate terms.
// M-step per 16-event K-step: records^T [2^10 gamma hi | lo] (M128 N32 K16), rows = statistics, into
// NACC = 2 TMEM accumulators used round robin (fewer same-sign truncations per accumulator: at the
// c3 config itself the covariance margin is 0.23 with two, 0.86 with one, for ~13% of pass time), read by
// thread = statistic row after every tile and accumulated in compensated FP32 pairs; the hi and lo
// rows of x^2 and x^ and the '1' row give the moments to ~2^-22 per event (a single fp16 rounding
// of x^2 left a 2^-12 / sqrt(N_k) noise that dominated the covariance error); gamma is split
// hi + lo too (its values cluster at 1, where one rounding is biased).  log pi_k + lognorm_k is
// added in FP32 after the E-step (ES_DTC_CST; in Theta it sets the size of the running sums).
// Output: raw moments about c in x^ units re-expressed exactly in FP64 about the model's means
// (finalize mode 2).
#include <cmath>
#include <cstdlib>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include "es_kernels.h"
#include "es_mma.cuh"

#ifndef ES_DTC_NACC
#define ES_DTC_NACC 2
#endif
#ifndef ES_DTC_NWG  // epilogue warpgroups
#define ES_DTC_NWG 3
#endif
#ifndef ES_DTC_CST  // 1: log pi_k + lognorm_k added in FP32 after the E-step instead of in Theta
#define ES_DTC_CST 1
#endif

namespace es {

namespace {

using namespace mma;

constexpr int DG = 16;   // features (padded)
constexpr int KC = 16;   // components (padded)
constexpr int GF = 7;    // features per record group
constexpr int NG = 3;    // record groups (7 + 7 + 2 features)
constexpr int SLOT1 = 14;
constexpr int NACC = ES_DTC_NACC;                // M-step TMEM accumulators (K-steps round robin)
constexpr uint32_t SGB = (TM / 8) * 128;         // 8 statistics x 128 events: 2 KB
constexpr uint32_t RECB = 4 * NG * SGB;          // 6 chunks x 2 slot groups: 24 KB
constexpr uint32_t GRB = 2 * (KC / 8) * SGB;     // gamma record (hi | lo): 8 KB
constexpr float GSCALE = 1024.f;                 // gamma records hold 2^10 gamma (normal fp16 range)
constexpr int NWG_DTC = ES_DTC_NWG;
constexpr int nthr_dtc() { return 128 * NWG_DTC + 96; }
// FP64 tile stages: a multiple of NWG, so that a stage's previous tile was converted by the same
// warpgroup (a converter two mbarrier phases ahead of its stage would pass the parity wait)
constexpr int XSD = NWG_DTC >= 3 ? NWG_DTC : 4;

struct SmemDT {
    double xd[XSD][DG * TM];                     // 64 KB  FP64 tiles (planar, TMA destination)
    unsigned char rec[NWG_DTC][2][RECB];         // 96 KB  statistic records (double-buffered per WG)
    unsigned char grec[NWG_DTC][GRB];            // gamma records; also the 4 slot groups the M-step
                                                 // (M = 128) reads past the last record (junk rows)
    unsigned char bt[NG][1024];                  // [Theta_hi | Theta_lo]: K-major 32 rows (hi: components, lo) x 16 slots
    float tk[KC], cst[KC];
    double wred[4 * NWG_DTC];
    uint64_t xfull[XSD], xfree[XSD], aeready[NWG_DTC], edone[NWG_DTC], mready[NWG_DTC], mdone[NWG_DTC];
    uint32_t tmem;
};

constexpr int ECOL = 0;                          // E accumulator of WG w: columns 32 w (hi Theta_hi + lo Theta_hi | hi Theta_lo)
constexpr int MCOL = 32 * NWG_DTC;               // M accumulators of WG w: MCOL + 32 NACC w
static_assert(sizeof(((SmemDT*)0)->grec) >= 4 * SGB, "junk rows of the last record");
constexpr uint32_t TCOLS = MCOL + 32 * NACC * NWG_DTC <= 256 ? 256 : 512;  // TMEM allocation (power of two)
static_assert(MCOL + 32 * NACC * NWG_DTC <= 512, "TMEM columns");

}  // namespace

__global__ void __launch_bounds__(nthr_dtc(), 1)
    k_em_diag_tc(const __grid_constant__ CUtensorMap xmap, int64_t n, int D, int K, const double* __restrict__ model,
                 const double* __restrict__ center, double xs, const __grid_constant__ NegCx ncx,
                 double* __restrict__ partial) {
    constexpr int NWG = NWG_DTC, NTHR = nthr_dtc();
    constexpr int WTMA = 4 * NWG, WE = 4 * NWG + 1, WM = 4 * NWG + 2;
    extern __shared__ __align__(128) unsigned char smraw[];
    SmemDT& S = *reinterpret_cast<SmemDT*>(smraw + ((128u - (su32(smraw) & 127u)) & 127u));
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    ModelView mv{K, D, const_cast<double*>(model)};
    const int64_t ntiles = (n + TM - 1) / TM;
    const int64_t J = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    // ------------------------------------------------------------------ staging
    for (int e = t; e < XSD * DG * TM; e += NTHR) (&S.xd[0][0])[e] = 0.0;  // planes >= D stay zero
    if (t < KC) {  // t_k: power of two putting component k's largest |coefficient| into (2^12, 2^13]
        const int k = t;
        float tk = 1.f;
        if (k < K) {
            double m = 0.0, cg[NG] = {0.0, 0.0, 0.0};
            for (int f = 0; f < D; ++f) {
                const double p = 1.0 / (mv.cov()[(int64_t)k * D * D + f * D + f] * xs * xs);  // x^ units
                const double mu = (mv.mu()[k * D + f] - center[f]) * xs;
                m = fmax(m, fmax(0.5 * p, fabs(p * mu)));
                cg[f < 2 * GF ? f / GF : 2] -= 0.5 * p * mu * mu;
            }
            if (!ES_DTC_CST) cg[0] += mv.logpi()[k] + mv.lognorm()[k];
            for (int g = 0; g < NG; ++g) m = fmax(m, fabs(cg[g]));
            if (m > 0.0) tk = (float)exp2(ceil(log2(m)) - 13.0);
        }
        S.tk[k] = tk;
        S.cst[k] = (ES_DTC_CST && k < K) ? (float)(mv.logpi()[k] + mv.lognorm()[k]) : 0.f;
    }
    __syncthreads();
    for (int e = t; e < NG * KC * 16; e += NTHR) {  // Theta: group g, component k, slot s
        const int g = e / (KC * 16), k = (e / 16) % KC, s = e % 16;
        double th = 0.0;
        if (k < K) {
            const double it = 1.0 / (double)S.tk[k];
            auto pm = [&](int f, double& p, double& mu) {
                p = 1.0 / (mv.cov()[(int64_t)k * D * D + f * D + f] * xs * xs);
                mu = (mv.mu()[k * D + f] - center[f]) * xs;
            };
            if (s < 2 * GF) {
                const int f = GF * g + (s < GF ? s : s - GF);
                if (f < D) {
                    double p, mu;
                    pm(f, p, mu);
                    th = (s < GF ? -0.5 * p : p * mu) * it;
                }
            } else if (s == SLOT1) {
                double c0 = (g == 0 && !ES_DTC_CST) ? mv.logpi()[k] + mv.lognorm()[k] : 0.0;
                for (int i = 0; i < GF; ++i) {
                    const int f = GF * g + i;
                    if (f < D) {
                        double p, mu;
                        pm(f, p, mu);
                        c0 -= 0.5 * p * mu * mu;
                    }
                }
                th = c0 * it;
            }
        }
        const __half hh = __double2half(th);
        const __half hl = __double2half(th - (double)__half2float(hh));
        *reinterpret_cast<__half*>(S.bt[g] + kmaj(k, s)) = hh;
        *reinterpret_cast<__half*>(S.bt[g] + kmaj(KC + k, s)) = hl;
    }
    if (warp == WE) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&S.tmem)), "r"(TCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        for (int i = 0; i < XSD; ++i) {
            mbar_init(&S.xfull[i], 1);
            mbar_init(&S.xfree[i], 4);
        }
        for (int i = 0; i < NWG; ++i) {
            mbar_init(&S.aeready[i], 4);
            mbar_init(&S.edone[i], 1);
            mbar_init(&S.mready[i], 4);
            mbar_init(&S.mdone[i], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    proxy_fence();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = S.tmem;
    auto tile_of = [&](int64_t j) { return (int64_t)blockIdx.x + j * gridDim.x; };

    if (warp < WTMA) {
        // ====================================================== epilogue warpgroups
        const int w = warp >> 2;
        const int p = t & 127;   // event of the tile = TMEM lane; as M-step row: statistic slot
        const int q = warp & 3;  // TMEM lane quadrant = record group of the hi rows this warp flushes
        const uint32_t lq = (uint32_t)(32 * q) << 16;
        const int64_t Jw = w < J ? (J - 1 - w) / NWG + 1 : 0;  // this WG's tiles: j = w + NWG jj
        float tkr[KC], cstr[KC];
#pragma unroll
        for (int k = 0; k < KC; ++k) {
            tkr[k] = S.tk[k];
            cstr[k] = S.cst[k];
        }
        // M-step row sums of this thread's statistic (rows 32q + lane, lanes < 15 of warps 0-2), 16
        // components in compensated FP32 pairs
        uint64_t ah[KC / 2], al[KC / 2];
#pragma unroll
        for (int k = 0; k < KC / 2; ++k) ah[k] = al[k] = 0;
        float llh = 0.f, lll = 0.f;

        auto convert = [&](int64_t jj) {
            const int64_t j = w + NWG * jj;
            const int s = (int)(j % XSD);
            mbar_wait(su32(&S.xfull[s]), (uint32_t)((j / XSD) & 1));
            float xh[DG];
#pragma unroll
            for (int f = 0; f < DG; ++f) xh[f] = (float)fma(S.xd[s][f * TM + p], xs, ncx.v[f]);
            __syncwarp();
            if (lane == 0) arrive(&S.xfree[s]);
            unsigned char* R = S.rec[w][jj & 1] + (p >> 3) * 128 + (p & 7) * 16;
#pragma unroll
            for (int g = 0; g < NG; ++g) {
                float v[16];
#pragma unroll
                for (int i = 0; i < GF; ++i) {
                    const int f = GF * g + i;
                    v[i] = f < DG ? xh[f] * xh[f] : 0.f;
                    v[GF + i] = f < DG ? xh[f] : 0.f;
                }
                v[SLOT1] = 1.f;
                v[15] = 0.f;
                uint32_t hi[8], lo[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    hi[i] = pack_h2(v[2 * i], v[2 * i + 1]);
                    const float2 hf = __half22float2(u2h(hi[i]));
                    lo[i] = pack_h2(v[2 * i] - hf.x, v[2 * i + 1] - hf.y);
                }
                *reinterpret_cast<uint4*>(R + (4 * g + 0) * SGB) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
                *reinterpret_cast<uint4*>(R + (4 * g + 1) * SGB) = make_uint4(hi[4], hi[5], hi[6], hi[7]);
                *reinterpret_cast<uint4*>(R + (4 * g + 2) * SGB) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
                *reinterpret_cast<uint4*>(R + (4 * g + 3) * SGB) = make_uint4(lo[4], lo[5], lo[6], lo[7]);
            }
            proxy_fence();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) arrive(&S.aeready[w]);
        };
        auto flush = [&](int64_t jj) {  // M-step accumulators of local tile jj -> compensated FP32 rows
            mbar_wait(su32(&S.mdone[w]), (uint32_t)(jj & 1));
            tc_fence_after();
            if (q < NG) {
                float v[KC];
#pragma unroll
                for (int k = 0; k < KC; ++k) v[k] = 0.f;
#pragma unroll
                for (int ac = 0; ac < NACC; ++ac) {  // columns: gamma_hi products 0-15, gamma_lo products 16-31
                    float mh[16], ml[16];
                    tmem_ld16(tmem + lq + MCOL + 32 * NACC * w + 32 * ac, mh);
                    tmem_ld16(tmem + lq + MCOL + 32 * NACC * w + 32 * ac + 16, ml);
                    tmem_wait_ld();
#pragma unroll
                    for (int k = 0; k < KC; ++k) v[k] += mh[k] + ml[k];
                }
#pragma unroll
                for (int k = 0; k < KC; k += 2) cacc2(ah[k / 2], al[k / 2], pack2(v[k], v[k + 1]));
            }
            tc_fence_before();
        };

        if (Jw > 0) convert(0);
        for (int64_t jj = 0; jj < Jw; ++jj) {
            const int64_t j = w + NWG * jj;
            const bool valid = tile_of(j) * TM + p < n;
            mbar_wait(su32(&S.edone[w]), (uint32_t)(jj & 1));
            tc_fence_after();
            float a[16], b[16];
            tmem_ld16(tmem + lq + ECOL + 32 * w, a);
            tmem_ld16(tmem + lq + ECOL + 32 * w + 16, b);
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < 16; ++k) a[k] += b[k];
            float wk[KC];
            float mx = -INFINITY;
#pragma unroll
            for (int k = 0; k < KC; ++k) {
                wk[k] = k < K ? (ES_DTC_CST ? fmaf(a[k], tkr[k], cstr[k]) : a[k] * tkr[k]) : -INFINITY;
                mx = fmaxf(mx, wk[k]);
            }
            if (jj > 0) flush(jj - 1);  // frees the M region, the gamma record and record buffer (jj + 1) & 1
            if (jj + 1 < Jw) convert(jj + 1);
            float e[KC], ssum = 0.f;
#pragma unroll
            for (int k = 0; k < KC; ++k) {
                e[k] = ex2((wk[k] - mx) * 1.4426950408889634f);
                ssum += e[k];
            }
            const float ll = mx + lg2(ssum) * 0.6931471805599453f;
            const float r = valid ? __fdividef(GSCALE, ssum) : 0.f;
            if (valid) cacc(llh, lll, ll);
            // gamma as fp16 hi + lo: most events have one gamma within 2^-12 of 1, where a single
            // rounding is not random (it rounds 1 - eps up to 1 for every such event)
            uint32_t gh[KC / 2], gl[KC / 2];
#pragma unroll
            for (int k = 0; k < KC; k += 2) {
                const float g0 = e[k] * r, g1 = e[k + 1] * r;
                gh[k / 2] = pack_h2(g0, g1);
                const float2 hf = __half22float2(u2h(gh[k / 2]));
                gl[k / 2] = pack_h2(g0 - hf.x, g1 - hf.y);
            }
            unsigned char* G = S.grec[w] + (p >> 3) * 128 + (p & 7) * 16;
            *reinterpret_cast<uint4*>(G) = make_uint4(gh[0], gh[1], gh[2], gh[3]);
            *reinterpret_cast<uint4*>(G + SGB) = make_uint4(gh[4], gh[5], gh[6], gh[7]);
            *reinterpret_cast<uint4*>(G + 2 * SGB) = make_uint4(gl[0], gl[1], gl[2], gl[3]);
            *reinterpret_cast<uint4*>(G + 3 * SGB) = make_uint4(gl[4], gl[5], gl[6], gl[7]);
            proxy_fence();
            __syncwarp();
            if (lane == 0) arrive(&S.mready[w]);
        }
        if (Jw > 0) flush(Jw - 1);
        // -------------------------------------------------------------- output
        // rows (group q, slot lane) of every WG -> FP64 scratch
        named_sync(1, 128 * NWG);
        // [NWG][NG][32 slots: hi chunk | lo chunk][KC] in the record buffers: every MMA that read
        // them completed (each WG waited for its last M-step before the barrier above)
        double* sc = reinterpret_cast<double*>(&S.rec[0][0][0]);
        static_assert(NWG_DTC * NG * 32 * KC * sizeof(double) <= sizeof(S.rec), "output scratch");
        if (q < NG) {
#pragma unroll
            for (int k = 0; k < KC; ++k)
                sc[((w * NG + q) * 32 + lane) * KC + k] = cval(ah[k >> 1], al[k >> 1], k & 1) * (1.0 / GSCALE);
        }
        {
            const double v = warp_sum((double)llh + (double)lll);
            if (lane == 0) S.wred[warp] = v;
        }
        named_sync(1, 128 * NWG);
        const int SK = stat_k(D), NE = K * SK;
        double* myp = partial + (int64_t)blockIdx.x * (NE + 1);
        for (int e = t; e < NE; e += 128 * NWG) {
            const int k = e / SK, rr = e % SK;
            auto row = [&](int g, int s) {  // hi slot s of group g + its lo slot, fixed WG order
                double v = 0.0;
#pragma unroll
                for (int ww = 0; ww < NWG; ++ww)
                    v += sc[((ww * NG + g) * 32 + s) * KC + k] + sc[((ww * NG + g) * 32 + 16 + s) * KC + k];
                return v;
            };
            const double A0 = row(0, SLOT1);
            double v = 0.0;
            int f = -1;
            bool sq = false;
            if (rr == 0) {
                v = A0;
            } else if (rr <= D) {
                f = rr - 1;
            } else {
                int pi = rr - 1 - D, a = 0;
                while (pi >= D - a) {
                    pi -= D - a;
                    ++a;
                }
                if (pi == 0) {
                    f = a;
                    sq = true;
                }
            }
            if (f >= 0) {
                const int g = f < NG * GF - GF ? f / GF : NG - 1, i = f - GF * g;
                const double d = (mv.mu()[k * D + f] - center[f]) * xs;  // old mean, x^ units (exact FP64)
                const double A1 = row(g, GF + i);
                if (!sq) {
                    v = (A1 - A0 * d) / xs;
                } else {
                    const double A2 = row(g, i);
                    v = (A2 - 2.0 * d * A1 + d * d * A0) / (xs * xs);
                }
            }
            myp[e] = v;
        }
        if (t == 0) {
            double s = 0.0;
            for (int i = 0; i < 4 * NWG; ++i) s += S.wred[i];
            myp[NE] = s;
        }
    } else if (warp == WTMA) {
        // ========================================================== TMA producer
        if (lane == 0) {
            for (int64_t j = 0; j < J; ++j) {
                const int s = (int)(j % XSD);
                if (j >= XSD) mbar_wait_sleep(su32(&S.xfree[s]), (uint32_t)(((j - XSD) / XSD) & 1));
                mbar_expect_tx(su32(&S.xfull[s]), (uint32_t)(D * TM * 8));
                tma_load_2d(su32(&S.xd[s][0]), &xmap, (int)(tile_of(j) * TM), 0, su32(&S.xfull[s]));
            }
        }
    } else if (warp == WE) {
        // ==================================================== E-step MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc32 = idesc_f16(128, 32, 0), idesc16 = idesc_f16(128, 16, 0);
            uint64_t bhl[NG];
#pragma unroll
            for (int g = 0; g < NG; ++g) bhl[g] = sdesc(su32(S.bt[g]), 128, 256);  // rows 0-15: Theta_hi
            for (int64_t je = 0; je < J; ++je) {
                const int w = (int)(je % NWG);
                const int64_t jl = je / NWG;
                mbar_wait_sleep(su32(&S.aeready[w]), (uint32_t)(jl & 1));
                tc_fence_after();
                const uint32_t rb = su32(S.rec[w][jl & 1]);
                const uint32_t d = tmem + ECOL + 32 * w;
#pragma unroll
                for (int g = 0; g < NG; ++g) {
                    // K-major A: chunk (slot groups 2 ch, 2 ch + 1; LBO = slot-group stride),
                    // rows = events (SBO = 128 B per 8 events).  hi chunk x [Theta_hi | Theta_lo]
                    // (N = 32: columns 0-15 and 16-31), lo chunk x Theta_hi onto columns 0-15.
                    const uint64_t ah = sdesc(rb + (4 * g) * SGB, SGB, 128);
                    const uint64_t alo = sdesc(rb + (4 * g + 2) * SGB, SGB, 128);
                    mma_f16(d, ah, bhl[g], idesc32, g > 0 ? 1u : 0u);
                    mma_f16(d, alo, bhl[g], idesc16, 1u);
                }
                commit(&S.edone[w]);
            }
        }
    } else if (warp == WM) {
        // ===================================================== M-step MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_f16(128, 32, 1);  // N: gamma_hi (16) | gamma_lo (16)
            for (int64_t jm = 0; jm < J; ++jm) {
                const int w = (int)(jm % NWG);
                const int64_t jl = jm / NWG;
                mbar_wait_sleep(su32(&S.mready[w]), (uint32_t)(jl & 1));
                tc_fence_after();
                const uint64_t da = sdesc(su32(S.rec[w][jl & 1]), 128, SGB);
                const uint64_t dg = sdesc(su32(S.grec[w]), 128, SGB);
#pragma unroll
                for (int ks = 0; ks < TM / 16; ++ks)
                    mma_f16(tmem + MCOL + 32 * NACC * w + 32 * (ks % NACC), da + 16 * ks, dg + 16 * ks, idesc,
                            ks >= NACC ? 1u : 0u);
                commit(&S.mdone[w]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == WE) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
}

// ES_EM_DIAG_TC=0 keeps the FP32 SIMT k_em_diag_mixed pass; =2 (diagnostics) also takes
// iterations with fewer than kOnePassMinNk events in some component.  Read per call.
int em_diag_tc_mode() {
    const char* e = getenv("ES_EM_DIAG_TC");
    return (e && e[0] == '0') ? 0 : (e && e[0] == '2') ? 2 : 1;
}
bool em_diag_tc_enabled(int D, int K) { return em_diag_tc_mode() != 0 && D <= DG && K <= KC; }

void launch_em_diag_tc(const CUtensorMap* xmap, int64_t n, int D, int K, const double* model, const double* center,
                       const double* center_host, double xs, double* partial, int num_sms, int* nblk, cudaStream_t s,
                       LaunchStats& ls) {
    NegCx ncx{};
    for (int j = 0; j < D && j < DG; ++j) ncx.v[j] = -center_host[j] * xs;
    const int64_t ntiles = (n + TM - 1) / TM;
    const int grid = (int)std::min<int64_t>(num_sms, std::max<int64_t>(ntiles, 1));
    *nblk = grid;
    const size_t smem = sizeof(SmemDT) + 128;
    static bool a = false;
    if (!a) {
        cudaFuncSetAttribute(k_em_diag_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        a = true;
    }
    k_em_diag_tc<<<grid, nthr_dtc(), smem, s>>>(*xmap, n, D, K, model, center, xs, ncx, partial);
    ++ls.launches;
}

}  // namespace es
