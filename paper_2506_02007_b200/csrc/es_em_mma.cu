// es_em_mma.cu — fused EM pass with BOTH the E-step whitening and the M-step
// Gram on the 5th-gen tensor cores (default for D <= 16, K <= 8).
//
// Per 128-event tile (one CTA per SM, persistent over tiles):
//   converter WG  thread = event: coalesced loads of the FP64 planes (one tile of
//                 prefetch in registers), x^ = (x - c) xs -> an FP32 row (for the
//                 records) and the fp16 hi + lo K-major UMMA operand.
//   MMA warp      E:  U = b' + W' x^  as 4 kind::f16 dispatches (1 * fp32(b') first, then x_hi W_hi,
//                     x_hi W_lo, x_lo W_hi) -> TMEM, M = N = 128;
//                 M:  Gram of the tile's per-event records over its 128 events
//                     (8 K-steps of 16 events), M = 128 rows (k, a).
//   epilogue WG   thread = event = TMEM lane: squared norms of U, log-sum-exp,
//                 sqrt(responsibilities) s_k, the records; and thread = (k, a) =
//                 TMEM lane of the Gram accumulator: the flush of the Gram of the
//                 previous-but-one tile (double-buffered in TMEM, flushed every
//                 tile), FP32 over <= 8 tiles, then FP64 in shared memory.
//
// Records (fp16, MN-major, one 19-group row per event):
//   groups 0..15: R_h = fp16(s_k (x^ - m_k)) | 16: s_h |
//   17: s_l | 18: s_h/2, and (NPASS = 2) a second record 2 R_l = fp16(2 (r - R_h)).
// Pass 1:  R_h^T [R_h | s_h | s_l]                      (N = 144; N = 136 without s_l)
// Pass 2:  (2 R_l)^T R_h -> Gram columns, (2 R_l)^T (s_h/2) -> s_h columns (N = 128 + 8)
// so that P = R_h^T R_h + 2 R_l^T R_h and sym(P) = R_h^T R_h + R_l^T R_h + R_h^T R_l
// (the Gram to ~2^-21), and the first moment R_h s_h + R_h s_l + R_l s_h.
// NPASS = 1 keeps only R_h^T [R_h | s_h] (2^-12 per-event rounding noise).
//
// Numerics.  tcgen05 accumulates in FP32 with truncation
// toward zero (measured ~1 ulp of the running sum per dispatch,
// scripts/umma_probe.cu), so nothing that cancels is accumulated on the tensor
// core: U only feeds the responsibilities, and the Gram is of records centred on
// a per-CTA running estimate of the new mean (recentred after tiles 1, 2, 4, ...
// with an exact FP64 re-expression; re-expressed about the starting centre at the
// end), whose truncation bias is ~8 ulp of a same-sign per-tile sum (~6e-7).
// xs is a power of two bringing max|x - c| into (8, 16]; t_k (a power of two)
// puts the largest |entry| of W'/t_k, b'/t_k into (2^12, 2^13] so the fp16 lo
// parts of all but negligible entries are normal numbers.
#include <cmath>
#include <cstdlib>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include "es_kernels.h"
#include "es_mma.cuh"

#ifndef ES_EM_KB
#define ES_EM_KB 2
#endif

namespace es {

#ifdef ES_EM_TRACE
// debug timeline of CTA 0 (scripts/em_trace.py): clock64 per (event, tile)
constexpr int TR_EV = 12, TR_T = 128;
__device__ long long g_em_trace[TR_EV][TR_T];
#define TRACE(ev, j)                                                          \
    do {                                                                      \
        if (blockIdx.x == 0 && (j) < TR_T) g_em_trace[ev][(j)] = clock64();   \
    } while (0)
#else
#define TRACE(ev, j) \
    do {             \
    } while (0)
#endif

namespace {

using namespace mma;

// NWG epilogue warpgroups take tiles round robin (2; 3 is an NPASS = 1 option,
// ES_EM_MMA_WG), then a TMA warp and an MMA-issuer warp.
constexpr int nthr(int nwg) { return 128 * nwg + 96; }  // + TMA warp, E-issuer warp, Gram-issuer warp
constexpr uint32_t GRP = (TM / 8) * 128;   // one MN-major group of 8 columns: 16 K-groups x 128 B
constexpr uint32_t RECL = 16 * GRP;        // 32768 B
constexpr int MREG0 = 128;                 // two Gram regions (tile parity) from TMEM column 128
constexpr int mregs(int npass) { return npass == 2 ? 144 : 136; }
constexpr int ta0(int npass) { return MREG0 + 2 * mregs(npass); }  // x^ hi/lo A operands, 16 columns per WG
constexpr int tone(int npass, int nwg) { return ta0(npass) + 16 * nwg; }  // ones (bias dispatch A operand)
static_assert(tone(1, 3) + 8 <= 512 && tone(2, 2) + 8 <= 512, "TMEM columns");

template <int NPASS, int NWG>
struct Smem {
    static constexpr int XS = NPASS == 2 ? 3 : 4;       // FP64 tile stages (TMA)
    static constexpr uint32_t RECH = (NPASS == 2 ? 19 : 17) * GRP;
    double xd[XS][DM * TM];                             // 48 / 64 KB  FP64 tiles (planar, TMA destination)
    unsigned char rech[NWG][RECH];                      // hi records (per warpgroup)
    unsigned char recl[NPASS == 2 ? NWG : 1][NPASS == 2 ? RECL : 16];  // 2 x lo records
    unsigned char bw[2][OPB];                           // W' hi / lo
    unsigned char bb[OPB];                              // fp32(b') as three fp16 parts in K columns 0-2
    double c[DM];
    double shift[NWG][KMAX * DM];                       // record centre - starting centre (FP64, exact)
    double dl[NWG][KMAX * DM], s1x[NWG][KMAX * DM];     // recentring exchange
    double wred[4 * NWG][KMAX + 1];                     // per-warp partial N_k | logL
    double ntot[NWG][KMAX];
    float nmu[NWG][KMAX * DM];                          // -(record centre), x^ units, FP32
    float cst[KMAX];                                    // log pi_k + lognorm_k
    float hq[KMAX];                                     // 0.5 t_k^2
    float tk[KMAX];
    uint64_t xfull[XS], xfree[XS], aeready[NWG], edone[NWG], mready[NWG], mdone[NWG], rfree[2], efree;
    uint32_t tmem;
};

}  // namespace

template <int NPASS, bool F32, int NWG>
__global__ void __launch_bounds__(nthr(NWG), 1) k_em_mma(const __grid_constant__ CUtensorMap xmap, int64_t n, int D,
                                                          int K, const double* __restrict__ model,
                                                          const double* __restrict__ center, double xs,
                                                          const __grid_constant__ NegCx ncx,
                                                          const __grid_constant__ NegCxF ncxf, const float xsf,
                                                          double* __restrict__ partial) {
    using Sm = Smem<NPASS, NWG>;
    constexpr int XS = Sm::XS, NTHR = nthr(NWG), MREGS = mregs(NPASS), TA0 = ta0(NPASS), TONE = tone(NPASS, NWG);
    constexpr int WTMA = 4 * NWG, WMMA = 4 * NWG + 1, WGRM = 4 * NWG + 2;
    extern __shared__ __align__(128) unsigned char smraw[];
    // keep the shared-window provenance of the pointer (generic LD/ST otherwise)
    Sm& S = *reinterpret_cast<Sm*>(smraw + ((128u - (su32(smraw) & 127u)) & 127u));
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    ModelView mv{K, D, const_cast<double*>(model)};
    const int64_t ntiles = (n + TM - 1) / TM;
    const int64_t J = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    // ------------------------------------------------------------------ staging
    for (int j = t; j < DM; j += NTHR) S.c[j] = j < D ? center[j] : 0.0;
    for (int e = t; e < XS * DM * TM; e += NTHR) (&S.xd[0][0])[e] = 0.0;  // planes >= D stay zero
    stage_estep(mv, K, D, center, S.c, xs, S.bw[0], S.bw[1], S.bb, S.cst, nullptr, S.hq, S.tk, t, NTHR);
    for (int e = t; e < KMAX * DM; e += NTHR) {
        const int k = e / DM, f = e % DM;
        const float m0 = (k < K && f < D) ? -(float)((mv.mu()[k * D + f] - center[f]) * xs) : 0.f;
        for (int w = 0; w < NWG; ++w) {
            S.nmu[w][e] = m0;
            S.shift[w][e] = 0.0;
        }
    }
    if (warp == WMMA) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&S.tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        for (int i = 0; i < XS; ++i) {
            mbar_init(&S.xfull[i], 1);
            mbar_init(&S.xfree[i], 4);
        }
        for (int i = 0; i < NWG; ++i) {
            mbar_init(&S.aeready[i], 4);
            mbar_init(&S.edone[i], 1);
            mbar_init(&S.mready[i], 4);
            mbar_init(&S.mdone[i], 1);
        }
        for (int i = 0; i < 2; ++i) mbar_init(&S.rfree[i], 4);
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
        if (NPASS == 2) {  // the s_l columns start at zero (only the R_h^T pass writes them, accumulating)
            const uint32_t zero[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
            for (int rg = 0; rg < 2; ++rg)
                tmem_st8(tmem + ((uint32_t)(32 * warp) << 16) + MREG0 + MREGS * rg + TM + KMAX, zero);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    if (warp < WTMA) {
        // ====================================================== epilogue warpgroups
        // WG w takes tiles j = w, w + NWG, ...: converts its FP64 tile, then (thread =
        // event = TMEM lane) reads U, forms the responsibilities and the records; as
        // thread = (k, a) it flushes the Gram of its tile (region j & 1) and releases it.
        const int w = warp >> 2;
        const int p = t & 127;             // event row of the tile / Gram row (k, a)
        const int q = warp & 3;            // TMEM lane quadrant
        const uint32_t lq = (uint32_t)(32 * q) << 16;
        const int hsel = lane >> 4;        // Gram row (k, a): k = 2q + hsel, a = lane & 15
        const int kk = p >> 4, aa = p & 15;
        // three warpgroups (128 registers): constants from shared memory, next tile
        // converted after the records instead of being held in registers across them
        constexpr bool LATE = NWG == 3;
        float cst[KMAX], hq[KMAX];
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
            cst[k] = LATE ? 0.f : S.cst[k];
            hq[k] = LATE ? 0.f : S.hq[k];
        }
        // statistics in compensated FP32 pairs (hi, lo): Gram row, first moment, N_k; logL in FP64
        uint64_t g2h[DM / 2], g2l[DM / 2], nkh[KMAX / 2], nkl[KMAX / 2];
        float g1h = 0.f, g1l = 0.f, llh = 0.f, lll = 0.f;
#pragma unroll
        for (int b = 0; b < DM / 2; ++b) g2h[b] = g2l[b] = 0;
#pragma unroll
        for (int k = 0; k < KMAX / 2; ++k) nkh[k] = nkl[k] = 0;
        auto g2v = [&](int b) { return cval(g2h[b >> 1], g2l[b >> 1], b & 1); };
        auto set2 = [&](uint64_t& hi, uint64_t& lo, double a, double b) {
            const float ah = (float)a, bh = (float)b;
            hi = pack2(ah, bh);
            lo = pack2((float)(a - (double)ah), (float)(b - (double)bh));
        };

        auto flush = [&](int64_t jj) {  // Gram of this WG's local tile jj (tile w + NWG jj) -> FP64
            if (p == 0) TRACE(6, w + NWG * jj);
            mbar_wait(su32(&S.mdone[w]), (uint32_t)(jj & 1));
            tc_fence_after();
            const int rg = (int)((w + NWG * jj) & 1);
            const uint32_t xg = (uint32_t)(MREG0 + MREGS * rg);
            float v[32], f0, f1, m1;
            tmem_ld32(tmem + lq + xg + 32 * q, v);
            tmem_ld2(tmem + lq + xg + TM + 2 * q, f0, f1);
            if (NPASS == 2) {
                float e0, e1;
                tmem_ld2(tmem + lq + xg + TM + KMAX + 2 * q, e0, e1);
                tmem_wait_ld();
                m1 = hsel ? f1 + e1 : f0 + e0;
                // zero the s_l columns for the region's next Gram (its first dispatches are the lo
                // passes, which do not write them)
                const uint32_t zero[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
                tmem_st8(tmem + lq + xg + TM + KMAX, zero);
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            } else {
                tmem_wait_ld();
                m1 = hsel ? f1 : f0;
            }
#pragma unroll
            for (int b = 0; b < DM; b += 2)
                cacc2(g2h[b / 2], g2l[b / 2], hsel ? pack2(v[16 + b], v[17 + b]) : pack2(v[b], v[b + 1]));
            cacc(g1h, g1l, m1);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) arrive(&S.rfree[rg]);
            if (p == 0) TRACE(7, w + NWG * jj);
        };
        // N_k of this WG (fixed-order reduction) -> S.ntot[w]
        auto wg_counts = [&]() {
#pragma unroll
            for (int k = 0; k < KMAX; ++k) {
                const double v = warp_sum(cval(nkh[k >> 1], nkl[k >> 1], k & 1));
                if (lane == 0) S.wred[warp][k] = v;
            }
            named_sync(4 + w, 128);
            if (p < KMAX) {
                double s = 0.0;
                for (int i = 0; i < 4; ++i) s += S.wred[4 * w + i][p];
                S.ntot[w][p] = s;
            }
            named_sync(4 + w, 128);
        };
        // Move this WG's accumulation centre for component k to its running estimate of
        // the new mean (x^ units, rounded to FP32 for the records) and re-express the
        // FP64 statistics about it exactly:
        //   P' = P - s1 d^T - d s1^T + N d d^T,  s1' = s1 - N d.
        // `back` re-expresses about the kernel's starting centre instead (d = -shift).
        auto recentre = [&](bool back) {
            wg_counts();
            const double N = S.ntot[w][kk];
            double g1 = (double)g1h + (double)g1l;
            double d = 0.0;
            if (back) {
                d = -S.shift[w][p];
            } else if (kk < K && aa < D && N > 0.5) {
                const float cur = -S.nmu[w][p];
                const float nw = (float)((double)cur + g1 / N);
                d = (double)nw - (double)cur;
            }
            S.dl[w][p] = d;
            S.s1x[w][p] = g1;
            named_sync(4 + w, 128);
#pragma unroll
            for (int bb = 0; bb < DM; bb += 2) {
                double nv[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const double db = S.dl[w][kk * DM + bb + h], sb = S.s1x[w][kk * DM + bb + h];
                    nv[h] = g2v(bb + h) + fma(N * d, db, -fma(g1, db, d * sb));
                }
                set2(g2h[bb / 2], g2l[bb / 2], nv[0], nv[1]);
            }
            g1 = fma(-N, d, g1);
            g1h = (float)g1;
            g1l = (float)(g1 - (double)g1h);
            if (!back) {
                S.nmu[w][p] = -(float)(-(double)S.nmu[w][p] + d);
                S.shift[w][p] += d;
            }
            named_sync(4 + w, 128);
        };

        int64_t pendt = -1;  // last local tile whose Gram is not flushed yet
        int64_t jj = 0;      // local tile index
        // convert tile j: x^ = (x - c) xs -> FP32 row (registers) + fp16 hi/lo E-step A operand
        // in this WG's TMEM columns (lane = event, tcgen05.st)
        auto convert = [&](int64_t j, uint64_t (&x2)[DM / 2]) {
            const int s = (int)(j % XS);
            mbar_wait(su32(&S.xfull[s]), (uint32_t)((j / XS) & 1));
            uint32_t hw[DM / 2], lw[DM / 2];
#pragma unroll
            for (int f = 0; f < DM; f += 2) {
                float v0, v1;
                if (F32) {  // FP32 pipe: x within 4x of its spread about c (see launch_em_mma)
                    v0 = fmaf(__double2float_rn(S.xd[s][f * TM + p]), xsf, ncxf.v[f]);
                    v1 = fmaf(__double2float_rn(S.xd[s][(f + 1) * TM + p]), xsf, ncxf.v[f + 1]);
                } else {
                    v0 = (float)fma(S.xd[s][f * TM + p], xs, ncx.v[f]);
                    v1 = (float)fma(S.xd[s][(f + 1) * TM + p], xs, ncx.v[f + 1]);
                }
                x2[f / 2] = pack2(v0, v1);
                const uint32_t h = pack_h2(v0, v1);
                const float2 hf = __half22float2(u2h(h));
                hw[f / 2] = h;
                float l0, l1;
                unpack2(sub2(x2[f / 2], pack2(hf.x, hf.y)), l0, l1);
                lw[f / 2] = pack_h2(l0, l1);
            }
            tmem_st8(tmem + lq + TA0 + 16 * w, hw);
            tmem_st8(tmem + lq + TA0 + 16 * w + 8, lw);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {  // per warp: its 32 events are read and staged
                arrive(&S.xfree[s]);
                arrive(&S.aeready[w]);
            }
            if (p == 0) TRACE(5, j);
        };
        uint64_t x2[DM / 2], x2n[DM / 2];
        if (w < J) convert(w, x2);
        for (int64_t j = w; j < J; j += NWG, ++jj) {
            const bool valid = tile_of(j) * TM + p < n;
            // ---- E-step epilogue
            mbar_wait(su32(&S.edone[w]), (uint32_t)(jj & 1));
            tc_fence_after();
            if (p == 0) TRACE(3, j);
            float wk[KMAX];
            float mx = -INFINITY;
            // U in batches of KB components (one TMEM load wait per batch); the E region is
            // released as soon as the last batch is in registers
            constexpr int KB = ES_EM_KB;
#pragma unroll
            for (int k0 = 0; k0 < KMAX; k0 += KB) {
                float u[KB][16];
#pragma unroll
                for (int k = 0; k < KB; ++k) tmem_ld16(tmem + lq + 16 * (k0 + k), u[k]);
                tmem_wait_ld();
                if (k0 + KB == KMAX) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) arrive(&S.efree);
                    if (p == 0) TRACE(4, j);
                }
#pragma unroll
                for (int k = 0; k < KB; ++k) {
                    uint64_t q2 = 0, q3 = 0;
#pragma unroll
                    for (int r = 0; r < 16; r += 4) {
                        const uint64_t ua = pack2(u[k][r], u[k][r + 1]), ub = pack2(u[k][r + 2], u[k][r + 3]);
                        ffma2(q2, ua, ua);
                        ffma2(q3, ub, ub);
                    }
                    float qa, qb, qc, qd;
                    unpack2(q2, qa, qb);
                    unpack2(q3, qc, qd);
                    const int kk2 = k0 + k;
                    wk[kk2] = LATE ? S.cst[kk2] - S.hq[kk2] * ((qa + qb) + (qc + qd))
                                   : cst[kk2] - hq[kk2] * ((qa + qb) + (qc + qd));
                    mx = fmaxf(mx, wk[kk2]);
                }
            }
            // E(j) has consumed this WG's A operand: stage the next tile now, so that its
            // E-step is ready long before this tile's records are
            if (!LATE && j + NWG < J) convert(j + NWG, x2n);
            float ssum = 0.f;
#pragma unroll
            for (int k = 0; k < KMAX; ++k) ssum += ex2((wk[k] - mx) * 1.4426950408889634f);
            const float ll = mx + lg2(ssum) * 0.6931471805599453f;
            float sg[KMAX];
#pragma unroll
            for (int k = 0; k < KMAX; ++k) {
                sg[k] = valid ? ex2((wk[k] - ll) * 0.7213475204444817f) : 0.f;
            }
#pragma unroll
            for (int k = 0; k < KMAX; k += 2) {
                const uint64_t s2v = pack2(sg[k], sg[k + 1]);
                cacc2(nkh[k / 2], nkl[k / 2], mul2(s2v, s2v));
            }
            if (valid) cacc(llh, lll, ll);
            // ---- records (buffers w are free once the Gram of the previous tile completed)
            // (Accumulating two tiles' Grams in TMEM before a flush doubles the FP32
            // truncation bias and fails the 2^25-event parity test; measured no faster.)
            if (pendt >= 0) {
                flush(pendt);
                pendt = -1;
            }
            unsigned char* rh = S.rech[w] + (p >> 3) * 128 + (p & 7) * 16;
            unsigned char* rl = S.recl[NPASS == 2 ? w : 0] + (p >> 3) * 128 + (p & 7) * 16;
#pragma unroll
            for (int k = 0; k < KMAX; ++k) {
                const uint64_t s2 = pack2(sg[k], sg[k]);
                const ulonglong2* nm = reinterpret_cast<const ulonglong2*>(S.nmu[w] + k * DM);
                uint32_t oh[8], ol[8];
#pragma unroll
                for (int r = 0; r < 8; r += 2) {
                    const ulonglong2 m2 = nm[r / 2];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const uint64_t rr = mul2(add2(x2[r + h], h ? m2.y : m2.x), s2);
                        float lo, hi;
                        unpack2(rr, lo, hi);
                        oh[r + h] = pack_h2(lo, hi);
                        if (NPASS == 2) {
                            // R_h rounded to nearest (a truncated R_h would bias R_l and leave
                            // a -2^-22 diagonal bias in the dropped R_l^T R_l term)
                            const float2 hf = __half22float2(u2h(oh[r + h]));
                            const uint64_t dd = sub2(rr, pack2(hf.x, hf.y));
                            unpack2(add2(dd, dd), lo, hi);  // 2 R_l (exact doubling)
                            ol[r + h] = pack_h2(lo, hi);
                        }
                    }
                }
                *reinterpret_cast<uint4*>(rh + (2 * k) * GRP) = make_uint4(oh[0], oh[1], oh[2], oh[3]);
                *reinterpret_cast<uint4*>(rh + (2 * k + 1) * GRP) = make_uint4(oh[4], oh[5], oh[6], oh[7]);
                if (NPASS == 2) {
                    *reinterpret_cast<uint4*>(rl + (2 * k) * GRP) = make_uint4(ol[0], ol[1], ol[2], ol[3]);
                    *reinterpret_cast<uint4*>(rl + (2 * k + 1) * GRP) = make_uint4(ol[4], ol[5], ol[6], ol[7]);
                }
            }
            {
                uint32_t sh[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) sh[r] = pack_h2(sg[2 * r], sg[2 * r + 1]);
                *reinterpret_cast<uint4*>(rh + 16 * GRP) = make_uint4(sh[0], sh[1], sh[2], sh[3]);
                if (NPASS == 2) {
                    uint32_t sl[4], s5[4];
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const float2 hf = __half22float2(u2h(sh[r]));
                        sl[r] = pack_h2(sg[2 * r] - hf.x, sg[2 * r + 1] - hf.y);
                        s5[r] = pack_h2(0.5f * hf.x, 0.5f * hf.y);  // s_h / 2, exact
                    }
                    *reinterpret_cast<uint4*>(rh + 17 * GRP) = make_uint4(sl[0], sl[1], sl[2], sl[3]);
                    *reinterpret_cast<uint4*>(rh + 18 * GRP) = make_uint4(s5[0], s5[1], s5[2], s5[3]);
                }
            }
            proxy_fence();
            __syncwarp();
            if (lane == 0) arrive(&S.mready[w]);
            if (p == 0) TRACE(8, j);
            pendt = jj;
            // recentre after local tiles 1, 2, 4, 8, ... (drain this WG's Gram first)
            if (((jj + 1) & jj) == 0 && j + NWG < J) {
                flush(jj);
                pendt = -1;
                recentre(false);
            }
            if (LATE) {
                if (j + NWG < J) convert(j + NWG, x2);
            } else {
#pragma unroll
                for (int r = 0; r < DM / 2; ++r) x2[r] = x2n[r];
            }
        }
        if (pendt >= 0) flush(pendt);
        recentre(true);
        // -------------------------------------------------------------- output
        // Sum the WGs' statistics (fixed order) about the starting centre
        // c + mu^_k / xs (x units; scale by xs^-1, xs^-2, exact) and symmetrise the
        // Gram, sym(P) = (P + P^T) / 2.  The record buffers are free now (scratch).
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
            const double v = warp_sum(cval(nkh[k >> 1], nkl[k >> 1], k & 1));
            if (lane == 0) S.wred[warp][k] = v;
        }
        {
            const double v = warp_sum((double)llh + (double)lll);
            if (lane == 0) S.wred[warp][KMAX] = v;
        }
        double* rows = reinterpret_cast<double*>(&S.rech[0][0]);  // [NWG][128][17]
        static_assert(sizeof(S.rech) >= NWG * TM * (DM + 1) * sizeof(double), "output scratch");
        named_sync(7, 128 * NWG);  // all WGs drained: no Gram still reads the record buffers
#pragma unroll
        for (int b = 0; b < DM; ++b) rows[(w * TM + p) * (DM + 1) + b] = g2v(b);
        rows[(w * TM + p) * (DM + 1) + DM] = (double)g1h + (double)g1l;
        named_sync(7, 128 * NWG);
        if (w == 0) {
            const int SK = stat_k(D), NE = K * SK;
            double* myp = partial + (int64_t)blockIdx.x * (NE + 1);
            const double i1 = 1.0 / xs, i2 = i1 * i1;
            auto wsum = [&](int row, int col) {  // fixed WG order
                double s = 0.0;
#pragma unroll
                for (int g = 0; g < NWG; ++g) s += rows[(g * TM + row) * (DM + 1) + col];
                return s;
            };
            if (kk < K && aa < D) {
                double* blk = myp + kk * SK;
                blk[1 + aa] = wsum(p, DM) * i1;
                for (int bb = aa; bb < D; ++bb)
                    blk[1 + D + packed_index(aa, bb, D)] = 0.5 * (wsum(p, bb) + wsum(kk * DM + bb, aa)) * i2;
            }
            if (p < K) {
                double s = 0.0;
                for (int i = 0; i < 4 * NWG; ++i) s += S.wred[i][p];
                myp[p * SK] = s;
            }
            if (p == KMAX) {
                double s = 0.0;
                for (int i = 0; i < 4 * NWG; ++i) s += S.wred[i][KMAX];
                myp[NE] = s;
            }
        }
    } else if (warp == WTMA) {
        // ========================================================== TMA producer
        if (lane == 0) {
            for (int64_t j = 0; j < J; ++j) {
                const int s = (int)(j % XS);
                if (j >= XS) mbar_wait_sleep(su32(&S.xfree[s]), (uint32_t)(((j - XS) / XS) & 1));
                TRACE(0, j);
                mbar_expect_tx(su32(&S.xfull[s]), (uint32_t)(D * TM * 8));
                tma_load_2d(su32(&S.xd[s][0]), &xmap, (int)(tile_of(j) * TM), 0, su32(&S.xfull[s]));
            }
        }
    } else if (warp == WMMA) {
        // ==================================================== E-step MMA issuer
        // Two issuer warps (E-steps, Grams), each blocked on its mbarriers with a suspend
        // hint: no polling loop takes issue slots from the epilogue warps of its SM
        // sub-partition (a polling single issuer was ~7% of the kernel's instructions).
        if (lane == 0) {
            const uint64_t dbh = sdesc(su32(S.bw[0]), 128, 256), dbl = sdesc(su32(S.bw[1]), 128, 256);
            const uint64_t dbb = sdesc(su32(S.bb), 128, 256);
            for (int64_t je = 0; je < J; ++je) {
                const int w = (int)(je % NWG);
                mbar_wait_sleep(su32(&S.aeready[w]), (uint32_t)((je / NWG) & 1));
                if (je >= 1) mbar_wait_sleep(su32(&S.efree), (uint32_t)((je - 1) & 1));
                TRACE(1, je);
                tc_fence_after();
                const uint32_t tah = tmem + TA0 + 16 * w, tal = tah + 8;
                mma_f16_ta(tmem, tmem + TONE, dbb, kIdescE, 0u);  // fp32(b') exactly, first
                mma_f16_ta(tmem, tah, dbh, kIdescE, 1u);
                mma_f16_ta(tmem, tah, dbl, kIdescE, 1u);
                mma_f16_ta(tmem, tal, dbh, kIdescE, 1u);
                commit(&S.edone[w]);
                TRACE(9, je);
            }
        }
    } else if (warp == WGRM) {
        // ======================================================= Gram MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc1 = idesc_f16(128, NPASS == 2 ? 144 : 136, 1);
            constexpr uint32_t idesc2a = idesc_f16(128, 128, 1);
            constexpr uint32_t idesc2b = idesc_f16(128, 8, 1);
            // pass 1: D1 = R_h^T [R_h | s_h | s_l]; pass 2: P = D1 + (2 R_l)^T R_h on the Gram
            // columns, + (2 R_l)^T (s_h / 2) = R_l^T s_h on the s_h columns.
            // Gram of tile m (records of WG m % NWG into region m & 1).  Descriptors are
            // precomputed per records buffer; a K-step adds 256 B (16 in the address field).
            uint64_t dh0[NWG], dl0[NWG];
#pragma unroll
            for (int g = 0; g < NWG; ++g) {
                dh0[g] = sdesc(su32(S.rech[g]), 128, GRP);
                dl0[g] = sdesc(su32(S.recl[NPASS == 2 ? g : 0]), 128, GRP);
            }
            for (int64_t jm = 0; jm < J; ++jm) {
                const int mw = (int)(jm % NWG);
                mbar_wait_sleep(su32(&S.mready[mw]), (uint32_t)((jm / NWG) & 1));
                if (jm >= 2) mbar_wait_sleep(su32(&S.rfree[jm & 1]), (uint32_t)(((jm - 2) >> 1) & 1));
                TRACE(2, jm);
                tc_fence_after();
                const uint32_t xg = tmem + (uint32_t)(MREG0 + MREGS * (int)(jm & 1));
                const uint64_t dh = mw == 0 ? dh0[0] : (mw == 1 ? dh0[1] : dh0[NWG - 1]);
                const uint64_t dl = mw == 0 ? dl0[0] : (mw == 1 ? dl0[1] : dl0[NWG - 1]);
                if (NPASS == 2) {
                    // the small lo products first: the FP32 accumulator truncates ~1 ulp of its running
                    // sum per dispatch, so lo dispatches issued after the big R_h^T R_h ones tripled
                    // the Gram's same-sign truncation bias (the s_l columns were zeroed by the flush)
#pragma unroll
                    for (int ks = 0; ks < TM / 16; ++ks) {
                        mma_f16(xg, dl + 16 * ks, dh + 16 * ks, idesc2a, ks > 0 ? 1u : 0u);
                        mma_f16(xg + TM, dl + 16 * ks, dh + (18 * GRP >> 4) + 16 * ks, idesc2b, ks > 0 ? 1u : 0u);
                    }
                }
#pragma unroll
                for (int ks = 0; ks < TM / 16; ++ks)
                    mma_f16(xg, dh + 16 * ks, dh + 16 * ks, idesc1, (NPASS == 2 || ks > 0) ? 1u : 0u);
                commit(&S.mdone[mw]);
                TRACE(10, jm);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == WMMA) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// 2-D TMA descriptor over the planar event matrix: dims (rows, planes), box 128 rows x 16
// planes (the fused passes' FP64 tile), driver entry point resolved through the runtime.
bool make_event_tmap(CUtensorMap* map, const double* X, int64_t n, int64_t ld, int D) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return false;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    if (n <= 0 || D > 16) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)D};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
    const cuuint32_t box[2] = {TM, (cuuint32_t)D};
    const cuuint32_t estr[2] = {1, 1};
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(X), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Shapes of the fused tensor-core passes (k_em_mma / k_score_mma): the mixed path's domain.
bool em_mixed_supported(int D, int K) { return D <= DM && K <= KMAX; }

// ES_EM_KERNEL=fp64 runs the mixed-shape iterations on the strict FP64 kernel instead.
bool em_mma_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("ES_EM_KERNEL");
        v = (e && e[0] == 'f') ? 0 : 1;
    }
    return v == 1;
}

// ES_EM_MMA_PASSES=1|2 forces the record precision; otherwise (0) the caller decides.
int em_mma_passes() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("ES_EM_MMA_PASSES");
        v = (e && (e[0] == '1' || e[0] == '2')) ? e[0] - '0' : 0;
    }
    return v;
}

template <int NPASS, bool F32, int NWG>
static void launch_npass(const CUtensorMap* xmap, int64_t n, int D, int K, const double* model,
                         const double* center, double xs, const NegCx& ncx, double* partial, int grid,
                         cudaStream_t s) {
    const size_t smem = sizeof(Smem<NPASS, NWG>) + 128;
    static bool a = false;
    if (!a) {
        cudaFuncSetAttribute(k_em_mma<NPASS, F32, NWG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        a = true;
    }
    NegCxF ncxf{};
    for (int j = 0; j < DM; ++j) ncxf.v[j] = (float)ncx.v[j];
    k_em_mma<NPASS, F32, NWG><<<grid, nthr(NWG), smem, s>>>(*xmap, n, D, K, model, center, xs, ncx, ncxf,
                                                             (float)xs, partial);
}

// ES_EM_MMA_WG=3 runs the NPASS = 1 kernel with three epilogue warpgroups (128 registers
// per thread) instead of two; measured no faster (3.68-3.75 against 3.60-3.66 ms per pass).
static int em_mma_wgs() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("ES_EM_MMA_WG");
        v = (e && e[0] == '3') ? 3 : 2;
    }
    return v;
}

void launch_em_mma(const CUtensorMap* xmap, int64_t n, int D, int K, const double* model, const double* center,
                   const double* center_host, double xs, bool f32conv, int npass, double* partial, int num_sms,
                   int* nblk, cudaStream_t s, LaunchStats& ls) {
    NegCx ncx{};
    for (int j = 0; j < D && j < DM; ++j) ncx.v[j] = -center_host[j] * xs;
    static int allow = -1;
    if (allow < 0) {
        const char* e = getenv("ES_EM_F32CONV");
        allow = (e && e[0] == '0') ? 0 : 1;
    }
    f32conv = f32conv && allow;
    const int64_t ntiles = (n + TM - 1) / TM;
    const int grid = (int)std::min<int64_t>(num_sms, std::max<int64_t>(ntiles, 1));
    *nblk = grid;
    if (em_mma_passes() != 0) npass = em_mma_passes();
    const bool w3 = em_mma_wgs() == 3;
    if (npass == 1 && f32conv && w3)
        launch_npass<1, true, 3>(xmap, n, D, K, model, center, xs, ncx, partial, grid, s);
    else if (npass == 1 && f32conv)
        launch_npass<1, true, 2>(xmap, n, D, K, model, center, xs, ncx, partial, grid, s);
    else if (npass == 1 && w3)
        launch_npass<1, false, 3>(xmap, n, D, K, model, center, xs, ncx, partial, grid, s);
    else if (npass == 1)
        launch_npass<1, false, 2>(xmap, n, D, K, model, center, xs, ncx, partial, grid, s);
    else if (f32conv)
        launch_npass<2, true, 2>(xmap, n, D, K, model, center, xs, ncx, partial, grid, s);
    else
        launch_npass<2, false, 2>(xmap, n, D, K, model, center, xs, ncx, partial, grid, s);
    ++ls.launches;
}

}  // namespace es

#ifdef ES_EM_TRACE
extern "C" int es_debug_em_trace(long long* out) {
    return (int)cudaMemcpyFromSymbol(out, es::g_em_trace, sizeof(es::g_em_trace));
}
#endif
