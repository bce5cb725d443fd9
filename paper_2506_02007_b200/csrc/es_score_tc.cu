// es_score_tc.cu — tensor-core scoring pass (score_samples / predict / detect).
//
// Per 256-event tile (8 warps, thread per event):
//   TMA 2-D tensor copies of the FP64 tile (prefetched two tiles ahead)
//   -> x' = x - c, TF32 hi/lo operand -> 2 x 9 tcgen05.mma (3xTF32, K = 24)
//   -> TMEM epilogue: FP32 log densities of all K components
//   -> FP64 recomputation of the candidate components (responsibility above
//      1e-6, or within FP32 rounding of either argmax), compacted into one
//      (event, component) list per tile so FP64 work follows the candidate
//      count, not the per-warp maximum; x is read from the same shared tile
//   -> ll, predict, best_k, best_logdens, flag (FP64-exact where it matters).
// The MMA of tile j+1 is issued before the FP64 refinement of tile j, so the
// tensor cores and the TMA engine run under the FP64 work.
#include <cmath>
#include <cstdlib>

#include "es_kernels.h"
#include "es_tc.cuh"

namespace es {

namespace {

using namespace tc;

constexpr int DM = 16;
constexpr int KMAX = 8;
constexpr int TT = 256;             // events per tile
constexpr int W64S = DM * DM + 2;   // FP64 W stride (bank skew between components)

struct SmemS {
    unsigned char Bh[kOpBytes], Bl[kOpBytes];
    unsigned char Ah[2][kOpBytes], Al[2][kOpBytes];   // [sub-tile]
    double xd[3][DM * TT];                            // TMA tiles (planar), triple-buffered
    double lnv[KMAX * TT];                            // FP64 log densities of refined (k, event)
    uint16_t cev[KMAX * TT + KMAX];                   // compacted candidate list: event
    uint8_t ccomp[KMAX * TT + KMAX];                  //                            component
    int wcnt[KMAX * 8], woff[KMAX * 8], ncand;
    alignas(16) double W64[KMAX * W64S];
    double mu64[KMAX * (DM + 2)];
    double ln64[KMAX], lp64[KMAX];
    double c[DM];
    double red[TT];
    float cst[KMAX], lnf[KMAX];
    uint64_t xfull[3], mma_done;
    uint32_t tmem;
};

}  // namespace

__global__ void __launch_bounds__(TT, 1) k_score_tc(const __grid_constant__ CUtensorMap xmap, int64_t n, int D, int K,
                                                     const double* __restrict__ model,
                                                     const double* __restrict__ center, ScoreOut o,
                                                     double* __restrict__ blocksum, int getenv_refine_all) {
    extern __shared__ __align__(1024) unsigned char smraw[];
    SmemS& S = *reinterpret_cast<SmemS*>(smraw);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    ModelView mv{K, D, const_cast<double*>(model)};
    const int64_t ntiles = (n + TT - 1) / TT;
    const int64_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    for (int j = t; j < DM; j += TT) S.c[j] = j < D ? center[j] : 0.0;
    __syncthreads();
    for (int e = t; e < kTileRows * kKA; e += TT) {
        const int row = e / kKA, kk = e % kKA, k = row / DM, r = row % DM;
        double v = 0.0;
        if (k < K && r < D) {
            const double* Wr = mv.W() + (int64_t)k * D * D + (int64_t)r * D;
            if (kk < D) {
                v = Wr[kk];
            } else if (kk == DM) {
                double b = 0.0;
                for (int j = 0; j <= r; ++j) b = fma(Wr[j], mv.mu()[k * D + j] - S.c[j], b);
                v = -b;
            }
        }
        const uint32_t h = tf32((float)v);
        const uint32_t l = tf32((float)(v - (double)__uint_as_float(h)));
        *reinterpret_cast<uint32_t*>(S.Bh + op_off(row, kk)) = h;
        *reinterpret_cast<uint32_t*>(S.Bl + op_off(row, kk)) = l;
    }
    for (int e = t; e < 2 * kTileRows * (kKA - DM); e += TT) {
        const int b2 = e / (kTileRows * (kKA - DM)), rr = e % (kTileRows * (kKA - DM));
        const int row = rr / (kKA - DM), kk = DM + rr % (kKA - DM);
        *reinterpret_cast<uint32_t*>(S.Ah[b2] + op_off(row, kk)) = kk == DM ? 0x3F800000u : 0u;
        *reinterpret_cast<uint32_t*>(S.Al[b2] + op_off(row, kk)) = 0u;
    }
    for (int e = t; e < KMAX * DM * DM; e += TT) {
        const int k = e / (DM * DM), rc = e % (DM * DM), r = rc / DM, cc = rc % DM;
        S.W64[k * W64S + rc] = (k < K && r < D && cc < D) ? mv.W()[(int64_t)k * D * D + r * D + cc] : 0.0;
    }
    for (int e = t; e < KMAX * DM; e += TT) {
        const int k = e / DM, j = e % DM;
        S.mu64[k * (DM + 2) + j] = (k < K && j < D) ? mv.mu()[k * D + j] : 0.0;
    }
    for (int k = t; k < KMAX; k += TT) {
        S.ln64[k] = k < K ? mv.lognorm()[k] : 0.0;
        S.lp64[k] = k < K ? mv.logpi()[k] : -INFINITY;
        S.cst[k] = k < K ? (float)(mv.logpi()[k] + mv.lognorm()[k]) : -INFINITY;
        S.lnf[k] = k < K ? (float)mv.lognorm()[k] : -INFINITY;
    }
    for (int e = t; e < 3 * DM * TT; e += TT) (&S.xd[0][0])[e] = 0.0;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&S.tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        for (int b = 0; b < 3; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&S.xfull[b])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&S.mma_done)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = S.tmem;
    const uint64_t dBh = umma_desc(su32(S.Bh)), dBl = umma_desc(su32(S.Bl));
    const int sub = t >> 7, row = t & 127;
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    auto tile_of = [&](int64_t j) { return (int64_t)blockIdx.x + j * gridDim.x; };
    auto prefetch = [&](int64_t j) {  // two 128-row boxes per 256-event tile
        if (j >= my_tiles) return;
        const int s = (int)(j % 3);
        const int r0 = (int)(tile_of(j) * TT);
        mbar_expect_tx(su32(&S.xfull[s]), (uint32_t)(2 * D * 128 * 8));
        // box = 128 rows x D planes lands as [plane][128]; place the halves at [plane][0..127] / [plane][128..255]
        // by loading each 128-row half into its own [D][128] sub-buffer
        tma_load_2d(su32(&S.xd[s][0]), &xmap, r0, 0, su32(&S.xfull[s]));
        tma_load_2d(su32(&S.xd[s][DM * 128]), &xmap, r0 + 128, 0, su32(&S.xfull[s]));
    };
    // x of (tile buffer s, event t): half h = t/128 lives at xd[s][h*DM*128 + plane*128 + (t%128)]
    auto xat = [&](int s, int plane) -> double { return S.xd[s][sub * DM * 128 + plane * 128 + row]; };
    auto aprep_and_mma = [&](int64_t j) {
        const int s = (int)(j % 3);
        mbar_wait(su32(&S.xfull[s]), (uint32_t)((j / 3) & 1));
        const bool valid = tile_of(j) * TT + t < n;
#pragma unroll
        for (int jj = 0; jj < DM; jj += 4) {
            uint32_t h[4], l[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float f = (valid && jj + q < D) ? (float)(xat(s, jj + q) - S.c[jj + q]) : 0.f;
                h[q] = tf32(f);
                l[q] = tf32(f - __uint_as_float(h[q]));
            }
            *reinterpret_cast<uint4*>(S.Ah[sub] + op_off(row, jj)) = make_uint4(h[0], h[1], h[2], h[3]);
            *reinterpret_cast<uint4*>(S.Al[sub] + op_off(row, jj)) = make_uint4(l[0], l[1], l[2], l[3]);
        }
        proxy_fence();
        tc_fence_before();
        __syncthreads();
        if (t == 0) {
            tc_fence_after();
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {
                const uint32_t d = tmem + 128 * s2;
                const uint64_t dAh = umma_desc(su32(S.Ah[s2])), dAl = umma_desc(su32(S.Al[s2]));
#pragma unroll
                for (int ks = 0; ks < kKA / 8; ++ks) {
                    const uint64_t ko = (uint64_t)((2 * ks * kLBO) >> 4);
                    mma_tf32(d, dAh + ko, dBh + ko, ks > 0 ? 1u : 0u);
                    mma_tf32(d, dAh + ko, dBl + ko, 1u);
                    mma_tf32(d, dAl + ko, dBh + ko, 1u);
                }
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             su32(&S.mma_done))
                         : "memory");
        }
    };

    double ll_acc = 0.0, nflag = 0.0;
    if (my_tiles > 0) {
        if (t == 0) {
            prefetch(0);
            prefetch(1);
        }
        aprep_and_mma(0);
    }
    const unsigned lt_mask = (1u << lane) - 1u;
    const bool refine_all = getenv_refine_all;
    for (int64_t j = 0; j < my_tiles; ++j) {
        const int s = (int)(j % 3);
        const int64_t i = tile_of(j) * TT + t;
        const bool valid = i < n;
        mbar_wait(su32(&S.mma_done), (uint32_t)(j & 1));
        tc_fence_after();
        float w[KMAX], ln[KMAX];
        float m = -INFINITY, bl = -INFINITY;
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
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
            const float q = qa + qb;
            ln[k] = S.lnf[k] - 0.5f * q;
            w[k] = S.cst[k] - 0.5f * q;
            m = fmaxf(m, w[k]);
            bl = fmaxf(bl, ln[k]);
        }
        tc_fence_before();
        // candidates needing FP64: responsibility above 1e-6 (FP32 error then moves ll by
        // < 1e-6 * 1e-3 relative), or within FP32 rounding of either argmax
        unsigned cand = 0;
        const float ldf = (float)o.log_delta;
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
            const float tol = 1e-3f * (1.f + fabsf(w[k]));
            bool c;
            if (refine_all)
                c = w[k] >= m - 13.9f || ln[k] >= bl - tol;
            else  // decisive only: near-ties of either argmax, or the best density near log delta
                c = w[k] >= m - tol || ln[k] >= bl - tol ||
                    (ln[k] == bl && fabsf(bl - ldf) <= 1e-3f * (1.f + fabsf(ldf)));
            if (valid && k < K && c) cand |= 1u << k;
        }
        // deterministic component-major compaction of (event, component) candidates: the
        // warps of the refinement then mostly share one component, so its FP64 W rows and
        // mean are shared-memory broadcasts instead of up to 8 distinct rows per load
        unsigned kb[KMAX];
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
            kb[k] = __ballot_sync(0xffffffffu, (cand >> k) & 1u);
            if (lane == 0) S.wcnt[k * 8 + warp] = __popc(kb[k]);
        }
        __syncthreads();  // TMEM drained; A operand free; wcnt visible
        if (t == 0) {
            int a2 = 0;
            for (int k = 0; k < KMAX; ++k) {  // (component, warp) order; each component's
                for (int wv = 0; wv < 8; ++wv) {  // segment padded to an even length
                    S.woff[k * 8 + wv] = a2;
                    a2 += S.wcnt[k * 8 + wv];
                }
                if (a2 & 1) {
                    S.cev[a2] = 0xFFFFu;
                    S.ccomp[a2] = (uint8_t)k;
                    ++a2;
                }
            }
            S.ncand = a2;
            prefetch(j + 2);
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
            if ((cand >> k) & 1u) {
                const int pos = S.woff[k * 8 + warp] + __popc(kb[k] & lt_mask);
                S.cev[pos] = (uint16_t)t;
                S.ccomp[pos] = (uint8_t)k;
            }
        }
        __syncthreads();
        if (j + 1 < my_tiles) aprep_and_mma(j + 1);  // MMA(j+1) overlaps the FP64 refinement of tile j
        // FP64 refinement, two events of one component per thread (each W row load serves both)
        const int nc = S.ncand;
        for (int pidx = 2 * t; pidx < nc; pidx += 2 * TT) {
            const int k = S.ccomp[pidx];
            const int e0 = S.cev[pidx], e1r = S.cev[pidx + 1];
            const int e1 = e1r == 0xFFFF ? e0 : e1r;
            const double* Wk = S.W64 + k * W64S;
            const double* mk = S.mu64 + k * (DM + 2);
            double d0[DM], d1[DM];
#pragma unroll
            for (int jj = 0; jj < DM; ++jj) {
                d0[jj] = S.xd[s][(e0 >> 7) * DM * 128 + jj * 128 + (e0 & 127)] - mk[jj];
                d1[jj] = S.xd[s][(e1 >> 7) * DM * 128 + jj * 128 + (e1 & 127)] - mk[jj];
            }
            double q0 = 0.0, q1 = 0.0;
#pragma unroll
            for (int r = 0; r < DM; ++r) {
                double a0 = 0.0, a1 = 0.0;
#pragma unroll
                for (int jj = 0; jj <= r; jj += 2) {  // W rows read as double2 (upper triangle is zero)
                    const double2 wv = *reinterpret_cast<const double2*>(Wk + r * DM + jj);
                    a0 = fma(wv.x, d0[jj], a0);
                    a1 = fma(wv.x, d1[jj], a1);
                    if (jj + 1 <= r) {
                        a0 = fma(wv.y, d0[jj + 1], a0);
                        a1 = fma(wv.y, d1[jj + 1], a1);
                    }
                }
                q0 = fma(a0, a0, q0);
                q1 = fma(a1, a1, q1);
            }
            S.lnv[k * TT + e0] = S.ln64[k] - 0.5 * q0;
            if (e1r != 0xFFFF) S.lnv[k * TT + e1] = S.ln64[k] - 0.5 * q1;
        }
        __syncthreads();
        double mm = -INFINITY, bb = -INFINITY;
        int am = 0, ab = 0;
        double w64[KMAX];
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
            const double l = ((cand >> k) & 1u) ? S.lnv[k * TT + t] : (double)ln[k];
            w64[k] = S.lp64[k] + l;
            if (k >= K) continue;
            if (w64[k] > mm) { mm = w64[k]; am = k; }
            if (l > bb) { bb = l; ab = k; }
        }
        // log-sum-exp about the FP64 maximum: the max term is exactly 1, the others are summed
        // with FP32 exp (relative 1e-7 of a sum >= 1 -> ll error < 2e-7 absolute)
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
    }
    S.red[t] = ll_acc;
    __syncthreads();
    for (int st = TT / 2; st > 0; st >>= 1) {
        if (t < st) S.red[t] += S.red[t + st];
        __syncthreads();
    }
    if (t == 0) blocksum[2 * blockIdx.x] = S.red[0];
    __syncthreads();
    S.red[t] = nflag;
    __syncthreads();
    for (int st = TT / 2; st > 0; st >>= 1) {
        if (t < st) S.red[t] += S.red[t + st];
        __syncthreads();
    }
    if (t == 0) blocksum[2 * blockIdx.x + 1] = S.red[0];
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

bool score_tc_supported(int D, int K, const ScoreOut& o) {
    const char* e = getenv("ES_SCORE_KERNEL");
    if (e && e[0] == 's') return false;  // "simt" selects k_score_fast
    return D <= 16 && K <= KMAX && !o.gamma && !o.lnk;
}

void launch_score_tc(const CUtensorMap* xmap, int64_t n, int D, int K, const double* model, const double* center,
                     const ScoreOut& o, double* blocksum, int num_sms, int* nblk, cudaStream_t s, LaunchStats& ls) {
    *nblk = num_sms;
    const size_t smem = sizeof(SmemS) + 1024;
    static bool a = false;
    if (!a) {
        cudaFuncSetAttribute(k_score_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        a = true;
    }
    static int refine_all = -1;
    if (refine_all < 0) {
        const char* e = getenv("ES_SCORE_REFINE");
        refine_all = (e && e[0] == 'm') ? 0 : 1;  // ES_SCORE_REFINE=min: decisive components only
    }
    k_score_tc<<<num_sms, TT, smem, s>>>(*xmap, n, D, K, model, center, o, blocksum, refine_all);
    ++ls.launches;
}

}  // namespace es
