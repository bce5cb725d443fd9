// es_ws.cu — warp-specialized fused EM pass (default for D <= 16, K <= 8).
//
// One CTA per SM, 12 warps in three warpgroups:
//   WG0 (warps 0-3, 104 regs): producer.  Per 128-event tile: waits for the
//       bulk-prefetched FP64 tile, forms x' = x - c, writes the TF32 hi/lo UMMA
//       operand and FP32 rows, issues 9 tcgen05.mma (3xTF32, K=24) into one of
//       two TMEM accumulators, then runs the epilogue of the previous tile: one
//       TMEM row per thread (= event), log-sum-exp over K, responsibilities,
//       ballot-compacted per-component gamma lists into a ring slot.
//   WG1-2 (warps 4-11, 200 regs): consumers.  Warp 4+k owns component k's
//       sufficient statistics in registers (packed FP32 pairs, FFMA2), walks its
//       gamma list of every tile, and flushes into FP64 shared accumulators every
//       64 tiles.
// Producer and consumers meet only through mbarriers on a 4-slot ring (no
// CTA-wide barrier in the steady state), so the consumer for a broad
// component no longer stalls every other warp each tile.  setmaxnreg moves
// registers from the producer to the consumers.
#include <cmath>
#include <cstdlib>
#include <cudaTypedefs.h>

#include "es_kernels.h"
#include "es_tc.cuh"

namespace es {

namespace {

using namespace tc;

constexpr int DM = 16;
constexpr int KMAX = 8;
constexpr int TM = 128;            // events per tile (= UMMA M)
constexpr int NPROD = 128;         // producer threads
constexpr int NTHR = 384;          // 4 producer + 8 consumer warps
constexpr int XS = 3;              // X prefetch stages
constexpr int RS = 4;              // producer -> consumer ring slots
constexpr int XR = 20;             // FP32 row stride (16 + pad)
constexpr int NS = 1 + DM + DM * (DM + 1) / 2;
constexpr int NP = 64, NSG = 8;    // Gram pairs / singles (see k_em_tc)

struct Ring {                      // one producer -> consumer slot
    float xr[TM * XR];             // x' rows (FP32)
    float lg[KMAX * TM];           // gamma sub-lists: [k][producer warp][32]
    uint8_t lt[KMAX * TM];         // event index sub-lists
    int cnt[KMAX * 4];             // sub-list lengths [k][producer warp]
};

struct Smem {
    unsigned char Bh[kOpBytes], Bl[kOpBytes];          // 2 x 12 KB, 16B-aligned core matrices
    unsigned char Ah[2][kOpBytes], Al[2][kOpBytes];    // double-buffered A operand
    double xd[XS][DM * TM];                            // bulk-prefetched FP64 tiles (planar)
    Ring ring[RS];
    double acc[KMAX * NS];                             // FP64 statistics
    double red[NPROD];
    double c[DM];
    float nmu[KMAX * DM];                              // -mu'_k
    float cst[KMAX];
    float thr[KMAX];
    unsigned bal[4 * KMAX];
    uint64_t xfull[XS], mma_done[2], full[RS], empty[RS];
    uint32_t tmem;
};

__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void prod_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

}  // namespace

__global__ void __launch_bounds__(NTHR, 1) k_em_ws(const __grid_constant__ CUtensorMap xmap, int64_t n, int D, int K,
                                                    const double* __restrict__ model,
                                                    const double* __restrict__ center, double* __restrict__ partial) {
    extern __shared__ __align__(1024) unsigned char smraw[];
    Smem& S = *reinterpret_cast<Smem*>(smraw);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    ModelView mv{K, D, const_cast<double*>(model)};
    const int64_t ntiles = (n + TM - 1) / TM;
    const int64_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    // ------------------------------------------------------------ staging
    for (int j = t; j < DM; j += NTHR) S.c[j] = j < D ? center[j] : 0.0;
    __syncthreads();
    for (int e = t; e < kTileRows * kKA; e += NTHR) {
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
    for (int e = t; e < 2 * kTileRows * (kKA - DM); e += NTHR) {
        const int b2 = e / (kTileRows * (kKA - DM)), rr = e % (kTileRows * (kKA - DM));
        const int row = rr / (kKA - DM), kk = DM + rr % (kKA - DM);
        *reinterpret_cast<uint32_t*>(S.Ah[b2] + op_off(row, kk)) = kk == DM ? 0x3F800000u : 0u;
        *reinterpret_cast<uint32_t*>(S.Al[b2] + op_off(row, kk)) = 0u;
    }
    for (int e = t; e < KMAX * DM; e += NTHR) {
        const int k = e / DM, j = e % DM;
        S.nmu[e] = (k < K && j < D) ? -(float)(mv.mu()[k * D + j] - S.c[j]) : 0.f;
    }
    for (int k = t; k < KMAX; k += NTHR) {
        S.cst[k] = k < K ? (float)(mv.logpi()[k] + mv.lognorm()[k]) : -INFINITY;
        // certified pruning: skipped mass <= 1e-9 N_k
        S.thr[k] = k < K ? fmaxf((float)(1e-9 * mv.pi()[k]), 1e-30f) : INFINITY;
    }
    for (int e = t; e < KMAX * NS; e += NTHR) S.acc[e] = 0.0;
    for (int e = t; e < XS * DM * TM; e += NTHR) (&S.xd[0][0])[e] = 0.0;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&S.tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        for (int i = 0; i < XS; ++i) mbar_init(&S.xfull[i], 1);
        for (int i = 0; i < 2; ++i) mbar_init(&S.mma_done[i], 1);
        for (int i = 0; i < RS; ++i) {
            mbar_init(&S.full[i], 4);  // one arrival per producer warp
            mbar_init(&S.empty[i], 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = S.tmem;

    if (warp < 4) {
        // ============================================================ producer
        asm volatile("setmaxnreg.dec.sync.aligned.u32 104;\n" ::: "memory");
        const int p = t;  // tile row / TMEM lane
        const uint32_t lane_base = (uint32_t)(32 * warp) << 16;
        const unsigned lt_mask = (1u << lane) - 1u;
        const uint64_t dBh = umma_desc(su32(S.Bh)), dBl = umma_desc(su32(S.Bl));
        double ll_acc = 0.0;
        auto tile_of = [&](int64_t j) { return (int64_t)blockIdx.x + j * gridDim.x; };
        // one TMA tensor copy per tile: box = 128 rows x D planes (rows past n are zero-filled)
        auto prefetch = [&](int64_t j) {
            if (j >= my_tiles) return;
            const int s = (int)(j % XS);
            mbar_expect_tx(su32(&S.xfull[s]), (uint32_t)(D * TM * 8));
            tma_load_2d(su32(&S.xd[s][0]), &xmap, (int)(tile_of(j) * TM), 0, su32(&S.xfull[s]));
        };
        if (p == 0)
            for (int j = 0; j < XS; ++j) prefetch(j);

        auto epilogue = [&](int64_t j) {
            const int64_t tile = tile_of(j);
            const bool valid = tile * TM + p < n;
            const int ab = (int)(j & 1);
            mbar_wait(su32(&S.mma_done[ab]), (uint32_t)((j >> 1) & 1));
            tc_fence_after();
            float w[KMAX];
            float m = -INFINITY;
#pragma unroll
            for (int k = 0; k < KMAX; ++k) {
                float u[16];
                tmem_ld16(tmem + lane_base + 128 * ab + 16 * k, u);
                tmem_wait_ld();
                uint64_t q2 = 0;
#pragma unroll
                for (int r = 0; r < 16; r += 2) {
                    const uint64_t uu = pack2(u[r], u[r + 1]);
                    ffma2(q2, uu, uu);
                }
                float qa, qb;
                unpack2(q2, qa, qb);
                w[k] = S.cst[k] - 0.5f * (qa + qb);
                m = fmaxf(m, w[k]);
            }
            tc_fence_before();
            float ssum = 0.f;
#pragma unroll
            for (int k = 0; k < KMAX; ++k) ssum += __expf(w[k] - m);
            const float ll = m + __logf(ssum);
            if (valid) ll_acc += (double)ll;
            Ring& R = S.ring[j % RS];
            // per-warp sub-lists: no cross-warp prefix, no producer barrier
#pragma unroll
            for (int k = 0; k < KMAX; ++k) {
                const float gk = __expf(w[k] - ll);
                const unsigned b = __ballot_sync(0xffffffffu, valid && gk >= S.thr[k]);
                if ((b >> lane) & 1u) {
                    const int pos = (k * 4 + warp) * 32 + __popc(b & lt_mask);
                    R.lt[pos] = (uint8_t)p;
                    R.lg[pos] = gk;
                }
                if (lane == 0) R.cnt[k * 4 + warp] = __popc(b);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.full[j % RS]);
        };

        for (int64_t j = 0; j < my_tiles; ++j) {
            const int64_t tile = tile_of(j);
            const int64_t i = tile * TM + p;
            const bool valid = i < n;
            const int xs = (int)(j % XS);
            const int ab = (int)(j & 1);
            Ring& R = S.ring[j % RS];
            // ring slot j%RS must have been released by the consumers (tile j-RS)
            if (j >= RS) mbar_wait_sleep(su32(&S.empty[j % RS]), (uint32_t)(((j / RS) - 1) & 1));
            mbar_wait(su32(&S.xfull[xs]), (uint32_t)((j / XS) & 1));
            unsigned char* ah = S.Ah[ab];
            unsigned char* al = S.Al[ab];
            float* xr = R.xr + p * XR;
#pragma unroll
            for (int jj = 0; jj < DM; jj += 4) {
                float f[4];
                uint32_t h[4], l[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const double xv = S.xd[xs][(jj + q) * TM + p];
                    f[q] = (valid && jj + q < D) ? (float)(xv - S.c[jj + q]) : 0.f;
                    h[q] = tf32(f[q]);
                    l[q] = tf32(f[q] - __uint_as_float(h[q]));
                }
                *reinterpret_cast<float4*>(xr + jj) = make_float4(f[0], f[1], f[2], f[3]);
                *reinterpret_cast<uint4*>(ah + op_off(p, jj)) = make_uint4(h[0], h[1], h[2], h[3]);
                *reinterpret_cast<uint4*>(al + op_off(p, jj)) = make_uint4(l[0], l[1], l[2], l[3]);
            }
            proxy_fence();
            tc_fence_before();
            prod_sync();  // operand + rows complete; X stage xs consumed; TMEM buffer ab drained (epilogue j-2)
            if (p == 0) {
                prefetch(j + XS);
                tc_fence_after();
                const uint32_t d = tmem + 128 * ab;
                const uint64_t dAh = umma_desc(su32(ah)), dAl = umma_desc(su32(al));
#pragma unroll
                for (int ks = 0; ks < kKA / 8; ++ks) {
                    const uint64_t ko = (uint64_t)((2 * ks * kLBO) >> 4);
                    mma_tf32(d, dAh + ko, dBh + ko, ks > 0 ? 1u : 0u);
                    mma_tf32(d, dAh + ko, dBl + ko, 1u);
                    mma_tf32(d, dAl + ko, dBh + ko, 1u);
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 su32(&S.mma_done[ab]))
                             : "memory");
            }
            if (j >= 1) epilogue(j - 1);
        }
        if (my_tiles > 0) epilogue(my_tiles - 1);
        S.red[p] = ll_acc;
    } else {
        // ============================================================ consumers
        asm volatile("setmaxnreg.inc.sync.aligned.u32 200;\n" ::: "memory");
        const int kw = warp - 4;
        const bool mact = kw < K;
        uint64_t accp[NP];
        float accs[NSG];
        uint64_t acc1[DM / 2];
        float accn = 0.f;
#pragma unroll
        for (int j = 0; j < NP; ++j) accp[j] = 0;
#pragma unroll
        for (int j = 0; j < NSG; ++j) accs[j] = 0.f;
#pragma unroll
        for (int j = 0; j < DM / 2; ++j) acc1[j] = 0;
        auto flush1 = [&](float v, int idx) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if ((idx & 31) == lane) S.acc[kw * NS + idx] += (double)v;
        };
        auto flush = [&]() {
            flush1(accn, 0);
            accn = 0.f;
#pragma unroll
            for (int mm = 0; mm < DM / 2; ++mm) {
                float lo, hi;
                unpack2(acc1[mm], lo, hi);
                flush1(lo, 1 + 2 * mm);
                flush1(hi, 2 + 2 * mm);
                acc1[mm] = 0;
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
                for (int mm = (a + 1) / 2; mm < DM / 2; ++mm) {
                    float lo, hi;
                    unpack2(accp[ip], lo, hi);
                    flush1(lo, base + (2 * mm - a));
                    flush1(hi, base + (2 * mm + 1 - a));
                    accp[ip++] = 0;
                }
            }
        };
        const uint64_t* nmu2 = reinterpret_cast<const uint64_t*>(S.nmu + (mact ? kw : 0) * DM);
        int64_t j = 0;
        while (j < my_tiles) {
            // one flush site per super-tile of 64 tiles (FP32 partials stay short)
            for (int st = 0; st < 64 && j < my_tiles; ++st, ++j) {
                mbar_wait_sleep(su32(&S.full[j % RS]), (uint32_t)((j / RS) & 1));
                const Ring& R = S.ring[j % RS];
                if (mact) {
                    // the 4 producer-warp sub-lists, walked as one dense list
                    const int c0 = R.cnt[kw * 4 + 0], c1 = R.cnt[kw * 4 + 1], c2 = R.cnt[kw * 4 + 2];
                    const int p1 = c0, p2 = c0 + c1, p3 = c0 + c1 + c2;
                    const int nk = p3 + R.cnt[kw * 4 + 3];
                    for (int e0 = 0; e0 < nk; e0 += 32) {
                        const int e = e0 + lane;
                        const bool ve = e < nk;
                        // branch-free (sub-list, offset) of dense index e
                        const int b1 = e >= p1, b2 = e >= p2, b3 = e >= p3;
                        const int ix = (kw * 4 + b1 + b2 + b3) * 32 + e - (b1 * c0 + b2 * c1 + b3 * c2);
                        const int tt = ve ? R.lt[ix] : 0;
                        const float gg = ve ? R.lg[ix] : 0.f;
                        const float4* xr4 = reinterpret_cast<const float4*>(R.xr + tt * XR);
                        uint64_t d2[DM / 2];
#pragma unroll
                        for (int q = 0; q < DM / 4; ++q) {
                            const float4 v = xr4[q];
                            d2[2 * q] = add2(pack2(v.x, v.y), nmu2[2 * q]);
                            d2[2 * q + 1] = add2(pack2(v.z, v.w), nmu2[2 * q + 1]);
                        }
                        accn += gg;
                        const uint64_t g2 = pack2(gg, gg);
#pragma unroll
                        for (int mm = 0; mm < DM / 2; ++mm) ffma2(acc1[mm], g2, d2[mm]);
                        int ip = 0, is = 0;
#pragma unroll
                        for (int a = 0; a < DM; ++a) {
                            float dl, dh;
                            unpack2(d2[a / 2], dl, dh);
                            const float ga = gg * ((a & 1) ? dh : dl);
                            const uint64_t ga2 = pack2(ga, ga);
                            if (a & 1) {
                                accs[is] = fmaf(ga, dh, accs[is]);
                                ++is;
                            }
#pragma unroll
                            for (int mm = (a + 1) / 2; mm < DM / 2; ++mm) {
                                ffma2(accp[ip], ga2, d2[mm]);
                                ++ip;
                            }
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&S.empty[j % RS]);
            }
            if (mact) flush();
        }
    }
    __syncthreads();
    // ---------------------------------------------------------------- output
    const int SK = stat_k(D), NE = K * SK;
    double* myp = partial + (int64_t)blockIdx.x * (NE + 1);
    for (int e = t; e < NE; e += NTHR) {
        const int k = e / SK, r = e % SK;
        int jx;
        if (r <= D) {
            jx = r;
        } else {
            int pp = r - 1 - D, a = 0;
            while (pp >= D - a) {
                pp -= D - a;
                ++a;
            }
            const int b = a + pp;
            jx = 1 + DM + (a * DM - (a * (a - 1)) / 2 + (b - a));
        }
        myp[e] = S.acc[k * NS + jx];
    }
    if (t == 0) {
        double s = 0.0;
        for (int q = 0; q < NPROD; ++q) s += S.red[q];
        myp[NE] = s;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

bool em_ws_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("ES_EM_KERNEL");
        v = (!e || e[0] == 'w') ? 1 : 0;  // default: warp-specialized; "tc" / "simt" select the others
    }
    return v == 1;
}

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

void launch_em_ws(const CUtensorMap* xmap, int64_t n, int D, int K, const double* model, const double* center,
                  double* partial, int num_sms, int* nblk, cudaStream_t s, LaunchStats& ls) {
    *nblk = num_sms;
    const size_t smem = sizeof(Smem) + 1024;
    static bool a = false;
    if (!a) {
        cudaFuncSetAttribute(k_em_ws, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        a = true;
    }
    k_em_ws<<<num_sms, NTHR, smem, s>>>(*xmap, n, D, K, model, center, partial);
    ++ls.launches;
}

}  // namespace es
