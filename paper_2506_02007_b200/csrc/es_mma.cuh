// es_mma.cuh — tcgen05 building blocks shared by the fused EM pass (es_em_mma.cu) and
// the scoring pass (es_score_mma.cu): kind::f16 MMA issue (operands in shared memory or
// A in TMEM), UMMA descriptors, TMEM loads/stores, mbarriers, fp16 packing, and the
// E-step operand staging  U = W' x^ + b'  (W'/t_k and b'/t_k split into fp16 hi + lo).
#pragma once
#include <cmath>
#include <cstdint>
#include <cuda_fp16.h>

#include "es_layout.h"
#include "es_tc.cuh"

namespace es {
namespace mma {

using namespace tc;

constexpr int DM = 16, KMAX = 8, TM = 128;
constexpr uint32_t OPB = 4096;  // one 128 x 16 fp16 K-major operand

// kind::f16 instruction descriptor: D = F32, A = B = F16, N>>3 @17, M>>4 @24,
// transpose (MN-major) A @15, B @16.
constexpr uint32_t idesc_f16(int M, int N, int mn) {
    return (1u << 4) | ((uint32_t)mn << 15) | ((uint32_t)mn << 16) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}
constexpr uint32_t kIdescE = idesc_f16(128, 128, 0);

// -c xs per feature (kernel parameter: constant-bank operands, no shared-memory loads)
struct NegCx {
    double v[DM];
};
struct NegCxF {  // the same rounded to FP32 (FP32-pipe conversion)
    float v[DM];
};

// byte offset of (row, k) in a K-major 128 x 16 fp16 operand (SWIZZLE_NONE core matrices)
__device__ __forceinline__ uint32_t kmaj(int row, int k) {
    return (uint32_t)((row >> 3) * 256 + (k >> 3) * 128 + (row & 7) * 16 + (k & 7) * 2);
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}
__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_f16_ta(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}
__device__ __forceinline__ uint64_t sub2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ float ex2(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float lg2(float x) {
    float r;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ void commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count));
}
__device__ __forceinline__ void arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* b, uint32_t parity) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(su32(b)), "r"(parity)
        : "memory");
    return done != 0;
}
__device__ __forceinline__ void named_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
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
__device__ __forceinline__ void tmem_ld2(uint32_t taddr, float& a, float& b) {
    uint32_t r0, r1;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(taddr) : "memory");
    a = __uint_as_float(r0);
    b = __uint_as_float(r1);
}
__device__ __forceinline__ __half2 u2h(uint32_t u) { return *reinterpret_cast<__half2*>(&u); }
// round-to-nearest, saturating fp32 pair -> fp16x2 (lo in the low half)
__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
// Compensated FP32 accumulation of two lanes, (hi, lo) += x (Fast2Sum: the rounding error
// of hi + x is exact while |hi| >= |x|, which holds once a few tiles are in): ~44-bit
// accumulation on the FP32 pipe instead of F2F + DADD on the much narrower FP64 pipe.
__device__ __forceinline__ void cacc2(uint64_t& hi, uint64_t& lo, uint64_t x) {
    const uint64_t s2 = add2(hi, x);
    lo = add2(lo, sub2(x, sub2(s2, hi)));
    hi = s2;
}
__device__ __forceinline__ void cacc(float& hi, float& lo, float x) {
    const float s = hi + x;
    lo += x - (s - hi);
    hi = s;
}
__device__ __forceinline__ double cval(uint64_t hi, uint64_t lo, int h) {
    float a, b, c, d;
    unpack2(hi, a, b);
    unpack2(lo, c, d);
    return h ? (double)b + (double)d : (double)a + (double)c;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}


// E-step operands for components k < K (all threads of the CTA; S.c must hold the
// centre and be visible): bw[0|1] = fp16 hi | lo of W'/t_k (W' = W / xs, K-major rows
// (k, a)), bb = b'/t_k hi, lo in K columns 0, 1 (b' = -W (mu - c)); cst = log pi + lognorm,
// lnf = lognorm, hq = t_k^2 / 2.  t_k (a power of two) puts each component's largest |entry|
// into (2^12, 2^13], so the fp16 lo parts of all but negligible entries are normal numbers.
__device__ inline void stage_estep(const ModelView& mv, int K, int D, const double* __restrict__ center,
                                   const double* cs, double xs, unsigned char* bw0, unsigned char* bw1,
                                   unsigned char* bb, float* cstv, float* lnfv, float* hqv, float* tkv, int t,
                                   int nthr) {
    if (t < KMAX) {
        const int k = t;
        float cst = -INFINITY, lnf = -INFINITY, tk = 1.f;
        if (k < K) {
            cst = (float)(mv.logpi()[k] + mv.lognorm()[k]);
            lnf = (float)mv.lognorm()[k];
            double m = 0.0;
            const double* W = mv.W() + (int64_t)k * D * D;
            for (int a = 0; a < D; ++a) {
                double b = 0.0;
                for (int f = 0; f <= a; ++f) {
                    m = fmax(m, fabs(W[a * D + f] / xs));
                    b = fma(W[a * D + f], mv.mu()[k * D + f] - center[f], b);
                }
                m = fmax(m, fabs(b));
            }
            if (m > 0.0) tk = (float)exp2(ceil(log2(m)) - 13.0);
        }
        cstv[k] = cst;
        if (lnfv) lnfv[k] = lnf;
        hqv[k] = 0.5f * tk * tk;
        tkv[k] = tk;
    }
    __syncthreads();
    for (int e = t; e < TM * DM; e += nthr) {
        const int row = e / DM, f = e % DM, k = row / DM, a = row % DM;
        double w = 0.0, b = 0.0;
        if (k < K && a < D) {
            const double* Wr = mv.W() + (int64_t)k * D * D + (int64_t)a * D;
            const double inv_t = 1.0 / (double)tkv[k];
            if (f <= a) w = Wr[f] / xs * inv_t;
            if (f < 2) {
                double s = 0.0;
                for (int q = 0; q <= a; ++q) s = fma(Wr[q], mv.mu()[k * D + q] - cs[q], s);
                b = -s * inv_t;
            }
        }
        const __half wh = __double2half(w);
        const __half wl = __double2half(w - (double)__half2float(wh));
        *reinterpret_cast<__half*>(bw0 + kmaj(row, f)) = wh;
        *reinterpret_cast<__half*>(bw1 + kmaj(row, f)) = wl;
        // b' rounded once to FP32 and split exactly into three fp16 parts (11 + 11 + 2 bits):
        // the bias dispatch, issued first, then leaves exactly fp32(b') in the accumulator,
        // and the whitening dispatches add onto it, so the running sums stay of the size of
        // U instead of |W' x^| ~ |b'| (FP32 truncation ~1 ulp of the running sum per dispatch)
        const float b32 = (float)b;
        const __half bh = __float2half_rn(b32);
        const float r1 = b32 - __half2float(bh);
        const __half bm = __float2half_rn(r1);
        const __half bl = __float2half_rn(r1 - __half2float(bm));
        *reinterpret_cast<__half*>(bb + kmaj(row, f)) =
            f == 0 ? bh : (f == 1 ? bm : (f == 2 ? bl : __half(0.f)));
    }
}

}  // namespace mma
}  // namespace es
