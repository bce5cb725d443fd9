// umma_probe.cu — standalone sm_100a probe for the tcgen05 shapes the EM pass uses.
//   1. kind::f16, MN-major A and B (the M-step Gram: D = P^T P over K = 128 events,
//      M = 128, N = 136), both LBO/SBO conventions, checked against a host FP64 GEMM;
//   2. kind::f16, K-major A and B (E-step: M = N = 128, K = 16), checked likewise;
//   3. dispatch throughput: cycles per (4 x N128 + 8 x N136) K=16 dispatch group,
//      with and without concurrent STS.128 traffic from 4 warps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o umma_probe umma_probe.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}
// kind::f16: D=F32 (bits 4-5 = 1), A=B=F16 (0), a_major bit 15, b_major bit 16, N>>3 @17, M>>4 @24
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N, int amn, int bmn) {
    return (1u << 4) | ((uint32_t)amn << 15) | ((uint32_t)bmn << 16) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}\n"
            : "=r"(done)
            : "r"(su32(bar)), "r"(phase)
            : "memory");
    }
}
__device__ __forceinline__ void ld32(uint32_t taddr, float* v) {
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
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
}

constexpr int KE = 128, NM = 136;

// mode 0: MN-major gram (LBO = K-group stride 128, SBO = MN-group stride 2048)
// mode 1: MN-major gram with the two offsets exchanged in the descriptor
// mode 2: K-major E-step, A[128x16] x B[128x16]
__global__ void k_check(const __half* P, const __half* A, const __half* B, float* out, int mode) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int t = threadIdx.x, warp = t >> 5;
    unsigned char* buf = sm;
    if (mode < 2) {
        for (int e = t; e < KE * NM; e += blockDim.x) {
            const int i = e / NM, m = e % NM;
            const uint32_t off = (m / 8) * 2048 + (i / 8) * 128 + (i % 8) * 16 + (m % 8) * 2;
            *reinterpret_cast<__half*>(buf + off) = P[e];
        }
    } else {
        for (int e = t; e < 128 * 16; e += blockDim.x) {
            const int r = e / 16, k = e % 16;
            const uint32_t off = (r / 8) * 256 + (k / 8) * 128 + (r % 8) * 16 + (k % 8) * 2;
            *reinterpret_cast<__half*>(buf + off) = A[e];
            *reinterpret_cast<__half*>(buf + 4096 + off) = B[e];
        }
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tbase;
    if (t == 0) {
        if (mode < 2) {
            const uint32_t lbo = mode == 0 ? 128 : 2048, sbo = mode == 0 ? 2048 : 128;
            for (int ks = 0; ks < KE / 16; ++ks) {
                const uint64_t d = desc(su32(buf) + ks * 256, lbo, sbo);
                mma_f16(tm, d, d, idesc_f16(128, NM, 1, 1), ks > 0);
            }
        } else {
            mma_f16(tm, desc(su32(buf), 128, 256), desc(su32(buf + 4096), 128, 256), idesc_f16(128, 128, 0, 0), 0);
        }
        commit(&bar);
    }
    mbar_wait(&bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int ncol = mode < 2 ? 160 : 128;
    for (int c0 = 0; c0 < ncol; c0 += 32) {
        float v[32];
        ld32(tm + ((uint32_t)(32 * warp) << 16) + c0, v);
        for (int j = 0; j < 32; ++j)
            if (c0 + j < (mode < 2 ? NM : 128)) out[t * 160 + c0 + j] = v[j];
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}

// throughput: thread 0 issues R groups; warps 1-4 optionally stream STS.128 (34 KB per group)
__global__ void k_rate(int R, int which, int sts, long long* cyc) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar[2];
    __shared__ uint32_t tbase;
    __shared__ volatile int stop;
    const int t = threadIdx.x, warp = t >> 5;
    for (int e = t; e < (96 * 1024) / 16; e += blockDim.x) reinterpret_cast<uint4*>(sm)[e] = make_uint4(0x3c003c00u, 0, 0, 0);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        stop = 0;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[0])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tbase;
    if (t == 0) {
        const long long c0 = clock64();
        const uint32_t ebase = su32(sm), mbase = su32(sm + 16384);
        for (int r = 0; r < R; ++r) {
            if (which & 1)
                for (int q = 0; q < 4; ++q)
                    mma_f16(tm + 128 * (r & 1), desc(ebase + q * 4096, 128, 256), desc(ebase + 8192, 128, 256),
                            idesc_f16(128, 128, 0, 0), q > 0);
            if (which & 2)
                for (int ks = 0; ks < 8; ++ks) {
                    const uint64_t d = desc(mbase + ks * 256, 128, 2048);
                    mma_f16(tm + 256, d, d, idesc_f16(128, NM, 1, 1), 1);
                }
        }
        commit(&bar[0]);
        mbar_wait(&bar[0], 0);
        cyc[blockIdx.x] = clock64() - c0;
        stop = 1;
    } else if (sts && warp >= 1 && warp <= 4) {
        // 128 threads x 17 STS.128 per "group" into a 34 KB region (separate from the MMA operands)
        uint4* dst = reinterpret_cast<uint4*>(sm + 64 * 1024);
        const uint4 v = make_uint4(t, t, t, t);
        int it = 0;
        while (!stop) {
#pragma unroll
            for (int q = 0; q < 17; ++q) dst[(q * 128 + (t - 32)) & 2047] = v;
            ++it;
        }
        if (t == 32) cyc[gridDim.x + blockIdx.x] = it;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}


// accumulation rounding: D += A B over R dispatches of K=16 (all-positive fp16); host compares with exact sums
__global__ void k_accum(const __half* A, const __half* B, int R, float* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int t = threadIdx.x, warp = t >> 5;
    for (int e = t; e < R * 128 * 16; e += blockDim.x) {
        const int r = e / 2048, row = (e / 16) % 128, k = e % 16;
        const uint32_t off = r * 4096 + (row / 8) * 256 + (k / 8) * 128 + (row % 8) * 16 + (k % 8) * 2;
        *reinterpret_cast<__half*>(sm + off) = A[e];
        *reinterpret_cast<__half*>(sm + R * 4096 + off) = B[e];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tbase;
    if (t == 0) {
        for (int r = 0; r < R; ++r)
            mma_f16(tm, desc(su32(sm) + r * 4096, 128, 256), desc(su32(sm) + R * 4096 + r * 4096, 128, 256),
                    idesc_f16(128, 128, 0, 0), r > 0);
        commit(&bar);
    }
    mbar_wait(&bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (int c0 = 0; c0 < 128; c0 += 32) {
        float v[32];
        ld32(tm + ((uint32_t)(32 * warp) << 16) + c0, v);
        for (int j = 0; j < 32; ++j) out[t * 128 + c0 + j] = v[j];
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm));
}


// A from TMEM: thread m writes row m of A (16 fp16 = 8 x 32-bit columns) with tcgen05.st, B K-major in smem
__global__ void k_atmem(const __half* A, const __half* B, float* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int t = threadIdx.x, warp = t >> 5;
    for (int e = t; e < 128 * 16; e += blockDim.x) {
        const int r = e / 16, k = e % 16;
        const uint32_t off = (r / 8) * 256 + (k / 8) * 128 + (r % 8) * 16 + (k % 8) * 2;
        *reinterpret_cast<__half*>(sm + off) = B[e];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tbase;
    {   // row t of A -> TMEM lane t, columns 160..167
        uint32_t r[8];
        for (int c = 0; c < 8; ++c) {
            __half2 h = __halves2half2(A[t * 16 + 2 * c], A[t * 16 + 2 * c + 1]);
            r[c] = *reinterpret_cast<uint32_t*>(&h);
        }
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                         tm + ((uint32_t)(32 * warp) << 16) + 160),
                     "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                     : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (t == 0) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tm), "r"(tm + 160),
            "l"(desc(su32(sm), 128, 256)), "r"(idesc_f16(128, 128, 0, 0)), "r"(0));
        commit(&bar);
    }
    mbar_wait(&bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (int c0 = 0; c0 < 128; c0 += 32) {
        float v[32];
        ld32(tm + ((uint32_t)(32 * warp) << 16) + c0, v);
        for (int j = 0; j < 32; ++j) out[t * 128 + c0 + j] = v[j];
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);    \
            exit(1);                                                                           \
        }                                                                                      \
    } while (0)

int main() {
    srand(1);
    std::vector<__half> P(KE * NM), A(128 * 16), B(128 * 16);
    std::vector<double> Pd(KE * NM), Ad(128 * 16), Bd(128 * 16);
    for (int e = 0; e < KE * NM; ++e) {
        P[e] = __float2half((float)(rand() % 2001 - 1000) / 256.f);
        Pd[e] = __half2float(P[e]);
    }
    for (int e = 0; e < 128 * 16; ++e) {
        A[e] = __float2half((float)(rand() % 2001 - 1000) / 256.f);
        B[e] = __float2half((float)(rand() % 2001 - 1000) / 256.f);
        Ad[e] = __half2float(A[e]);
        Bd[e] = __half2float(B[e]);
    }
    __half *dP, *dA, *dB;
    float* dout;
    CK(cudaMalloc(&dP, P.size() * 2));
    CK(cudaMalloc(&dA, A.size() * 2));
    CK(cudaMalloc(&dB, B.size() * 2));
    CK(cudaMalloc(&dout, 128 * 160 * 4));
    CK(cudaMemcpy(dP, P.data(), P.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaFuncSetAttribute(k_check, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    std::vector<float> out(128 * 160);
    for (int mode = 0; mode < 3; ++mode) {
        CK(cudaMemset(dout, 0, 128 * 160 * 4));
        k_check<<<1, 128, 64 * 1024>>>(dP, dA, dB, dout, mode);
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost));
        double maxerr = 0, maxref = 0;
        const int nc = mode < 2 ? NM : 128;
        for (int m = 0; m < 128; ++m)
            for (int n = 0; n < nc; ++n) {
                double ref = 0;
                if (mode < 2)
                    for (int i = 0; i < KE; ++i) ref += Pd[i * NM + m] * Pd[i * NM + n];
                else
                    for (int k = 0; k < 16; ++k) ref += Ad[m * 16 + k] * Bd[n * 16 + k];
                maxerr = fmax(maxerr, fabs(ref - out[m * 160 + n]));
                maxref = fmax(maxref, fabs(ref));
            }
        printf("check mode %d: max|err| %.3e  max|ref| %.3e  -> %s\n", mode, maxerr, maxref,
               maxerr <= 1e-5 * maxref ? "OK" : "MISMATCH");
    }


    {   // A from TMEM check
        float* d3;
        CK(cudaMalloc(&d3, 128 * 128 * 4));
        CK(cudaFuncSetAttribute(k_atmem, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192));
        k_atmem<<<1, 128, 8192>>>(dA, dB, d3);
        CK(cudaDeviceSynchronize());
        std::vector<float> o(128 * 128);
        CK(cudaMemcpy(o.data(), d3, o.size() * 4, cudaMemcpyDeviceToHost));
        double maxerr = 0;
        for (int m = 0; m < 128; ++m)
            for (int n = 0; n < 128; ++n) {
                double ref = 0;
                for (int k = 0; k < 16; ++k) ref += Ad[m * 16 + k] * Bd[n * 16 + k];
                maxerr = fmax(maxerr, fabs(ref - o[m * 128 + n]));
            }
        printf("A-in-TMEM check: max|err| %.3e -> %s\n", maxerr, maxerr < 1e-3 ? "OK" : "MISMATCH");
    }
    for (int mode = 0; mode < 3; ++mode) {   // accumulation rounding: all +, all -, mixed signs
        const int R = 12;
        std::vector<__half> a(R * 2048), b(R * 2048);
        std::vector<double> ad(R * 2048), bd(R * 2048);
        for (int e = 0; e < R * 2048; ++e) {
            const float sa = mode == 1 ? -1.f : 1.f;
            const float sb = mode == 2 ? ((rand() & 1) ? -1.f : 1.f) : 1.f;
            a[e] = __float2half(sa * (0.5f + (float)(rand() % 100000) / 100000.f));
            b[e] = __float2half(sb * (0.5f + (float)(rand() % 100000) / 100000.f * (1.f + (e % 7))));
            ad[e] = __half2float(a[e]);
            bd[e] = __half2float(b[e]);
        }
        __half *da, *db;
        float* dout2;
        CK(cudaMalloc(&da, a.size() * 2));
        CK(cudaMalloc(&db, b.size() * 2));
        CK(cudaMalloc(&dout2, 128 * 128 * 4));
        CK(cudaMemcpy(da, a.data(), a.size() * 2, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(db, b.data(), b.size() * 2, cudaMemcpyHostToDevice));
        CK(cudaFuncSetAttribute(k_accum, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * R * 4096));
        k_accum<<<1, 128, 2 * R * 4096>>>(da, db, R, dout2);
        CK(cudaDeviceSynchronize());
        std::vector<float> o(128 * 128);
        CK(cudaMemcpy(o.data(), dout2, o.size() * 4, cudaMemcpyDeviceToHost));
        double sum_rel = 0, sum_abs_rel = 0, sum_ulp = 0, sum_err_scaled = 0;
        int npos = 0, nneg = 0;
        for (int m = 0; m < 128; ++m)
            for (int n = 0; n < 128; ++n) {
                double ref = 0;
                for (int r = 0; r < R; ++r)
                    for (int k = 0; k < 16; ++k) ref += ad[r * 2048 + m * 16 + k] * bd[r * 2048 + n * 16 + k];
                const double err = (double)o[m * 128 + n] - ref;
                double amax = 0;
                for (int r = 0; r < R; ++r)
                    for (int k = 0; k < 16; ++k) amax = fmax(amax, fabs(ad[r * 2048 + m * 16 + k] * bd[r * 2048 + n * 16 + k]));
                sum_err_scaled += err / ldexp(1.0, ilogb(amax) - 23);
                sum_rel += err / ref;
                sum_abs_rel += fabs(err) / ref;
                sum_ulp += err / (ldexp(1.0, ilogb(ref) - 23));
                npos += err > 0;
                nneg += err < 0;
            }
        printf("accum mode %d R=%d: mean signed rel err %.3e, mean |rel err| %.3e, mean err %.3f ulp(result) %.3f ulp(max product), +%d / -%d\n", mode, R,
               sum_rel / 16384, sum_abs_rel / 16384, sum_ulp / 16384, sum_err_scaled / 16384, npos, nneg);
    }
    long long* dcyc;
    CK(cudaMalloc(&dcyc, 2 * 148 * sizeof(long long)));
    CK(cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
    const int R = 4000;
    const char* names[] = {"", "E only (4 x N128)", "M only (8 x N136)", "E+M"};
    for (int sts = 0; sts < 2; ++sts)
        for (int which = 1; which <= 3; ++which) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            k_rate<<<148, 160, 100 * 1024>>>(100, which, sts, dcyc);
            cudaEventRecord(e0);
            k_rate<<<148, 160, 100 * 1024>>>(R, which, sts, dcyc);
            cudaEventRecord(e1);
            CK(cudaDeviceSynchronize());
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            std::vector<long long> c(2 * 148);
            CK(cudaMemcpy(c.data(), dcyc, c.size() * 8, cudaMemcpyDeviceToHost));
            double mx = 0, mean = 0;
            for (int b = 0; b < 148; ++b) {
                mx = fmax(mx, (double)c[b]);
                mean += c[b] / 148.0;
            }
            printf("rate %-20s sts=%d: %.1f cycles/group (max %.1f), %.3f us/group wall, clk~%.0f MHz, sts iters/group %.2f\n",
                   names[which], sts, mean / R, mx / R, ms * 1e3 / R, mx / (ms * 1e3), sts ? (double)c[148] / R : 0.0);
        }
    return 0;
}
