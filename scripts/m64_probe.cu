// m64_probe.cu — where does a cta_group::1 M = 64 kind::f16 accumulator land in TMEM, and
// can a second M = 64 MMA target TMEM lanes 64..127 (lane field of the D address)?
// D[m][n] = (m + 1) + 256 n (+ 1000 for the second MMA); TMEM prefilled with -1.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o m64_probe m64_probe.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
    return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ uint32_t kmaj(int row, int k) {
    return (uint32_t)((row >> 3) * 256 + (k >> 3) * 128 + (row & 7) * 16 + (k & 7) * 2);
}
constexpr int NC = 64;  // TMEM columns read back

__global__ void probe(float* out, int second_lane) {
    __shared__ __align__(1024) unsigned char a0[64 * 32], a1[64 * 32], b[16 * 32];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int t = threadIdx.x, warp = t >> 5;
    for (int i = t; i < 64 * 16; i += 128) {
        const int m = i / 16, k = i % 16;
        *reinterpret_cast<__half*>(a0 + kmaj(m, k)) = __float2half(k == 0 ? (float)(m + 1) : (k == 1 ? 1.f : 0.f));
        *reinterpret_cast<__half*>(a1 + kmaj(m, k)) =
            __float2half(k == 0 ? (float)(m + 1001) : (k == 1 ? 1.f : 0.f));
    }
    for (int i = t; i < 16 * 16; i += 128) {
        const int n = i / 16, k = i % 16;
        *reinterpret_cast<__half*>(b + kmaj(n, k)) = __float2half(k == 0 ? 1.f : (k == 1 ? 256.f * n : 0.f));
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
    // prefill -1
    {
        const uint32_t neg = __float_as_uint(-1.f);
        for (int c = 0; c < NC; c += 8)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                             tm + ((uint32_t)(32 * warp) << 16) + c),
                         "r"(neg)
                         : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (t == 0) {
        const uint32_t id = idesc_f16(64, 16);
        const uint64_t da0 = desc(su32(a0), 128, 256), da1 = desc(su32(a1), 128, 256), db = desc(su32(b), 128, 256);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm),
                     "l"(da0), "l"(db), "r"(id), "r"(0));
        const uint32_t d2 = tm + ((uint32_t)second_lane << 16) + 32;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d2),
                     "l"(da1), "l"(db), "r"(id), "r"(0));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    }
    {
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                         : "=r"(done) : "r"(su32(&bar)) : "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (int c = 0; c < NC; ++c) {
        uint32_t r;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(tm + ((uint32_t)(32 * warp) << 16) + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        out[t * NC + c] = __uint_as_float(r);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm));
}

int main() {
    float* d;
    cudaMalloc(&d, 128 * NC * 4);
    float h[128 * NC];
    for (int sl : {0, 64, 16}) {
        probe<<<1, 128>>>(d, sl);
        cudaError_t e = cudaDeviceSynchronize();
        printf("second MMA lane offset %d: %s\n", sl, cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        for (int lane = 0; lane < 128; ++lane) {
            printf("lane %3d:", lane);
            for (int c : {0, 1, 2, 15, 16, 31, 32, 33, 47, 48})
                printf(" %7.0f", h[lane * NC + c]);
            printf("\n");
        }
    }
    return 0;
}
