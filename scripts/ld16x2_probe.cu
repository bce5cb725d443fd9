// ld16x2_probe.cu — which TMEM lane / column each thread reads with
// tcgen05.ld.16x32bx2 (immHalfSplitoff): value = lane * 1000 + column.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o ld16x2_probe ld16x2_probe.cu
#include <cstdio>
#include <cstdint>

__global__ void probe(float* out) {
    __shared__ uint32_t tbase;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tbase;
    for (int c = 0; c < 64; ++c) {
        const float v = (float)(t * 1000 + c);  // TMEM lane t (warp w writes lanes 32w..32w+31)
        asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tm + ((uint32_t)(32 * warp) << 16) + c),
                     "r"(__float_as_uint(v))
                     : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t r0, r1;
    asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x2.b32 {%0,%1}, [%2], 16;"
                 : "=r"(r0), "=r"(r1)
                 : "r"(tm + ((uint32_t)(32 * warp) << 16) + 4));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    out[2 * t] = __uint_as_float(r0);
    out[2 * t + 1] = __uint_as_float(r1);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tm));
    (void)lane;
}

int main() {
    float* d;
    cudaMalloc(&d, 256 * 4);
    probe<<<1, 128>>>(d);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    float h[256];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    for (int t : {0, 1, 15, 16, 17, 31, 32, 47, 48, 63})
        printf("thread %2d: %8.0f %8.0f\n", t, h[2 * t], h[2 * t + 1]);
    return 0;
}
