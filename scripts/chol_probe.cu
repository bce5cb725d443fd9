// chol_probe.cu — single-warp latency of FP64 building blocks and of the two Cholesky + inverse
// forms (es_chol.cuh) on a 16 x 16 SPD matrix, in clock64 cycles.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2506_02007_b200/csrc -o scripts/chol_probe scripts/chol_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "es_chol.cuh"

using namespace es;

__global__ void k_probe(long long* cyc, double* out) {
    __shared__ double A[16 * 17], L[16 * 17], W[16 * 17], sc[2];
    const int lane = threadIdx.x;
    for (int e = threadIdx.x; e < 16 * 17; e += blockDim.x) {
        const int i = e / 17, j = e % 17;
        A[e] = (j < 16) ? (i == j ? 20.0 : 1.0 / (1 + i + j)) : 0.0;
    }
    __syncwarp();
    __syncthreads();
    double x = lane * 1e-3 + 1.0, acc = 0.0;
    long long t0 = clock64();
    for (int i = 0; i < 1000; ++i) x = fma(x, 1.0000001, 1e-9);
    long long t1 = clock64();
    for (int i = 0; i < 100; ++i) x = sqrt(x + 1.0);
    long long t2 = clock64();
    for (int i = 0; i < 100; ++i) x = 1.0 / (x + 1.0);
    long long t3 = clock64();
    for (int i = 0; i < 100; ++i) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31) + 1e-9;
    long long t4 = clock64();
    double ld = 0.0;
    bool ok = chol_inv_cta(A, L, W, 16, 17, &ld, sc);
    long long t5 = clock64();
    if (threadIdx.x < 32) ok &= chol_inv_warp(A, L, W, 16, 17, &ld);
    __syncthreads();
    long long t6 = clock64();
    for (int i = 0; i < 100; ++i) x = ldexp(x, -1) + 1.0;
    long long t7 = clock64();
    for (int i = 0; i < 16; ++i) acc += log(x + i);
    long long t8 = clock64();
    if (threadIdx.x == 0) {
        cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
        cyc[6] = t7 - t6; cyc[7] = t8 - t7;
    }
    if (threadIdx.x < 32) out[lane] = x + acc + ld + ok + W[lane] + L[lane];
}

__global__ void k_flush(double* buf, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        buf[i] = buf[i] * 0.5 + 1.0;
}

int main() {
    long long* c; double* o; double* fl;
    const size_t nf = (size_t)1 << 28;  // 2 GB streamed through L2 before the cold runs
    cudaMallocManaged(&c, 8 * sizeof(long long));
    cudaMalloc(&o, 64 * sizeof(double));
    cudaMalloc(&fl, nf * sizeof(double));
    cudaMemset(fl, 0, nf * sizeof(double));
    for (int r = 0; r < 6; ++r) {
        if (r >= 3) k_flush<<<148 * 8, 256>>>(fl, nf);  // cold L2 and instruction caches
        if (r >= 3) printf("after an L2 flush: ");
        k_probe<<<1, 256>>>(c, o);
        cudaDeviceSynchronize();
        printf("cycles: 1000 dep DFMA %lld | 100 dep sqrt %lld | 100 dep div %lld | 100 dep shfl.f64 %lld | "
               "chol_inv_cta(256 thr) %lld | chol_inv_warp %lld | 100 ldexp %lld | 16 log %lld\n",
               c[0], c[1], c[2], c[3], c[4], c[5], c[6], c[7]);
    }
    return 0;
}
