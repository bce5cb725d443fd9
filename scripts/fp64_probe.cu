// fp64_probe.cu — FP64 throughput on this GPU: SIMT DFMA vs mma.sync m8n8k4 f64 (DMMA).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe fp64_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(int iters, double* out) {
    double a[16];
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3 + i;
    const double b = 1.0000001, c = 1e-9;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
    double s = 0;
    for (int i = 0; i < 16; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dmma(int iters, double* out) {
    double acc[8][2];
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
    const double a = 1.0 + threadIdx.x * 1e-6, b = 0.5;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[i][0]), "+d"(acc[i][1])
                         : "d"(a), "d"(b));
    double s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    double* out;
    cudaMalloc(&out, 148 * 1024 * sizeof(double));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        const int it = 20000;
        cudaEventRecord(e0);
        k_dfma<<<148 * 4, 256>>>(it, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double dfma = 148.0 * 4 * 256 * it * 16;
        printf("DFMA: %.2f TFLOP/s (%.1f DFMA/clk/SM at 1.9 GHz)\n", 2 * dfma / (ms * 1e-3) / 1e12,
               dfma / (ms * 1e-3) / 148 / 1.9e9);
        cudaEventRecord(e0);
        k_dmma<<<148 * 4, 256>>>(it, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double mac = 148.0 * 4 * (256 / 32) * it * 8 * 256;
        printf("DMMA m8n8k4: %.2f TFLOP/s (%.1f MAC/clk/SM at 1.9 GHz)\n", 2 * mac / (ms * 1e-3) / 1e12,
               mac / (ms * 1e-3) / 148 / 1.9e9);
    }
    return 0;
}
