// Microbenchmark: measured FP64 pipe throughput on this GPU (the "alu"
// roofline denominator of DESIGN.md).  8 independent DFMA chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1.2345) out[0] = s;
}
__global__ void ffma_loop(float* out, int iters, float a, float b) {
    float x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, x[(i + 1) & 7]);
    }
    float s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1.2345f) out[0] = s;
}
__global__ void dmma_loop(double* out, int iters) {
    double c[8][2];
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    double a = 1e-3 * threadIdx.x, b = 0.999;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 1.2345) out[0] = s;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* d; cudaMalloc(&d, 64);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 20000, blocks = sms * 8, threads = 256;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        dfma_loop<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double fmas = (double)blocks * threads * iters * 8;
        printf("DFMA: %.3f ms  %.2f TDFMA/s  %.2f TFLOP/s fp64  per-SM-per-clk@1965MHz=%.1f\n", ms,
               fmas / ms * 1e-9, 2 * fmas / ms * 1e-9, fmas / (ms * 1e-3) / sms / 1.965e9);
    }
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        dmma_loop<<<blocks, threads>>>(d, iters / 4);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double fmas = (double)blocks * (threads / 32) * (iters / 4) * 8 * 256;
        printf("DMMA: %.3f ms  %.2f TFLOP/s fp64 tensor  FMA/SM/clk@1965MHz=%.1f\n", ms, 2 * fmas / ms * 1e-9,
               fmas / (ms * 1e-3) / sms / 1.965e9);
    }
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        ffma_loop<<<blocks, threads>>>((float*)d, iters, 0.999999f, 1e-7f);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double fmas = (double)blocks * threads * iters * 8;
        printf("FFMA: %.3f ms  %.2f TFLOP/s fp32  per-SM-per-clk@1965MHz=%.1f\n", ms, 2 * fmas / ms * 1e-9,
               fmas / (ms * 1e-3) / sms / 1.965e9);
    }
    return 0;
}
