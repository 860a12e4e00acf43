// Do the FP64 SIMT pipe (DFMA) and the FP64 tensor pipe (DMMA) overlap?
// Kernel A: every warp runs DFMA chains; kernel B: every warp runs DMMA;
// kernel C: even warps DFMA, odd warps DMMA (same per-warp work as A/B).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dfma_work(double* out, int iters) {
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], 0.999999, 1e-7);
    double s = 0; for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1.2345) out[0] = s;
}
__device__ __forceinline__ void dmma_work(double* out, int iters) {
    double c[8][2];
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    double a = 1e-3 * threadIdx.x, b = 0.999;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    double s = 0; for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 1.2345) out[0] = s;
}
// per warp: DFMA path does iters*8 DFMA per lane = 256*iters FMA per warp;
// DMMA path does (iters/32)*8 DMMA = 256*iters/32*... keep FMA counts equal:
// one DMMA m8n8k4 = 256 FMA = 8 DFMA per lane.
__global__ void kA(double* o, int it) { dfma_work(o, it); }
__global__ void kB(double* o, int it) { dmma_work(o, it / 8); }
__global__ void kC(double* o, int it) { if ((threadIdx.x >> 5) & 1) dmma_work(o, it / 8); else dfma_work(o, it); }
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* d; cudaMalloc(&d, 64);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 16000, blocks = sms * 8, threads = 256;
    const double fmas = (double)blocks * threads * iters * 8;   // same FMA count in every kernel
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(e0); kA<<<blocks, threads>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1); printf("DFMA only : %.3f ms  %.1f TFLOP/s\n", ms, 2 * fmas / ms * 1e-9);
        cudaEventRecord(e0); kB<<<blocks, threads>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1); printf("DMMA only : %.3f ms  %.1f TFLOP/s\n", ms, 2 * fmas / ms * 1e-9);
        cudaEventRecord(e0); kC<<<blocks, threads>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1); printf("half/half : %.3f ms  %.1f TFLOP/s (separate pipes -> ~2x)\n", ms, 2 * fmas / ms * 1e-9);
    }
    return 0;
}
