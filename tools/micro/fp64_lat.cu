// Dependent-chain latencies on the B200 (one warp): DFMA, DADD, FFMA, IMNMX
// on the high word (the greedy's ReLU), LDS.128 -> DADD.  nvcc -arch=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double* out, long long* cyc, const double* in, int n) {
    __shared__ double2 sm[64];
    if (threadIdx.x < 64) sm[threadIdx.x] = make_double2(in[threadIdx.x], in[threadIdx.x + 1]);
    __syncthreads();
    double a = in[threadIdx.x], b = in[threadIdx.x + 32], c = in[threadIdx.x + 64];
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) a = fma(a, b, c);                 // DFMA chain
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) a = a + b;                        // DADD chain
    long long t2 = clock64();
    float fa = (float)a, fb = (float)b, fc = (float)c;
    for (int i = 0; i < n; ++i) fa = fmaf(fa, fb, fc);            // FFMA chain
    long long t3 = clock64();
    for (int i = 0; i < n; ++i) {                                 // DADD -> IMNMX(hi) chain
        a = a + b;
        int hi = __double2hiint(a), lo = __double2loint(a);
        a = __hiloint2double(max(hi, 0), lo);
    }
    long long t4 = clock64();
    int idx = threadIdx.x & 63;
    for (int i = 0; i < n; ++i) {                                 // LDS.128 -> DADD -> index chain
        double2 v = sm[idx];
        a = a + v.x;
        idx = (idx + (__double2loint(a) & 1)) & 63;
    }
    long long t5 = clock64();
    out[threadIdx.x] = a + fa;
    if (threadIdx.x == 0) {
        cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
    }
}

int main() {
    double *in, *out;
    long long* cyc;
    cudaMalloc(&in, 256 * 8);
    cudaMalloc(&out, 256 * 8);
    cudaMallocManaged(&cyc, 8 * 8);
    double h[256];
    for (int i = 0; i < 256; ++i) h[i] = 1.0 + i * 1e-9;
    cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
    const int n = 4096;
    for (int r = 0; r < 2; ++r) k<<<1, 32>>>(out, cyc, in, n);
    cudaDeviceSynchronize();
    printf("cycles per dependent op (1 warp): DFMA %.1f  DADD %.1f  FFMA %.1f  DADD+IMNMX %.1f  LDS.128+DADD+idx %.1f\n",
           (double)cyc[0] / n, (double)cyc[1] / n, (double)cyc[2] / n, (double)cyc[3] / n, (double)cyc[4] / n);
    return 0;
}
