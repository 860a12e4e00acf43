// Shared-memory load throughput on the B200 (one CTA of 256 threads = 8 warps
// on one SM): LDS.128 / LDS.64 / LDS.32 with (a) 2 distinct addresses per warp
// (the greedy's v/w slices: lanes of a device pair share one of two 16-byte
// slots), (b) all lanes the same address, (c) 32 distinct consecutive slots.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE, typename T>
__global__ void k(T* out, long long* cyc, int n) {
    __shared__ __align__(16) T sm[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = T{};
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int base = MODE == 0 ? (lane & 1) * 17 : MODE == 1 ? 0 : lane;
    T acc[8] = {};
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            T v = sm[(base + j * 64 + i) & 2047];
            acc[j].x += v.x;
            acc[j].y += v.y;
        }
    }
    __syncthreads();
    long long t1 = clock64();
    T s = acc[0];
#pragma unroll
    for (int j = 1; j < 8; ++j) { s.x += acc[j].x; s.y += acc[j].y; }
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int MODE, typename T>
double run(T* out, long long* cyc, int n) {
    k<MODE, T><<<1, 256>>>(out, cyc, n);
    k<MODE, T><<<1, 256>>>(out, cyc, n);
    cudaDeviceSynchronize();
    return (double)cyc[0] / (n * 8.0 * 8.0);   // cycles per warp-LDS on the SM
}

int main() {
    double4* o4; double2* o2; float2* o1; long long* cyc;
    cudaMalloc(&o4, 256 * sizeof(double4)); cudaMalloc(&o2, 256 * sizeof(double2)); cudaMalloc(&o1, 256 * 8);
    cudaMallocManaged(&cyc, 64);
    const int n = 2048;
    printf("SM cycles per warp-LDS (8 warps): LDS.128 2-addr %.2f bcast %.2f distinct %.2f | "
           "LDS.64 2-addr %.2f bcast %.2f distinct %.2f\n",
           run<0>(o2, cyc, n), run<1>(o2, cyc, n), run<2>(o2, cyc, n),
           run<0>(o1, cyc, n), run<1>(o1, cyc, n), run<2>(o1, cyc, n));
    return 0;
}
