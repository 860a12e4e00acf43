// Dependent-chain latencies of warp-collective instructions on the B200 (one
// warp): REDUX.MIN (__reduce_min_sync), SHFL.IDX, VOTE.BALLOT + POPC, and the
// MATCH.ANY used by k_greedy_replay experiments.  nvcc -arch=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(unsigned* out, long long* cyc, const unsigned* in, int n) {
    unsigned v = in[threadIdx.x];
    const unsigned kf = 0xffffffffu;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) v = __reduce_min_sync(kf, v + threadIdx.x) ^ threadIdx.x;
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) v = __shfl_sync(kf, v, (v + threadIdx.x) & 31);
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) v = __popc(__ballot_sync(kf, (v >> (threadIdx.x & 7)) & 1)) + v;
    long long t3 = clock64();
    for (int i = 0; i < n; ++i) v = __match_any_sync(kf, v & 7) + v;
    long long t4 = clock64();
    for (int i = 0; i < n; ++i) v = __reduce_add_sync(kf, v) + threadIdx.x;
    long long t5 = clock64();
    out[threadIdx.x] = v;
    if (threadIdx.x == 0) {
        cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
    }
}

int main() {
    unsigned *in, *out;
    long long* cyc;
    cudaMalloc(&in, 32 * 4);
    cudaMalloc(&out, 32 * 4);
    cudaMalloc(&cyc, 5 * 8);
    cudaMemset(in, 0, 32 * 4);
    const int n = 4096;
    for (int rep = 0; rep < 2; ++rep) k<<<1, 32>>>(out, cyc, in, n);
    long long h[5];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const char* nm[5] = {"REDUX.MIN", "SHFL.IDX", "VOTE+POPC", "MATCH.ANY", "REDUX.SUM"};
    for (int i = 0; i < 5; ++i) printf("%-10s %.1f cycles per dependent op (incl. 1-2 ALU ops)\n", nm[i], (double)h[i] / n);
    return 0;
}
