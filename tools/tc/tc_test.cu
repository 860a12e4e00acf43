// Standalone check of the hand-written tcgen05 (kind::tf32) path:
// D[128 x N] = A[128 x K] . B[N x K]^T, operands K-major in shared memory
// (no swizzle, canonical core-matrix layout), accumulator in TMEM, read back
// with tcgen05.ld.  Plain and split-TF32 x3 (A_hi B_hi + A_hi B_lo + A_lo B_hi).
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;   // version 1 (Blackwell)
    return d;                 // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
}

__host__ __device__ constexpr uint32_t make_idesc_tf32(int M, int N) {
    return (1u << 4)            // c_format F32
         | (2u << 7)            // a_format TF32
         | (2u << 10)           // b_format TF32
         | ((uint32_t)(N >> 3) << 17)
         | ((uint32_t)(M >> 4) << 24);
}

// K-major canonical layout: element (r, k) of a [rows x K] operand
__device__ __forceinline__ int kmaj_off(int r, int k, int rows) {   // in floats
    return (k >> 2) * (rows * 4) + (r >> 3) * 32 + (r & 7) * 4 + (k & 3);
}

__device__ __forceinline__ float tf32_hi(float x) {
    uint32_t u = __float_as_uint(x) & 0xFFFFE000u;   // keep 10 mantissa bits (truncate)
    return __uint_as_float(u);
}

template <int N, int K, bool SPLIT>
__global__ void tc_gemm(const float* A, const float* B, float* D) {
    extern __shared__ __align__(128) float sm[];
    float* sAh = sm;                 // [128 x K]
    float* sAl = sAh + 128 * K;
    float* sBh = sAl + 128 * K;      // [N x K]
    float* sBl = sBh + N * K;
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t mbar;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 128 * K; i += blockDim.x) {
        const int r = i / K, k = i % K;
        const float x = A[i], hi = tf32_hi(x);
        sAh[kmaj_off(r, k, 128)] = hi;
        sAl[kmaj_off(r, k, 128)] = x - hi;
    }
    for (int i = tid; i < N * K; i += blockDim.x) {
        const int r = i / K, k = i % K;
        const float x = B[i], hi = tf32_hi(x);
        sBh[kmaj_off(r, k, N)] = hi;
        sBl[kmaj_off(r, k, N)] = x - hi;
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(N < 32 ? 32 : N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");   // generic-proxy smem writes -> async proxy (MMA)
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base;
    if (tid == 0) {
        const uint32_t idesc = make_idesc_tf32(128, N);
        const int nmma = SPLIT ? 3 : 1;
        for (int s = 0; s < K / 8; ++s) {
            for (int q = 0; q < nmma; ++q) {
                const float* a = (q == 2) ? sAl : sAh;
                const float* b = (q == 1) ? sBl : sBh;
                const uint64_t ad = make_desc(smem_u32(a + 2 * s * 128 * 4), 128 * 16, 128);
                const uint64_t bd = make_desc(smem_u32(b + 2 * s * N * 4), N * 16, 128);
                const uint32_t acc = (s > 0 || q > 0) ? 1u : 0u;
                asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                             " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}"
                             ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
    }
    // wait for the MMAs (phase 0)
    {
        uint32_t done = 0;
        while (!done) {
            asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                         : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
        }
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    // each warp reads its 32 lanes (rows), 8 columns at a time
    const int row = warp * 32 + (tid & 31);
    for (int c0 = 0; c0 < N; c0 += 8) {
        uint32_t r[8];
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int j = 0; j < 8; ++j) D[row * N + c0 + j] = __uint_as_float(r[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(N < 32 ? 32 : N));
}

int main() {
    constexpr int N = 64, K = 32;
    std::vector<float> A(128 * K), B(N * K), D(128 * N);
    unsigned s = 12345;
    auto rnd = [&]() { s = s * 1664525u + 1013904223u; return ((s >> 8) & 0xFFFF) / 65536.0f - 0.5f; };
    for (auto& x : A) x = rnd();
    for (auto& x : B) x = rnd();
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    const size_t smem = (size_t)(2 * 128 * K + 2 * N * K) * 4;
    for (int split = 0; split < 2; ++split) {
        if (split) { cudaFuncSetAttribute(tc_gemm<N, K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                     tc_gemm<N, K, true><<<1, 128, smem>>>(dA, dB, dD); }
        else { cudaFuncSetAttribute(tc_gemm<N, K, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
               tc_gemm<N, K, false><<<1, 128, smem>>>(dA, dB, dD); }
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double maxrel = 0, maxabs = 0;
        for (int i = 0; i < 128; ++i)
            for (int j = 0; j < N; ++j) {
                double ref = 0;
                for (int k = 0; k < K; ++k) ref += (double)A[i * K + k] * (double)B[j * K + k];
                double err = fabs(ref - D[i * N + j]);
                maxabs = fmax(maxabs, err);
                maxrel = fmax(maxrel, err / fmax(fabs(ref), 1e-3));
            }
        printf("%s: max abs err %.3e  max rel err %.3e  D[0]=%f D[last]=%f\n", split ? "3xTF32" : "TF32", maxabs, maxrel, D[0], D[128 * N - 1]);
    }
    return 0;
}
