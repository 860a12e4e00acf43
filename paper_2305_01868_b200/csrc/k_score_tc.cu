// k_score_tc.cu -- ns_score_plans bulk mode (NS_SCORE_TF32X3): the two
// communication-cost MLPs (2D -> 128 -> 64 -> 32 -> 16 -> D) as a
// chain of tcgen05 GEMMs on the 5th-generation tensor cores.
//
// Precision: every operand is split x = hi + lo with hi = x rounded to TF32
// (10-bit mantissa) and lo = x - hi (exact in fp32), and each layer computes
// A_hi B_hi + A_hi B_lo + A_lo B_hi with FP32 accumulation in TMEM ("3xTF32"):
// ~1e-6 relative, FP32-grade, within the north star's 1e-3 plan-cost
// tolerance.  The greedy search keeps the fp64 DMMA path (its decisions are
// compared at far smaller margins).
//
// Structure (one CTA of 128 threads per SM, persistent over 128-row tiles,
// one launch per model direction): the model's weights (hi/lo, K-major
// canonical no-swizzle layout) stay resident in shared memory; thread i owns
// plan row i = TMEM lane i.  Per tile: build the input rows, then for each
// layer one elected thread issues tcgen05.mma (A, B from shared-memory
// descriptors, D in TMEM), tcgen05.commit arrives on an mbarrier, and the
// 4 warps read their 32 TMEM lanes back (tcgen05.ld), apply bias + ReLU,
// re-split and write the next layer's A operand.  The 128-wide hidden layer is
// consumed by layer 2 in four 32-column K chunks through a double-buffered
// operand ring so the activations never need more than 64 KB of smem.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <algorithm>

#include "ns_device.cuh"
#include "ns_internal.cuh"

namespace ns {
namespace {

constexpr int kTile = 128;     // rows (plans) per tile = TMEM lanes = UMMA M

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// UMMA shared-memory descriptor, K-major, SWIZZLE_NONE (canonical layout
// ((8,m),2):((16B,SBO),LBO)), version 1.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

// Instruction descriptor: kind::tf32, D f32, A/B tf32 K-major, M x N.
__device__ __forceinline__ uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// element (r, k) of a K-major [rows x K] operand, in floats
__device__ __forceinline__ int kmaj(int r, int k, int rows) {
    return (k >> 2) * (rows * 4) + (r >> 3) * 32 + (r & 7) * 4 + (k & 3);
}

__device__ __forceinline__ float tf32_rn(float x) {   // round to nearest TF32 (10-bit mantissa)
    uint32_t u = __float_as_uint(x);
    u += 0x1000u;
    return __uint_as_float(u & 0xFFFFE000u);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                 " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
                 "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    uint32_t done = 0;
    while (!done) {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done)
                     : "r"(su32(bar)), "r"(phase));
    }
}

// 16 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
}

// 16 consecutive fp32 columns, no wait (caller issues tcgen05.wait::ld)
__device__ __forceinline__ void tmem_ld16_nw(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr)
                 : "memory");
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
}

// 32 consecutive fp32 columns of this thread's TMEM lane (one load, one wait)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                   "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
                   "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
                   "=r"(r[30]), "=r"(r[31])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
}

struct TcArgs {
    long long row_begin, row_end;   // plan rows
    int D, K0p, N5p;                // 2D padded to 8, D padded to 16
    int dir;                        // 0 fwd (starts = comp - min comp), 1 bwd (starts = 0)
    const double* comp;             // [P][D]
    const int32_t* devdim;          // [P][D]
    float* out;                     // [P][D] MLP output of this direction
    const double* W[5];
    const double* b[5];
    double start_scale, dim_scale;
    int n_tiles;
    uint32_t rflags;
};

// weight smem layout: per layer hi block then lo block, each K-major [Np x Kp]
struct WLayout {
    int Kp[5], Np[5], K[5], N[5];
    int off[5];      // float offset of the hi block; lo block follows
    int total;       // floats
};

__device__ __forceinline__ WLayout wlayout(int D, int K0p, int N5p) {
    WLayout L;
    const int K[5] = {2 * D, 128, 64, 32, 16};
    const int N[5] = {128, 64, 32, 16, D};
    const int Kp[5] = {K0p, 128, 64, 32, 16};
    const int Np[5] = {128, 64, 32, 16, N5p};
    int o = 0;
    for (int l = 0; l < 5; ++l) {
        L.K[l] = K[l];
        L.N[l] = N[l];
        L.Kp[l] = Kp[l];
        L.Np[l] = Np[l];
        L.off[l] = o;
        o += 2 * Kp[l] * Np[l];
    }
    L.total = o;
    return L;
}

// Two tile groups per CTA (warps 0-3 and 4-7, 128 rows each, own 256 TMEM
// columns, own operand ring and mbarriers, named barriers): while one group
// runs its TMEM -> register -> smem epilogue, the other's MMAs keep the
// tensor core busy.  Every layer's A operand streams through a per-group
// ring of two 16-column K chunks (hi, lo): the epilogue of chunk c overlaps
// the MMAs of chunk c - 1.
constexpr int kGroups = 2;
constexpr int kKc = 16;                       // K columns per operand chunk
constexpr int kABuf = kTile * kKc * 2;        // floats per operand buffer (hi + lo)

__global__ void __launch_bounds__(128 * kGroups, 1) k_plan_mlp_tc(const TcArgs a) {
    extern __shared__ __align__(128) float tsm[];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t s_bar[kGroups][2];   // per group: operand buffer 0 / 1 consumed
    __shared__ float s_bias[128 + 64 + 32 + 16 + 64];
    const int tid = threadIdx.x, warp = tid >> 5;
    const int grp = tid >> 7, gtid = tid & 127, gwarp = warp & 3;
    const WLayout L = wlayout(a.D, a.K0p, a.N5p);
    float* sW = tsm;                                   // weights (resident, shared by both groups)
    float* sA = tsm + L.total + grp * 2 * kABuf;       // this group's two operand buffers
    // ---- resident weights: hi/lo split, K-major, zero padded
    for (int l = 0; l < 5; ++l) {
        const int Kp = L.Kp[l], Np = L.Np[l], K = L.K[l], N = L.N[l];
        float* hi = sW + L.off[l];
        float* lo = hi + Kp * Np;
        for (int i = tid; i < Kp * Np; i += blockDim.x) {
            const int n = i / Kp, k = i % Kp;
            const float x = (n < N && k < K) ? (float)a.W[l][(size_t)n * K + k] : 0.0f;
            const float h = tf32_rn(x);
            hi[kmaj(n, k, Np)] = h;
            lo[kmaj(n, k, Np)] = x - h;
        }
    }
    {
        const int N[5] = {128, 64, 32, 16, a.D};
        const int off[5] = {0, 128, 192, 224, 240};
        for (int l = 0; l < 5; ++l)
            for (int i = tid; i < N[l]; i += blockDim.x) s_bias[off[l] + i] = (float)a.b[l][i];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&s_tmem)),
                     "r"(256 * kGroups));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int g = 0; g < kGroups; ++g)
            for (int i = 0; i < 2; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&s_bar[g][i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = s_tmem + (uint32_t)(grp * 256);               // this group's columns
    const uint32_t lane_base = tmem + ((uint32_t)(gwarp * 32) << 16);   // this warp's 32 TMEM lanes
    uint64_t* bar = s_bar[grp];
    uint32_t ph[2] = {0, 0};   // mbarrier phases (every thread waits on every commit, in order)

    // the group's operand writes -> visible to the async proxy, then the MMA issue
    auto gsync = [&]() {
        asm volatile("fence.proxy.async.shared::cta;");
        asm volatile("tcgen05.fence::before_thread_sync;");
        asm volatile("bar.sync %0, 128;" ::"r"(1 + grp));
        asm volatile("tcgen05.fence::after_thread_sync;");
    };
    // this thread's row values v[0..n) (n multiple of 4) at chunk columns 0..n
    // as TF32 hi / lo splits: 128-bit stores of whole core-matrix rows
    // (eight threads fill one 128-byte wavefront, no bank conflicts)
    auto put_row = [&](float* Ahi, float* Alo, int n, const float* v) {
        for (int j = 0; j < n; j += 4) {
            float4 h4, l4;
            h4.x = tf32_rn(v[j]);
            h4.y = tf32_rn(v[j + 1]);
            h4.z = tf32_rn(v[j + 2]);
            h4.w = tf32_rn(v[j + 3]);
            l4.x = v[j] - h4.x;
            l4.y = v[j + 1] - h4.y;
            l4.z = v[j + 2] - h4.z;
            l4.w = v[j + 3] - h4.w;
            *reinterpret_cast<float4*>(&Ahi[kmaj(gtid, j, kTile)]) = h4;
            *reinterpret_cast<float4*>(&Alo[kmaj(gtid, j, kTile)]) = l4;
        }
    };
    // one layer: D[dcol..] = A . W_l^T over K input columns, A produced chunk
    // by chunk by make(c0, v) (Kc values of input columns c0..c0+Kc)
    auto layer = [&](int l, int K, uint32_t dcol, auto&& make) {
        const int Kc = K < kKc ? K : kKc;
        const int nch = K / Kc;
        const int Np = L.Np[l];
        const float* Bhi = sW + L.off[l];
        const float* Blo = Bhi + L.Kp[l] * Np;
        const uint32_t idesc = idesc_tf32(kTile, Np);
        for (int c = 0; c < nch; ++c) {
            const int b = c & 1;
            if (c >= 2) {   // chunk c - 2's MMAs have consumed buffer b
                mbar_wait(&bar[b], ph[b]);
                ph[b] ^= 1;
            }
            float* Ahi = sA + b * kABuf;
            float* Alo = Ahi + kTile * Kc;
            float v[kKc];
            make(c * Kc, v);
            put_row(Ahi, Alo, Kc, v);
            gsync();
            if (gtid == 0) {
                for (int s = 0; s < Kc / 8; ++s) {
                    const int kb = c * (Kc / 8) + s;   // k-step of the weight block
                    const uint64_t ahd = umma_desc(su32(Ahi + s * 8 * kTile), kTile * 16, 128);
                    const uint64_t ald = umma_desc(su32(Alo + s * 8 * kTile), kTile * 16, 128);
                    const uint64_t bhd = umma_desc(su32(Bhi + kb * 8 * Np), Np * 16, 128);
                    const uint64_t bld = umma_desc(su32(Blo + kb * 8 * Np), Np * 16, 128);
                    const uint32_t acc0 = (kb > 0) ? 1u : 0u;
                    mma_tf32(tmem + dcol, ahd, bhd, idesc, acc0);
                    mma_tf32(tmem + dcol, ahd, bld, idesc, 1u);
                    mma_tf32(tmem + dcol, ald, bhd, idesc, 1u);
                }
                commit(&bar[b]);
            }
        }
        // drain the last (up to) two chunks: every MMA of the layer has landed
        for (int c = nch >= 2 ? nch - 2 : 0; c < nch; ++c) {
            const int b = c & 1;
            mbar_wait(&bar[b], ph[b]);
            ph[b] ^= 1;
        }
        asm volatile("tcgen05.fence::after_thread_sync;");
    };
    // hidden-layer input: the previous layer's TMEM columns + bias, ReLU
    auto from_tmem = [&](int col0, const float* bias) {
        return [=](int c0, float (&v)[kKc]) {
            tmem_ld16(lane_base + col0 + c0, v);
#pragma unroll
            for (int j = 0; j < kKc; ++j) v[j] = fmaxf(v[j] + bias[c0 + j], 0.0f);
        };
    };

    // TMEM columns of a group: [0,128) layer-1 output, [128,192) layer 2,
    // [192,224) layer 3, [224,240) layer 4, [240,256) layer 5
    for (int tile = blockIdx.x * kGroups + grp; tile < a.n_tiles; tile += gridDim.x * kGroups) {
        const long long row = a.row_begin + (long long)tile * kTile + gtid;
        const bool rv = row < a.row_end;
        // ---- layer-1 input row: [starts / start_scale, devdim / dim_scale]
        double mn = CUDART_INF;
        if (rv && a.dir == 0 && !(a.rflags & NS_R10_ABS_STARTS))
            for (int d = 0; d < a.D; ++d) mn = fmin(mn, a.comp[row * a.D + d]);
        if (a.rflags & NS_R10_ABS_STARTS) mn = 0.0;   // R10 alternative: absolute starts
        layer(0, a.K0p, 0, [&](int c0, float (&v)[kKc]) {
            for (int j = 0; j < kKc; ++j) {
                const int k = c0 + j;
                float x = 0.0f;
                if (rv && k < 2 * a.D) {
                    if (k < a.D)
                        x = a.dir == 0 ? (float)((a.comp[row * a.D + k] - mn) / a.start_scale) : 0.0f;
                    else
                        x = (float)((double)a.devdim[row * a.D + k - a.D] / a.dim_scale);
                }
                v[j] = x;
            }
        });
        layer(1, 128, 128, from_tmem(0, s_bias));
        layer(2, 64, 192, from_tmem(128, s_bias + 128));
        layer(3, 32, 224, from_tmem(192, s_bias + 192));
        layer(4, 16, 240, from_tmem(224, s_bias + 224));
        // ---- output layer (no activation)
        {
            float v[16];
            tmem_ld16(lane_base + 240, v);
            if (rv)
                for (int d = 0; d < a.D; ++d) a.out[row * a.D + d] = v[d] + s_bias[240 + d];
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "r"(256 * kGroups));
}

__global__ void k_plan_cost_combine(const double* comp, const float* fwd, const float* bwd, const uint8_t* ok,
                                    long long pb, long long pe, int D, double* cost, int sum_of_max) {
    for (long long p = pb + (long long)blockIdx.x * blockDim.x + threadIdx.x; p < pe;
         p += (long long)gridDim.x * blockDim.x) {
        double c = -CUDART_INF;
        if (sum_of_max) {   // R11 alternative: sum of the per-term maxima
            double mc = -CUDART_INF, mf = -CUDART_INF, mb = -CUDART_INF;
            for (int d = 0; d < D; ++d) {
                mc = fmax(mc, comp[p * D + d]);
                mf = fmax(mf, (double)fwd[p * D + d]);
                mb = fmax(mb, (double)bwd[p * D + d]);
            }
            c = (mc + mf) + mb;
        } else {
            for (int d = 0; d < D; ++d)
                c = fmax(c, (comp[p * D + d] + (double)fwd[p * D + d]) + (double)bwd[p * D + d]);
        }
        cost[p] = ok[p] ? c : CUDART_NAN;
    }
}

// ---------------------------------------------------------------------------
// N2 on tcgen05 (NS_SCORE_TF32X3): per-device sum pooling of every plan as a
// one-hot contraction.  Row r = (plan, device d) of a 128-row tile:
//   U[r][n] = sum_t A[r][t] * B[n][t],  A[r][t] = [a_{p,t} == d] (exact in bf16),
// B[n][t] = the task's cached head row v_t (n < 64), the variant dim (n = 64,
// integers <= 128: exact) and 1 (n = 65: tables per device).  v is split in
// three bf16 pieces (v = hi + mid + lo to ~2^-24 relative) and the three
// pieces are accumulated into ONE fp32 TMEM accumulator by three MMAs per K
// step; a ones column of A (t = Tp) times B[n][Tp] = hb1_n adds the head bias
// on the tensor core, so u = hb1 + sum_{t on d} v_t comes out of TMEM ready.
// The one-hot operand is 2 bytes per (row, table) -- 1/8 of the 64 fp32 of a
// staged v row a SIMT warp reads per (plan, table).  Epilogue: ReLU and the
// H2 dot in fp64; a plan holding an id outside 0..D-1 is caught by its table
// count (sum over its D rows of column 65 != Tp).  Two tile groups of 8 warps
// per CTA (threads r and r + 128 of a group share TMEM lane r and split the
// K chunks of the build and the 64 features of the epilogue); each group has
// its own 128 TMEM columns, one-hot buffer, double-buffered cp.async staging
// of the assignment bytes (prefetched a tile ahead) and mbarrier.
constexpr int kPoolN = 80;      // per piece: 64 features + dims + count, padded to 16

struct PoolTcArgs {
    long long p_begin, p_end;
    int Tp, Kp, D, LG;          // Kp = Tp + 1 (ones column) rounded up to 16; rows per plan 1 << LG >= D
    int SG;                     // bytes of one assignment staging buffer
    const int8_t* assign;       // [P][Tp] (global plan index)
    const int32_t* rows;        // [Tp] variant rows
    const double* V;            // [rows][64]
    const int32_t* vdim;
    double* comp;               // [P][D]
    int32_t* devdim;            // [P][D]
    uint8_t* ok;                // [P]
    HeadParams head;
    float h2f[kV];              // H2 rounded to fp32 (epilogue partial dots)
    long long n_tiles;
};

__device__ __forceinline__ uint32_t bf16_bits(float x) {   // round to nearest even
    const uint32_t u = __float_as_uint(x);
    return (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                 " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
                 "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}

// piece k (0 hi, 1 mid, 2 lo) of x as bf16 bits: x = hi + mid + lo + O(2^-25 |x|)
__device__ __forceinline__ uint32_t bf16_piece(double x, int k) {
    const uint32_t hb = bf16_bits((float)x);
    if (k == 0) return hb;
    const double r1 = x - (double)__uint_as_float(hb << 16);
    const uint32_t mb = bf16_bits((float)r1);
    if (k == 1) return mb;
    return bf16_bits((float)(r1 - (double)__uint_as_float(mb << 16)));
}

__global__ void __launch_bounds__(512, 1) k_pool_tc(const PoolTcArgs a) {
    extern __shared__ __align__(128) uint8_t psm[];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t s_bar[2][2];   // per group, per accumulator buffer
    __shared__ double s_part[2][128];     // the upper half's partial head dot per row
    const int tid = threadIdx.x, warp = tid >> 5;
    const int grp = tid >> 8, gtid = tid & 255, gwarp = warp & 3;
    const int r = gtid & 127, hf = gtid >> 7;
    const int Kp = a.Kp, Tp = a.Tp, D = a.D, LG = a.LG, PT = 128 >> LG;
    const size_t bblk = (size_t)kPoolN * Kp * 2;                    // bytes of one piece block
    uint8_t* sB = psm;                                              // 3 x [80 x Kp] bf16, K-major
    uint8_t* sA = psm + 3 * bblk + (size_t)grp * 2 * 128 * Kp * 2;  // 2 x [128 x Kp] one-hot
    uint8_t* sG = psm + 3 * bblk + (size_t)4 * 128 * Kp * 2 + (size_t)grp * 2 * a.SG;  // 2 x [SG] bytes
    // ---- resident B (three piece blocks)
    for (int i = tid; i < 3 * kPoolN * Kp; i += blockDim.x) {
        const int k = i / (kPoolN * Kp), rem = i - k * (kPoolN * Kp);
        const int n = rem / Kp, t = rem - n * Kp;
        uint32_t bits = 0;
        if (t < Tp) {
            const int row = __ldg(a.rows + t);
            if (n < 64)
                bits = bf16_piece(__ldg(a.V + (size_t)row * kV + n), k);
            else if (k == 0 && n == 64)
                bits = bf16_bits((float)__ldg(a.vdim + row));
            else if (k == 0 && n == 65)
                bits = 0x3F80u;
        } else if (t == Tp && n < 64) {
            bits = bf16_piece(a.head.hb1[n], k);   // bias column (A's ones column)
        }
        *reinterpret_cast<uint16_t*>(sB + (size_t)k * bblk + (size_t)(t >> 3) * (kPoolN * 16) + (n >> 3) * 128 +
                                     (n & 7) * 16 + (t & 7) * 2) = (uint16_t)bits;
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&s_tmem)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int g = 0; g < 4; ++g) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&s_bar[g >> 1][g & 1])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = s_tmem + (uint32_t)(grp * 256);   // two 128-column accumulators per group
    const uint32_t lane_off = (uint32_t)(gwarp * 32) << 16;
    uint32_t phbits = 0;   // mbarrier phase per accumulator buffer
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kPoolN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const int pl = r >> LG, d = r & ((1 << LG) - 1);
    const uint32_t d4 = (uint32_t)d * 0x01010101u;
    auto gbar = [&]() { asm volatile("bar.sync %0, 256;" ::"r"(1 + grp)); };
    // stage a tile's assignment bytes (contiguous in global: PT plans x Tp) as
    // 16-byte cp.async chunks from the 16-byte aligned-down start
    const uintptr_t abase = reinterpret_cast<uintptr_t>(a.assign);
    auto stage = [&](long long tile, int buf) {
        if (tile < a.n_tiles) {
            const long long p0 = a.p_begin + tile * PT;
            const long long np = a.p_end - p0 < PT ? a.p_end - p0 : PT;
            const uintptr_t g0 = (abase + (uintptr_t)(p0 * Tp)) & ~(uintptr_t)15;
            const uintptr_t g1 = abase + (uintptr_t)((p0 + np) * Tp);
            const int nch = (int)((g1 - g0 + 15) >> 4);
            const uint32_t dst = su32(sG + (size_t)buf * a.SG);
            for (int c = gtid; c < nch; c += 256)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16 * c), "l"(g0 + 16 * (uintptr_t)c));
        }
        asm volatile("cp.async.commit_group;");
    };
    const int kh = Kp >> 4;                   // K chunks (8 tables) per half
    const int kc_last = (Tp - 1) >> 3;        // chunks from here on hold bytes past the row (masked)
    // one-hot rows of `tile` (staged in sG[buf]) into A[buf], then the MMAs into accumulator buf
    auto build_mma = [&](long long tile, int buf) {
        const long long p0 = a.p_begin + tile * PT;
        uint8_t* Ab = sA + (size_t)buf * 128 * Kp * 2;
        {
            const int o = (int)((abase + (uintptr_t)(p0 * Tp)) & 15) + pl * Tp;
            const uint32_t* g = reinterpret_cast<const uint32_t*>(sG + (size_t)buf * a.SG) + (o >> 2);
            const uint32_t sh = 8u * (uint32_t)(o & 3);
            uint8_t* arow = Ab + (r >> 3) * 128 + (r & 7) * 16;
            uint32_t w0 = g[2 * kh * hf];
            for (int kc = kh * hf; kc < kh * (hf + 1); ++kc) {
                const uint32_t w1 = g[2 * kc + 1], w2 = g[2 * kc + 2];
                uint32_t x0 = __funnelshift_r(w0, w1, sh), x1 = __funnelshift_r(w1, w2, sh);
                w0 = w2;
                uint32_t one0 = 0, one1 = 0;
                if (kc >= kc_last) {   // uniform: bytes past the row never match; the ones column
                    const int t0 = 8 * kc;
                    const int v0 = min(max(Tp - t0, 0), 4), v1 = min(max(Tp - t0 - 4, 0), 4);
                    x0 |= v0 >= 4 ? 0u : (0xFFFFFFFFu << (8 * v0));
                    x1 |= v1 >= 4 ? 0u : (0xFFFFFFFFu << (8 * v1));
                    const int j = Tp - t0;   // ones column position in this chunk (0..7), if any
                    if (j >= 0 && j < 4) one0 = 0xFFu << (8 * j);
                    if (j >= 4 && j < 8) one1 = 0xFFu << (8 * (j - 4));
                }
                // 0xFF per matching byte; the ones column's byte forced to match
                const uint32_t e0 = __vcmpeq4(x0, d4) | one0;
                const uint32_t e1 = __vcmpeq4(x1, d4) | one1;
                uint4 q;
                q.x = __byte_perm(e0, 0, 0x1100) & 0x3F803F80u;
                q.y = __byte_perm(e0, 0, 0x3322) & 0x3F803F80u;
                q.z = __byte_perm(e1, 0, 0x1100) & 0x3F803F80u;
                q.w = __byte_perm(e1, 0, 0x3322) & 0x3F803F80u;
                *reinterpret_cast<uint4*>(arow + (size_t)kc * (128 * 16)) = q;
            }
        }
        asm volatile("fence.proxy.async.shared::cta;");
        asm volatile("tcgen05.fence::before_thread_sync;");
        gbar();
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (gtid == 0) {
            for (int ks = 0; ks < (Kp >> 4); ++ks) {
                const uint64_t ad = umma_desc(su32(Ab + (size_t)ks * 2 * (128 * 16)), 128 * 16, 128);
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const uint64_t bd = umma_desc(su32(sB + k * bblk + (size_t)ks * 2 * (kPoolN * 16)), kPoolN * 16, 128);
                    mma_bf16(tmem + 128 * buf, ad, bd, idesc, (ks > 0 || k > 0) ? 1u : 0u);
                }
            }
            commit(&s_bar[grp][buf]);
        }
    };
    // head epilogue of `tile` from accumulator buf: comp = H2 . ReLU(u) + hb2 in
    // fp64; half hf reads features [32 hf, 32 hf + 32)
    auto epilogue = [&](long long tile, int buf) {
        mbar_wait(&s_bar[grp][buf], (phbits >> buf) & 1u);
        phbits ^= 1u << buf;
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t lb = tmem + 128 * buf + lane_off;
        const long long p0 = a.p_begin + tile * PT;
        const int np = (int)(a.p_end - p0 < PT ? a.p_end - p0 : PT);
        float u[32];
        tmem_ld32(lb + 32 * hf, u);
        // H2 . ReLU(u) as fp32 partial dots of 16 terms (their rounding is of
        // the order of the fp32 pooling's own), summed in fp64: 2 f32->f64
        // conversions per thread instead of 32 on the conversion pipe
        float dp[8];
        if (hf == 0) {
#pragma unroll
            for (int j = 0; j < 8; ++j) dp[j] = a.h2f[j] * fmaxf(u[j], 0.0f);
#pragma unroll
            for (int j = 8; j < 32; ++j) dp[j & 7] = fmaf(a.h2f[j], fmaxf(u[j], 0.0f), dp[j & 7]);
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) dp[j] = a.h2f[32 + j] * fmaxf(u[j], 0.0f);
#pragma unroll
            for (int j = 8; j < 32; ++j) dp[j & 7] = fmaf(a.h2f[32 + j], fmaxf(u[j], 0.0f), dp[j & 7]);
        }
        const double part = (double)((dp[0] + dp[1]) + (dp[2] + dp[3])) + (double)((dp[4] + dp[5]) + (dp[6] + dp[7]));
        int ddim = 0;
        bool bad = false;
        if (hf == 0) {   // warp-uniform: dims and table count of the row
            float dv[16];
            tmem_ld16(lb + 64, dv);
            ddim = (int)dv[0];
            int cnt = d < D ? (int)dv[1] : 0;
            for (int o = 1; o < (1 << LG); o <<= 1) cnt += __shfl_xor_sync(kFull, cnt, o);
            bad = cnt != Tp;   // some id of the plan lies outside 0..D-1
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        if (hf == 1) s_part[grp][r] = part;
        gbar();
        const long long p = p0 + pl;
        if (hf == 0 && pl < np && d < D) {
            a.comp[p * D + d] = ddim > 0 ? (part + s_part[grp][r]) + a.head.hb2 : 0.0;
            a.devdim[p * D + d] = ddim;
            if (d == 0) a.ok[p] = bad ? 0 : 1;
        }
    };
    // software pipeline per group: stage two tiles ahead, build + MMA one tile
    // ahead, so tile i+1's MMAs run under tile i's epilogue
    const long long tstride = (long long)gridDim.x * 2;
    long long tile = (long long)blockIdx.x * 2 + grp;
    stage(tile, 0);
    stage(tile + tstride, 1);
    if (tile < a.n_tiles) {
        asm volatile("cp.async.wait_group 1;");
        gbar();
        build_mma(tile, 0);
    }
    for (int it = 0; tile < a.n_tiles; tile += tstride, ++it) {
        const int buf = it & 1;
        if (tile + tstride < a.n_tiles) {
            asm volatile("cp.async.wait_group 0;");   // tile + 1's bytes
            gbar();
            stage(tile + 2 * tstride, buf);          // sG[buf] was read by this tile's build
            build_mma(tile + tstride, buf ^ 1);
        }
        epilogue(tile, buf);
    }
    asm volatile("cp.async.wait_group 0;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "r"(512));
}

}  // namespace

// Plan costs of rows [pb, pe) with the comm MLPs on tcgen05 (3xTF32).
// comp/devdim/ok/cost indexed by global plan index; fbuf/bbuf scratch [P][D].
ns_status launch_plan_cost_tc(ns_ctx* ctx, long long pb, long long pe, const double* comp, const int32_t* devdim,
                              const uint8_t* ok, float* fbuf, float* bbuf, double* cost) {
    const int D = ctx->model.D;
    if (D > 16) return set_err(ctx, NS_ERR_ARG, "NS_SCORE_TF32X3 supports D <= 16");
    if (pe <= pb) return NS_OK;
    TcArgs a;
    a.row_begin = pb;
    a.row_end = pe;
    a.D = D;
    a.K0p = ((2 * D + 7) / 8) * 8;
    a.N5p = 16;
    a.comp = comp;
    a.devdim = devdim;
    a.start_scale = ctx->model.start_scale;
    a.dim_scale = ctx->model.dim_scale;
    a.n_tiles = (int)((pe - pb + kTile - 1) / kTile);
    a.rflags = ctx->rflags;
    // weight floats: 2 * sum(Kp * Np)
    const int wfl = 2 * (a.K0p * 128 + 128 * 64 + 64 * 32 + 32 * 16 + 16 * 16);
    const size_t smem = (size_t)(wfl + kGroups * 2 * kABuf) * sizeof(float) + 128;
    cudaFuncSetAttribute(k_plan_mlp_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = std::min((a.n_tiles + kGroups - 1) / kGroups, ctx->sm_count);
    for (int dir = 0; dir < 2; ++dir) {
        a.dir = dir;
        a.out = dir == 0 ? fbuf : bbuf;
        for (int l = 0; l < 5; ++l) {
            a.W[l] = ctx->model.cW[dir][l];
            a.b[l] = ctx->model.cb[dir][l];
        }
        prof_begin(ctx, PK_FINALIZE);
        k_plan_mlp_tc<<<grid, 128 * kGroups, smem, ctx->stream>>>(a);
        prof_end(ctx);
        NS_LAUNCHED(ctx);
    }
    const long long n = pe - pb;
    k_plan_cost_combine<<<(unsigned)std::min<long long>((n + 255) / 256, 4096), 256, 0, ctx->stream>>>(
        comp, fbuf, bbuf, ok, pb, pe, D, cost, (ctx->rflags & NS_R11_SUM_OF_MAX) ? 1 : 0);
    NS_LAUNCHED(ctx);
    return NS_OK;
}


// Shared-memory bytes of k_pool_tc for a post-split list of Tp tables
// (0 when the tensor-core pooling does not apply).
static int pool_tc_kp(int Tp) { return ((Tp + 1 + 15) / 16) * 16; }   // + the ones column

static int pool_tc_sg(int Tp) {   // 16-byte lead-in + 64 plans + the last row's read-ahead
    const int Kp = pool_tc_kp(Tp);
    return ((16 + 64 * Tp + Kp + 16) + 15) / 16 * 16;
}

size_t pool_tc_smem(int Tp, int D) {
    if (D > 16 || Tp <= 0) return 0;
    const size_t Kp = (size_t)pool_tc_kp(Tp);
    const size_t smem = 3 * Kp * kPoolN * 2 + 4 * 128 * Kp * 2 + 2 * 2 * (size_t)pool_tc_sg(Tp);
    return smem <= 200 * 1024 ? smem : 0;
}

ns_status launch_pool_tc(ns_ctx* ctx, long long pb, long long pe, int Tp, int D, const int8_t* assign,
                         const int32_t* rows, const ns_tables* t, double* comp, int32_t* devdim, uint8_t* ok) {
    const size_t smem = pool_tc_smem(Tp, D);
    if (!smem) return set_err(ctx, NS_ERR_INTERNAL, "k_pool_tc shape");
    if (pe <= pb) return NS_OK;
    PoolTcArgs a;
    a.p_begin = pb;
    a.p_end = pe;
    a.Tp = Tp;
    a.Kp = pool_tc_kp(Tp);
    a.SG = pool_tc_sg(Tp);
    a.D = D;
    a.LG = 1;
    while ((1 << a.LG) < D) ++a.LG;
    a.assign = assign;
    a.rows = rows;
    a.V = t->d_V;
    a.vdim = t->d_vdim;
    a.comp = comp;
    a.devdim = devdim;
    a.ok = ok;
    a.head = ctx->model.head;
    for (int k = 0; k < kV; ++k) a.h2f[k] = (float)a.head.H2[k];
    const int PT = 128 >> a.LG;
    a.n_tiles = (pe - pb + PT - 1) / PT;
    cudaFuncSetAttribute(k_pool_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const long long grid = std::min<long long>((a.n_tiles + 1) / 2, ctx->sm_count);
    prof_begin(ctx, PK_SCORE);
    k_pool_tc<<<(unsigned)grid, 512, smem, ctx->stream>>>(a);
    prof_end(ctx);
    NS_LAUNCHED(ctx);
    return NS_OK;
}

}  // namespace ns
