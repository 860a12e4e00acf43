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

}  // namespace ns
