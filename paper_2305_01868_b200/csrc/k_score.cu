// k_score.cu -- ns_score_plans: the simulator f(c, t) over P explicit plans
// ("estimate the embedding cost of any sharding plan"), kernel N2.
//
// Per plan: per-device sum pooling of the cached hoisted rows
// u_d = hb1 + sum_{t on d} v_t (P:219 element-wise sum; hoist of the head's
// first layer), comp_d = H2 ReLU(u_d) + hb2 (0 if empty, R4), then the fwd /
// bwd comm MLPs and max over devices.  fp64, one warp per plan; the
// argmin over plans is a deterministic two-stage (cost, index) reduction.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "ns_device.cuh"
#include "ns_internal.cuh"

namespace ns {

struct ScoreArgs {
    long long p_begin, p_end;
    int Tp, D;
    const int8_t* assign;     // [P][Tp] (global plan index)
    const int32_t* rows;      // [Tp] variant rows of the post-split list
    const double* V;
    const int32_t* vdim;
    double* comp;             // [P][D] (global plan index)
    int32_t* devdim;          // [P][D]
    uint8_t* ok;              // [P] 0 if the plan holds an invalid device id
    HeadParams head;
};

// Per plan (one warp): u_d = hb1 + sum_{t: a_t = d} v_t in shared memory
// (lane = features k, k+32; tables in list order), comp_d = H2 ReLU(u_d) + hb2
// for non-empty devices, 0 otherwise (R4), device dims.
__global__ void __launch_bounds__(128) k_pool(const ScoreArgs a) {
    extern __shared__ double ssm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    const int D = a.D;
    const size_t per_warp = (size_t)D * kV + (D + 1) / 2;
    double* u = ssm + (size_t)w * per_warp;     // [D][64]
    int32_t* dd = (int32_t*)(u + (size_t)D * kV);
    for (long long p = a.p_begin + (long long)blockIdx.x * wpb + w; p < a.p_end; p += (long long)gridDim.x * wpb) {
        for (int i = lane; i < D * kV; i += 32) u[i] = a.head.hb1[i % kV];
        for (int d = lane; d < D; d += 32) dd[d] = 0;
        __syncwarp();
        const int8_t* pa = a.assign + p * a.Tp;
        bool bad = false;
        for (int t = 0; t < a.Tp; ++t) {
            const int d = pa[t];
            if (d < 0 || d >= D) {   // invalid device id: the plan scores NaN
                bad = true;
                continue;
            }
            const int row = __ldg(a.rows + t);
            const double* v = a.V + (size_t)row * kV;
            u[d * kV + lane] += __ldg(v + lane);
            u[d * kV + lane + 32] += __ldg(v + lane + 32);
            if (lane == 0) dd[d] += __ldg(a.vdim + row);
        }
        __syncwarp();
        for (int d = 0; d < D; ++d) {
            double part = a.head.H2[lane] * relu_exact(u[d * kV + lane]) +
                          a.head.H2[lane + 32] * relu_exact(u[d * kV + lane + 32]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(kFull, part, o);
            if (lane == 0) {
                a.comp[p * D + d] = dd[d] > 0 ? part + a.head.hb2 : 0.0;
                a.devdim[p * D + d] = dd[d];
            }
        }
        if (lane == 0) a.ok[p] = bad ? 0 : 1;
        __syncwarp();
    }
}

__global__ void k_mark_bad(const uint8_t* ok, double* cost, long long pb, long long pe) {
    for (long long p = pb + (long long)blockIdx.x * blockDim.x + threadIdx.x; p < pe; p += (long long)gridDim.x * blockDim.x)
        if (!ok[p]) cost[p] = CUDART_NAN;
}

// Staged pooling (T' * 512 B fits in shared memory): every plan of a call
// scores the same task, so each CTA stages the task's v rows and dims once
// (coalesced).  A warp scores a plan: it reads the assignment 32 tables at a
// time (one coalesced byte load), splits the chunk by device with one ballot
// per device, and lane k accumulates features (2k, 2k+1) of every device in
// registers over that device's tables in list order -- warp-level segmented
// adds over staged rows, no read-modify-write through memory.
// Transposed butterfly over the warp for DM values per lane (all devices at
// once): at each of the first log2(DM) levels a lane keeps half of its values
// and adds the partner's copy of them, so 2*DM - 1 + (5 - log2(DM)) shuffles
// of doubles replace DM full 5-level butterflies.  Afterwards lane L holds the
// warp sum of value dev(L) = bits (4, 3, ...) of L.
template <int DM>
__device__ __forceinline__ double warp_sum_multi(double (&v)[DM], int lane) {
    constexpr int LG = DM == 1 ? 0 : DM == 2 ? 1 : DM == 4 ? 2 : DM == 8 ? 3 : 4;
    int n = DM;
#pragma unroll
    for (int l = 0; l < LG; ++l) {
        const int o = 16 >> l;
        const bool hi = (lane & o) != 0;
        n >>= 1;
#pragma unroll
        for (int i = 0; i < DM / 2; ++i) {
            if (i < n) {
                const double send = hi ? v[i] : v[i + n];
                const double keep = hi ? v[i + n] : v[i];
                v[i] = keep + __shfl_xor_sync(kFull, send, o);
            }
        }
    }
    double x = v[0];
#pragma unroll
    for (int o = 16 >> LG; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
    return x;
}

// F32 (NS_SCORE_TF32X3 only, whose comm MLPs are FP32-grade anyway): the
// staged rows and the per-device sums are fp32 -- half the shared-memory
// bytes per (plan, table) visit and FP32-pipe adds; the head epilogue runs in
// fp64 on the fp32 sums (~1e-7 relative).
template <int DM, bool F32>
__global__ void __launch_bounds__(256) k_pool_staged(const ScoreArgs a) {
    using S = std::conditional_t<F32, float, double>;
    using S2 = std::conditional_t<F32, float2, double2>;
    extern __shared__ double ssm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    const int D = a.D, Tp = a.Tp;
    S* sv = reinterpret_cast<S*>(ssm);                           // [Tp][64]
    int* sdim = (int*)(sv + (size_t)Tp * kV);                    // [Tp]
    int* sdd = sdim + Tp + 16 * w;                               // [16] this warp's per-device dims
    for (int i = threadIdx.x; i < Tp * (kV / 2); i += blockDim.x) {
        const int t = i / (kV / 2), c = i % (kV / 2);
        const int row = __ldg(a.rows + t);
        const double2 x = __ldg(reinterpret_cast<const double2*>(a.V + (size_t)row * kV) + c);
        S2 y;
        y.x = (S)x.x;
        y.y = (S)x.y;
        reinterpret_cast<S2*>(sv + (size_t)t * kV)[c] = y;
    }
    for (int t = threadIdx.x; t < Tp; t += blockDim.x) sdim[t] = __ldg(a.vdim + __ldg(a.rows + t));
    __syncthreads();
    const double hb0 = a.head.hb1[2 * lane], hb1 = a.head.hb1[2 * lane + 1];
    const double w0 = a.head.H2[2 * lane], w1 = a.head.H2[2 * lane + 1];
    constexpr int LG = DM == 1 ? 0 : DM == 2 ? 1 : DM == 4 ? 2 : DM == 8 ? 3 : 4;
    const int my_dev = (lane >> (5 - LG)) & (DM - 1);   // device whose sum lane holds after warp_sum_multi
    for (long long p = a.p_begin + (long long)blockIdx.x * wpb + w; p < a.p_end; p += (long long)gridDim.x * wpb) {
        S acc[DM][2];
#pragma unroll
        for (int d = 0; d < DM; ++d) {
            acc[d][0] = (S)hb0;
            acc[d][1] = (S)hb1;
        }
        if (lane < 16) sdd[lane] = 0;
        __syncwarp();
        bool bad = false;
        const int8_t* pa = a.assign + p * Tp;
        for (int c0 = 0; c0 < Tp; c0 += 32) {
            const int t0 = c0 + lane;
            const int my_a = t0 < Tp ? (int)pa[t0] : 0;
            const bool ok = t0 < Tp && (unsigned)my_a < (unsigned)D;
            bad |= __any_sync(kFull, t0 < Tp && !ok);
            if (ok) atomicAdd(&sdd[my_a], sdim[t0]);   // device dims (integer: order-free)
            const S2* svc = reinterpret_cast<const S2*>(sv + (size_t)c0 * kV) + lane;
#pragma unroll
            for (int d = 0; d < DM; ++d) {
                if (d >= D) break;
                unsigned m = __ballot_sync(kFull, ok && my_a == d);
                while (m) {   // this device's tables of the chunk
                    const int j = 31 - __clz(m);
                    m ^= 1u << j;
                    const S2 vv = svc[j * (kV / 2)];
                    acc[d][0] += vv.x;
                    acc[d][1] += vv.y;
                }
            }
        }
        __syncwarp();
        double part[DM];
#pragma unroll
        for (int d = 0; d < DM; ++d)
            part[d] = w0 * relu_exact((double)acc[d][0]) + w1 * relu_exact((double)acc[d][1]);
        const double sum = warp_sum_multi<DM>(part, lane);
        // one lane per device writes (the lowest lane holding it)
        if ((lane & ((32 >> LG) - 1)) == 0 && my_dev < D) {
            const int ddim = sdd[my_dev];
            a.comp[p * D + my_dev] = ddim > 0 ? sum + a.head.hb2 : 0.0;
            a.devdim[p * D + my_dev] = ddim;
        }
        if (lane == 0) a.ok[p] = bad ? 0 : 1;
        __syncwarp();
    }
}

struct BestRec {
    double cost;
    long long idx;
};

__device__ __forceinline__ bool better(double c, long long i, double bc, long long bi) {
    return c < bc || (c == bc && i < bi);
}

// stage 1: per-block lexicographic (cost, index) minimum
__global__ void k_argmin(const double* cost, long long pb, long long pe, BestRec* out) {
    __shared__ double sc[32];
    __shared__ long long si[32];
    double bc = CUDART_INF;
    long long bi = 0x7fffffffffffffffll;
    for (long long p = pb + (long long)blockIdx.x * blockDim.x + threadIdx.x; p < pe;
         p += (long long)gridDim.x * blockDim.x) {
        const double c = cost[p];
        if (better(c, p, bc, bi)) {
            bc = c;
            bi = p;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double oc = __shfl_xor_sync(kFull, bc, o);
        const long long oi = __shfl_xor_sync(kFull, bi, o);
        if (better(oc, oi, bc, bi)) {
            bc = oc;
            bi = oi;
        }
    }
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        sc[w] = bc;
        si[w] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
            if (better(sc[k], si[k], bc, bi)) {
                bc = sc[k];
                bi = si[k];
            }
        out[blockIdx.x].cost = bc;
        out[blockIdx.x].idx = bi;
    }
}

// stage 2: one thread reduces the per-block records (and the gathered ranks)
__global__ void k_argmin_final(const BestRec* in, int n, BestRec* out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double bc = CUDART_INF;
    long long bi = 0x7fffffffffffffffll;
    for (int k = 0; k < n; ++k)
        if (better(in[k].cost, in[k].idx, bc, bi)) {
            bc = in[k].cost;
            bi = in[k].idx;
        }
    out->cost = bc;
    out->idx = bi;
}

// Packed keys of the cross-rank argmin (stage 0: cost key, stage 1: index
// key, stage 2: unpack the global winner into *best).
__device__ __forceinline__ uint64_t order_key(double c) {   // monotone map double -> u64
    const uint64_t u = (uint64_t)__double_as_longlong(c);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__global__ void k_rank_key(BestRec* best, uint64_t* key, int stage) {
    if (threadIdx.x != 0) return;
    if (stage == 0) {
        key[0] = order_key(best->cost);
    } else if (stage == 1) {
        key[1] = order_key(best->cost) == key[0] ? (uint64_t)best->idx : ~0ull;
    } else {
        const uint64_t k = key[0];
        const uint64_t u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
        best->cost = __longlong_as_double((long long)u);
        best->idx = (long long)key[1];
    }
}

// Scratch of one ns_score_plans call (this rank's slice of the P plans).
size_t score_workspace(const ns_ctx* ctx, int Tp, int D, long long P, bool dev_assign) {
    const int R = ctx->emulated ? 1 : ctx->nranks;
    const long long per = (P + R - 1) / R;
    const long long pb = std::min<long long>(P, per * (ctx->emulated ? 0 : ctx->rank));
    const long long np_ = std::min<long long>(P, pb + per) - pb;
    const int nblk_arg = 296;
    size_t need = 256 + (size_t)Tp * 4 + (size_t)P * 8 + (size_t)(nblk_arg + 2 + ctx->nranks) * sizeof(BestRec) +
                  (size_t)np_ * D * 20 + (size_t)np_ + 4096;
    if (!dev_assign) need += (size_t)np_ * Tp + 256;
    return need;
}

ns_status run_score_plans(ns_ctx* ctx, const ns_tables* t, int task, int D, const int32_t* col_plan, int n_col,
                          const int8_t* assign, int64_t P, int mode, double* cost_out, int64_t* best_index_out,
                          double* best_cost_out) {
    const int T = t->off[task + 1] - t->off[task];
    const int Tp = T + n_col;
    // post-split list of variant rows; validated by the caller
    std::vector<int32_t> rows(Tp);
    for (int i = 0; i < T; ++i) rows[i] = (t->off[task] + i) * kDepth;
    for (int k = 0; k < n_col; ++k) {
        rows[col_plan[k]] += 1;
        rows[T + k] = rows[col_plan[k]];
    }
    // partition the plans over ranks (contiguous blocks)
    const int R = ctx->emulated ? 1 : ctx->nranks;   // emulated ranks: one process scores every slice
    const long long per = (P + R - 1) / R;
    const long long pb = std::min<long long>(P, per * (ctx->emulated ? 0 : ctx->rank));
    const long long pe = std::min<long long>(P, pb + per);
    const bool dev_assign = is_device_ptr(assign);
    const int nblk_arg = 296;
    const long long np_ = pe - pb;
    const size_t need = score_workspace(ctx, Tp, D, P, dev_assign);
    char* base = (char*)arena_get(ctx, need);
    if (!base) return arena_error(ctx, "score", need);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        off = (off + 255) & ~size_t(255);
        char* p = base + off;
        off += bytes;
        return p;
    };
    int32_t* d_rows = (int32_t*)take((size_t)Tp * 4);
    double* d_cost = (double*)take((size_t)P * 8);
    BestRec* d_part = (BestRec*)take((size_t)nblk_arg * sizeof(BestRec));
    BestRec* d_best = (BestRec*)take(sizeof(BestRec));
    BestRec* d_all = (BestRec*)take((size_t)ctx->nranks * sizeof(BestRec));
    double* d_comp = (double*)take((size_t)np_ * D * 8) - pb * D;        // global plan indexing
    int32_t* d_dd = (int32_t*)take((size_t)np_ * D * 4) - pb * D;
    uint8_t* d_ok = (uint8_t*)take((size_t)np_) - pb;
    float* d_fwd = mode == NS_SCORE_TF32X3 ? (float*)take((size_t)np_ * D * 4) : nullptr;
    float* d_bwd = mode == NS_SCORE_TF32X3 ? (float*)take((size_t)np_ * D * 4) : nullptr;
    const int8_t* d_assign = assign;
    if (!dev_assign && pe > pb) {
        int8_t* tmp = (int8_t*)take((size_t)np_ * Tp);
        NS_CUDA(ctx, cudaMemcpyAsync(tmp, assign + pb * Tp, (size_t)np_ * Tp, cudaMemcpyHostToDevice, ctx->stream));
        d_assign = tmp - pb * Tp;   // indexed by global plan index
    }
    NS_CUDA(ctx, cudaMemcpyAsync(d_rows, rows.data(), (size_t)Tp * 4, cudaMemcpyHostToDevice, ctx->stream));
    ScoreArgs a;
    a.p_begin = pb;
    a.p_end = pe;
    a.Tp = Tp;
    a.D = D;
    a.assign = d_assign;
    a.rows = d_rows;
    a.V = t->d_V;
    a.vdim = t->d_vdim;
    a.comp = d_comp;
    a.devdim = d_dd;
    a.ok = d_ok;
    a.head = ctx->model.head;
    if (pe > pb) {
        {
            const bool f32 = mode == NS_SCORE_TF32X3;   // fp32 pooling in the FP32-grade mode
            const size_t stage = (size_t)Tp * kV * (f32 ? sizeof(float) : sizeof(double)) + (size_t)Tp * sizeof(int) +
                                 8 * 16 * sizeof(int) + 16;
            const size_t uw = (size_t)D * kV * sizeof(double);
            (void)uw;
            if (f32 && pool_tc_smem(Tp, D) && !getenv("NS_POOL_SIMT")) {
                // one-hot bf16 x3 contraction on tcgen05 (k_score_tc.cu)
                ns_status s = launch_pool_tc(ctx, pb, pe, Tp, D, d_assign, d_rows, t, d_comp, d_dd, d_ok);
                if (s != NS_OK) return s;
            } else if (D <= 16 && stage <= 160 * 1024) {
                // staged task rows, registers per device: 8 warps per CTA
                const int wpb = 8;
                const size_t smem = stage;
                long long blocks = (np_ + wpb - 1) / wpb;
                const long long cap = (long long)ctx->sm_count * std::max<long long>(1, (long long)((200 * 1024) / smem));
                if (blocks > cap) blocks = cap;
                prof_begin(ctx, PK_SCORE);
#define NS_POOL2(DM, F)                                                                                   \
    cudaFuncSetAttribute(k_pool_staged<DM, F>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);   \
    k_pool_staged<DM, F><<<(unsigned)blocks, wpb * 32, smem, ctx->stream>>>(a);
#define NS_POOL(DM)             \
    if (f32) {                  \
        NS_POOL2(DM, true)      \
    } else {                    \
        NS_POOL2(DM, false)     \
    }
                if (D <= 2) { NS_POOL(2) } else if (D <= 4) { NS_POOL(4) } else if (D <= 8) { NS_POOL(8) } else { NS_POOL(16) }
#undef NS_POOL
#undef NS_POOL2
                prof_end(ctx);
                NS_LAUNCHED(ctx);
            } else {
                const size_t per_warp = ((size_t)D * kV + (D + 1) / 2) * sizeof(double);
                int wpb = 4;
                while (wpb > 1 && per_warp * wpb > 96 * 1024) wpb >>= 1;
                const size_t smem = per_warp * wpb;
                if (smem > 48 * 1024)
                    cudaFuncSetAttribute(k_pool, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                long long blocks = (np_ + wpb - 1) / wpb;
                const long long cap = (long long)ctx->sm_count * 16;
                if (blocks > cap) blocks = cap;
                prof_begin(ctx, PK_SCORE);
                k_pool<<<(unsigned)blocks, wpb * 32, smem, ctx->stream>>>(a);
                prof_end(ctx);
                NS_LAUNCHED(ctx);
            }
            if (mode == NS_SCORE_TF32X3) {
                ns_status s = launch_plan_cost_tc(ctx, pb, pe, d_comp, d_dd, d_ok, d_fwd - pb * D, d_bwd - pb * D, d_cost);
                if (s != NS_OK) return s;
            } else {
                ns_status s = launch_plan_cost(ctx, pb, pe, nullptr, d_comp, d_dd, d_cost);
                if (s != NS_OK) return s;
                k_mark_bad<<<(unsigned)std::min<long long>((np_ + 255) / 256, 4096), 256, 0, ctx->stream>>>(d_ok, d_cost,
                                                                                                           pb, pe);
                NS_LAUNCHED(ctx);
            }
        }
    }
    k_argmin<<<nblk_arg, 256, 0, ctx->stream>>>(d_cost, pb, pe, d_part);
    prof_end(ctx);
    NS_LAUNCHED(ctx);
    prof_begin(ctx, PK_OTHER);
    k_argmin_final<<<1, 32, 0, ctx->stream>>>(d_part, nblk_arg, d_best);
    prof_end(ctx);
    NS_LAUNCHED(ctx);
    if (comm_collective(ctx)) {   // (emulated ranks run the key stages with a no-op reduction)
        // global argmin over ranks: exact two-key NCCL allreduce-min -- first
        // the order-preserving 64-bit image of the best cost, then the lowest
        // plan index among the ranks holding that cost (lowest index on ties)
        uint64_t* d_key = reinterpret_cast<uint64_t*>(d_all);
        k_rank_key<<<1, 32, 0, ctx->stream>>>(d_best, d_key, 0);
        NS_LAUNCHED(ctx);
        ns_status s = comm_allreduce_min_u64(ctx, d_key, 1);
        if (s != NS_OK) return s;
        k_rank_key<<<1, 32, 0, ctx->stream>>>(d_best, d_key, 1);
        NS_LAUNCHED(ctx);
        if ((s = comm_allreduce_min_u64(ctx, d_key + 1, 1)) != NS_OK) return s;
        k_rank_key<<<1, 32, 0, ctx->stream>>>(d_best, d_key, 2);
        NS_LAUNCHED(ctx);
    }
    if (cost_out && pe > pb)
        NS_CUDA(ctx, cudaMemcpyAsync(cost_out + pb, d_cost + pb, (size_t)(pe - pb) * 8, cudaMemcpyDefault,
                                     ctx->stream));
    BestRec h;
    int32_t hflag = 0;
    NS_CUDA(ctx, cudaMemcpyAsync(&h, d_best, sizeof(BestRec), cudaMemcpyDeviceToHost, ctx->stream));
    NS_CUDA(ctx, cudaMemcpyAsync(&hflag, t->d_flag, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
    NS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    prof_collect(ctx);
    ns_status fs = check_tables_flag(ctx, t, &hflag);
    if (fs != NS_OK) return fs;
    if (best_index_out) *best_index_out = h.idx;
    if (best_cost_out) *best_cost_out = h.cost;
    return NS_OK;
}

}  // namespace ns
