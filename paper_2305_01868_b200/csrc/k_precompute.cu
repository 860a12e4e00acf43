// k_precompute.cu -- kernel N1: per-table cached cost-model precompute.
//
// For every table g of the batch and every column-split depth j (dim >> j,
// reachable by repeated halving, P:237 / table augmentation):
//   x = featurise(table, dim >> j)                       (reading R1)
//   e = ReLU(W2 ReLU(W1 x + b1) + b2)                    (encoder "128-32"; R2)
//   v = H1 e                                             (hoisted first head layer)
//   C({t}) = H2 ReLU(v + hb1) + hb2                       (head "32-64")
// Because the compute model sums table representations before the head
// (P:219), H1 (sum_t e_t) + hb1 = hb1 + sum_t v_t: the greedy later scores a
// device with 64-wide adds on cached v rows instead of re-running the MLP
// (SURVEY.md TL;DR 2).  All arithmetic is fp64.
//
// Work per row: 5*128 + 128*32 + 32*64 + 64 MAC = 6.8k DFMA.  Mapping: one
// warp per row, weights staged once per CTA in shared memory (transposed so
// lanes read consecutive addresses), persistent grid-stride loop.
#include <cuda_runtime.h>

#include "ns_internal.cuh"

namespace ns {
namespace {

constexpr int kWarps = 8;

struct PreArgs {
    const ns_table_desc* desc;
    int n_tables;
    int jlo, jhi;
    const double* enc1W;  // [128][5]
    const double* enc1b;
    const double* enc2W;  // [32][128]
    const double* enc2b;
    const double* H1;     // [64][32]
    HeadParams head;
    double* feat;
    double* V;
    double* C;
    int32_t* vdim;
    int64_t* vbytes;
};

__device__ __forceinline__ double relu_d(double x) { return x > 0.0 ? x : 0.0; }

__global__ void __launch_bounds__(kWarps * 32) k_precompute(const PreArgs a) {
    extern __shared__ double sm[];
    double* sW1 = sm;                      // [128][5]
    double* sb1 = sW1 + kH * kF;           // [128]
    double* sW2T = sb1 + kH;               // [128][32]  (k, o)
    double* sb2 = sW2T + kH * kE;          // [32]
    double* sH1T = sb2 + kE;               // [32][64]   (k, o)
    double* sAct = sH1T + kE * kV;         // [warps][128 + 32]
    for (int i = threadIdx.x; i < kH * kF; i += blockDim.x) sW1[i] = a.enc1W[i];
    for (int i = threadIdx.x; i < kH; i += blockDim.x) sb1[i] = a.enc1b[i];
    for (int i = threadIdx.x; i < kH * kE; i += blockDim.x) {
        int o = i / kH, k = i % kH;          // enc2W[o][k]
        sW2T[k * kE + o] = a.enc2W[i];
    }
    for (int i = threadIdx.x; i < kE; i += blockDim.x) sb2[i] = a.enc2b[i];
    for (int i = threadIdx.x; i < kV * kE; i += blockDim.x) {
        int o = i / kE, k = i % kE;          // H1[o][k]
        sH1T[k * kV + o] = a.H1[i];
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* h = sAct + warp * (kH + kE);
    double* e = h + kH;
    const int nj = a.jhi - a.jlo + 1;
    const long long nrows = (long long)a.n_tables * nj;
    for (long long r = (long long)blockIdx.x * kWarps + warp; r < nrows; r += (long long)gridDim.x * kWarps) {
        const int g = (int)(r / nj);
        const int j = a.jlo + (int)(r % nj);
        const ns_table_desc td = a.desc[g];
        // variant of depth j exists iff every ancestor dim is divisible by 8
        bool ok = true;
        int dim = td.dim;
        for (int k = 0; k < j; ++k) {
            if (dim % 8 != 0) ok = false;
            dim >>= 1;
        }
        const long long row = (long long)g * kDepth + j;
        if (!ok) {
            if (lane == 0) a.vdim[row] = 0;
            continue;
        }
        double x[kF];
        x[0] = (double)dim / 128.0;
        x[1] = log10((double)td.hash_size) / 8.0;
        x[2] = td.pooling_factor / 50.0;
        x[3] = td.skew / 2.0;
        x[4] = (double)td.hash_size * (double)dim * 4.0 / 1073741824.0;
        // layer 1: 5 -> 128, ReLU
        for (int o = lane; o < kH; o += 32) {
            double acc = 0.0;
#pragma unroll
            for (int f = 0; f < kF; ++f) acc = fma(sW1[o * kF + f], x[f], acc);
            h[o] = relu_d(acc + sb1[o]);
        }
        __syncwarp();
        // layer 2: 128 -> 32, ReLU (lane = output)
        {
            double acc = 0.0;
#pragma unroll 8
            for (int k = 0; k < kH; ++k) acc = fma(sW2T[k * kE + lane], h[k], acc);
            e[lane] = relu_d(acc + sb2[lane]);
        }
        __syncwarp();
        // hoisted head layer 1 without bias: v = H1 e (lane = outputs lane, lane+32)
        double v0 = 0.0, v1 = 0.0;
#pragma unroll 8
        for (int k = 0; k < kE; ++k) {
            const double ek = e[k];
            v0 = fma(sH1T[k * kV + lane], ek, v0);
            v1 = fma(sH1T[k * kV + lane + 32], ek, v1);
        }
        // single-table cost C({t}) = H2 ReLU(v + hb1) + hb2
        double part = a.head.H2[lane] * relu_d(v0 + a.head.hb1[lane]) +
                      a.head.H2[lane + 32] * relu_d(v1 + a.head.hb1[lane + 32]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
        a.V[row * kV + lane] = v0;
        a.V[row * kV + lane + 32] = v1;
        if (lane < kF) a.feat[row * kF + lane] = x[lane];
        if (lane == 0) {
            a.C[row] = part + a.head.hb2;
            a.vdim[row] = dim;
            a.vbytes[row] = td.hash_size * (long long)dim * 4;
        }
        __syncwarp();
    }
}

// Per task: validate the descriptors (device-resident input) and sum the
// dims (sum(dim) is invariant under column splits, so the grid of
// P:289 is fixed per task).
__global__ void k_tables_validate(const ns_table_desc* desc, const int32_t* off, int64_t* sumdim, int32_t* flag) {
    __shared__ long long s_sum;
    const int q = blockIdx.x;
    if (threadIdx.x == 0) s_sum = 0;
    __syncthreads();
    long long sum = 0;
    int bad = 0;
    for (int g = off[q] + threadIdx.x; g < off[q + 1]; g += blockDim.x) {
        const ns_table_desc d = desc[g];
        bad |= (d.dim < 4 || d.dim % 4 != 0 || d.dim > (1 << 20) || d.hash_size < 1 || !(d.pooling_factor > 0) ||
                !(d.skew >= 0) || d.reserved != 0);
        sum += d.dim;
    }
    atomicAdd((unsigned long long*)&s_sum, (unsigned long long)sum);
    if (bad) atomicOr(flag, 1);
    __syncthreads();
    if (threadIdx.x == 0) sumdim[q] = s_sum;
}

}  // namespace

void launch_tables_validate(ns_ctx* ctx, const ns_tables* t) {
    prof_begin(ctx, PK_VALIDATE);
    k_tables_validate<<<t->n_tasks, 128, 0, ctx->stream>>>(t->d_desc, t->d_off, t->d_sumdim, t->d_flag);
    prof_end(ctx);
    ctx->launches++;
}

void launch_precompute(ns_ctx* ctx, const ns_tables* t, int jlo, int jhi) {
    PreArgs a;
    a.desc = t->d_desc;
    a.n_tables = t->n_tables;
    a.jlo = jlo;
    a.jhi = jhi;
    a.enc1W = ctx->model.enc1W;
    a.enc1b = ctx->model.enc1b;
    a.enc2W = ctx->model.enc2W;
    a.enc2b = ctx->model.enc2b;
    a.H1 = ctx->model.H1;
    a.head = ctx->model.head;
    a.feat = t->d_feat;
    a.V = t->d_V;
    a.C = t->d_C;
    a.vdim = t->d_vdim;
    a.vbytes = t->d_vbytes;
    const size_t smem = sizeof(double) * (kH * kF + kH + kH * kE + kE + kE * kV + kWarps * (kH + kE));
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_precompute, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    long long rows = (long long)t->n_tables * (jhi - jlo + 1);
    long long blocks = (rows + kWarps - 1) / kWarps;
    long long cap = (long long)ctx->sm_count * 3;
    int grid = (int)(blocks < cap ? blocks : cap);
    if (grid < 1) grid = 1;
    prof_begin(ctx, PK_PRECOMPUTE);
    k_precompute<<<grid, kWarps * 32, smem, ctx->stream>>>(a);
    prof_end(ctx);
    ctx->launches++;
}

}  // namespace ns
