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
// Work per row: 5*128 + 128*32 + 32*64 + 64 MAC = 6.8k DFMA, run as a GEMM
// chain on the FP64 tensor cores (k_precompute_dmma in k_mlp.cu).  This file
// holds the descriptor validation that precedes it.
#include <cuda_runtime.h>

#include <algorithm>

#include "ns_internal.cuh"

namespace ns {
namespace {

// Per task: validate the descriptors (device-resident input) and sum the
// dims (sum(dim) is invariant under column splits, so the grid of
// P:289 is fixed per task).  One warp per task (grid-stride), shuffle sum.
__global__ void __launch_bounds__(256) k_tables_validate(const ns_table_desc* desc, const int32_t* off, int n_tasks,
                                                         int64_t* sumdim, int32_t* flag) {
    const int lane = threadIdx.x & 31;
    int bad = 0;
    for (int q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < n_tasks; q += (gridDim.x * blockDim.x) >> 5) {
        long long sum = 0;
        const int e = off[q + 1];
        for (int g = off[q] + lane; g < e; g += 32) {
            const ns_table_desc d = desc[g];
            bad |= (d.dim < 4 || d.dim % 4 != 0 || d.dim > kMaxDim || d.hash_size < 1 || !(d.pooling_factor > 0) ||
                    !(d.skew >= 0) || d.reserved != 0);
            sum += d.dim;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (lane == 0) sumdim[q] = sum;
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flag, 1);
}

}  // namespace

void launch_tables_validate(ns_ctx* ctx, const ns_tables* t) {
    prof_begin(ctx, PK_VALIDATE);
    const long long warps = t->n_tasks > 0 ? t->n_tasks : 1;
    const unsigned blocks = (unsigned)std::min<long long>((warps + 7) / 8, (long long)ctx->sm_count * 8);
    k_tables_validate<<<blocks, 256, 0, ctx->stream>>>(t->d_desc, t->d_off, t->n_tasks, t->d_sumdim, t->d_flag);
    prof_end(ctx);
    ctx->launches++;
}

}  // namespace ns
