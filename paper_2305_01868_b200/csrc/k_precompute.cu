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

}  // namespace ns
