// k_embag.cu -- SURVEY §8(f) row F3 (single-GPU half): the real-cost
// evaluator's computation side.  The paper measures a device's computation
// cost by running the fused embedding-bag operation of the tables placed on
// it, forward and backward, 10 warm-ups then the median of 100 runs
// (App. A.2; FBGEMM table-batched embeddings).
//
// B200 design (HBM-bound gathers):
//  * table-batched: one launch covers every table of the shard; a device-side
//    descriptor array gives each table's weights (fp32 [rows][dim], reading
//    R7's 4 bytes per element), bag offsets and indices;
//  * forward (sum pooling): a "bag group" of dim/4 lanes owns one bag
//    (sample b, table t) and streams its rows as 16-byte vectors (one 128-bit
//    load per lane per row: a 512-byte row of a dim-128 table is one
//    coalesced warp access), 4 rows in flight per lane; 32 / (dim/4) bags per
//    warp; the pooled vector goes straight to out[b][col_t ...];
//  * backward + SGD (the optimizer fused into the backward, as FBGEMM does):
//    each bag's output gradient is loaded once and -lr * grad is added to
//    every row the bag gathered with one 16-byte vector atomic
//    (red.global.add.v4.f32, sm_90+) per lane and row -- no sort, no
//    gradient buffer; rows repeated across bags (Zipf-hot rows) accumulate
//    in L2.  The summation order of repeated rows is not fixed (fp32
//    atomics), so parity is checked against an error bound, not bit-exactly.
//  * work items: a persistent grid strides over (table, bag-group) items, the
//    tables' items concatenated (per-table item offsets).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "ns_internal.cuh"

namespace ns {
namespace {

struct BagTab {
    float* W;              // [rows][dim]
    const int64_t* idx;    // [offsets[B]]
    const int32_t* off;    // [B + 1]
    long long rows;
    int dim, col;          // dimension, first output column
    int lanes, bpw;        // lanes per bag (dim / 4), bags per warp (32 / lanes)
    long long item0;       // first warp item of this table
    int cta0;              // hot backward: first CTA of this table
};

// Hot rows (backward): Zipf-like indices send a large share of a table's
// updates to a few rows (the hottest row takes 5-38% of a C2 shard table's
// lookups), and vector atomics on one address serialise in L2 -- the shard's
// backward ran 4.5x slower than with uniform indices.  Each table gets kHot
// direct-mapped hot slots (slot = hash of the row id); a detection kernel
// samples the table's indices and puts the most frequent row of each slot
// there.  The backward adds an update of a hot row to the CTA's shared-memory
// copy (red.shared) and flushes each copy once per CTA with vector atomics;
// every other row keeps the direct vector atomic.  Which rows are hot only
// changes the summation order, never the result's definition.
#ifndef NS_BAG_HOT_LOG2
#define NS_BAG_HOT_LOG2 4
#endif
constexpr int kHot = 1 << NS_BAG_HOT_LOG2;
__device__ __forceinline__ int hot_slot(long long r) {
    return (int)(((unsigned long long)r * 0x9E3779B97F4A7C15ull) >> (64 - NS_BAG_HOT_LOG2));
}

__device__ __forceinline__ int find_table(const BagTab* tabs, int n, long long item) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {   // last table with item0 <= item
        const int mid = (lo + hi + 1) >> 1;
        if (tabs[mid].item0 <= item) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

__global__ void __launch_bounds__(256) k_bag_forward(const BagTab* __restrict__ tabs, int n_tabs, long long n_items,
                                                     int B, int out_ld, float* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const long long warps = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long it = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < n_items; it += warps) {
        const int t = find_table(tabs, n_tabs, it);
        const BagTab tb = tabs[t];
        const int g = lane / tb.lanes, l = lane % tb.lanes;
        const long long b = (it - tb.item0) * tb.bpw + g;
        if (g >= tb.bpw || b >= B) continue;
        const int i0 = tb.off[b], i1 = tb.off[b + 1];
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        int i = i0;
        for (; i + 4 <= i1; i += 4) {   // 4 rows in flight
            const long long r0 = __ldg(tb.idx + i), r1 = __ldg(tb.idx + i + 1), r2 = __ldg(tb.idx + i + 2),
                            r3 = __ldg(tb.idx + i + 3);
            const float4 a0 = __ldg(reinterpret_cast<const float4*>(tb.W + r0 * tb.dim) + l);
            const float4 a1 = __ldg(reinterpret_cast<const float4*>(tb.W + r1 * tb.dim) + l);
            const float4 a2 = __ldg(reinterpret_cast<const float4*>(tb.W + r2 * tb.dim) + l);
            const float4 a3 = __ldg(reinterpret_cast<const float4*>(tb.W + r3 * tb.dim) + l);
            acc.x += a0.x; acc.y += a0.y; acc.z += a0.z; acc.w += a0.w;
            acc.x += a1.x; acc.y += a1.y; acc.z += a1.z; acc.w += a1.w;
            acc.x += a2.x; acc.y += a2.y; acc.z += a2.z; acc.w += a2.w;
            acc.x += a3.x; acc.y += a3.y; acc.z += a3.z; acc.w += a3.w;
        }
        for (; i < i1; ++i) {
            const long long r = __ldg(tb.idx + i);
            const float4 a = __ldg(reinterpret_cast<const float4*>(tb.W + r * tb.dim) + l);
            acc.x += a.x; acc.y += a.y; acc.z += a.z; acc.w += a.w;
        }
        reinterpret_cast<float4*>(out + (size_t)b * out_ld + tb.col)[l] = acc;
    }
}

__global__ void __launch_bounds__(256) k_bag_backward_sgd(const BagTab* __restrict__ tabs, int n_tabs,
                                                          long long n_items, int B, int out_ld,
                                                          const float* __restrict__ gout, float lr) {
    const int lane = threadIdx.x & 31;
    const long long warps = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long it = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < n_items; it += warps) {
        const int t = find_table(tabs, n_tabs, it);
        const BagTab tb = tabs[t];
        const int g = lane / tb.lanes, l = lane % tb.lanes;
        const long long b = (it - tb.item0) * tb.bpw + g;
        if (g >= tb.bpw || b >= B) continue;
        float4 gv = __ldg(reinterpret_cast<const float4*>(gout + (size_t)b * out_ld + tb.col) + l);
        gv.x *= -lr; gv.y *= -lr; gv.z *= -lr; gv.w *= -lr;
        const int i0 = tb.off[b], i1 = tb.off[b + 1];
        for (int i = i0; i < i1; ++i) {
            const long long r = __ldg(tb.idx + i);
            atomicAdd(reinterpret_cast<float4*>(tb.W + r * tb.dim) + l, gv);   // red.global.add.v4.f32
        }
    }
}

// One CTA per table: count a strided sample of up to 8192 of its indices in a
// shared-memory hash, then per hot slot keep the most frequent sampled row
// seen at least max(4, S / 512) times (>= ~0.2% of the lookups).
__global__ void __launch_bounds__(256) k_bag_hot_detect(const BagTab* __restrict__ tabs, int B,
                                                        long long* __restrict__ hot_keys) {
    constexpr int HS = 2048;
    __shared__ unsigned long long key[HS];
    __shared__ int cnt[HS];
    __shared__ unsigned long long best[kHot];
    const BagTab tb = tabs[blockIdx.x];
    for (int i = threadIdx.x; i < HS; i += blockDim.x) {
        key[i] = ~0ull;
        cnt[i] = 0;
    }
    if (threadIdx.x < kHot) best[threadIdx.x] = 0;
    __syncthreads();
    const long long n = tb.idx ? (long long)tb.off[B] : 0;
    const int S = (int)std::min<long long>(n, 8192);   // (blockDim.x == 256: at most 32 samples per thread)
    const long long stride = S ? n / S : 1;
    // the sampled loads are independent: issue a thread's (<= 32) loads before any insertion
    constexpr int kPer = 8192 / 256;
    unsigned long long rs[kPer];
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        const int j = threadIdx.x + q * (int)blockDim.x;
        rs[q] = j < S ? (unsigned long long)__ldg(tb.idx + (long long)j * stride) : ~0ull;
    }
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        const unsigned long long r = rs[q];
        if (r == ~0ull) continue;
        int sl = (int)((r * 0x9E3779B97F4A7C15ull) >> 53);   // 11 bits
        for (int probe = 0; probe < 32; ++probe, sl = (sl + 1) & (HS - 1)) {
            const unsigned long long prev = atomicCAS(&key[sl], ~0ull, r);
            if (prev == ~0ull || prev == r) {
                atomicAdd(&cnt[sl], 1);
                break;
            }
        }
    }
    __syncthreads();
    const int thr = max(4, S / 512);
    for (int i = threadIdx.x; i < HS; i += blockDim.x)
        if (cnt[i] >= thr) atomicMax(&best[hot_slot((long long)key[i])], ((unsigned long long)cnt[i] << 40) | key[i]);
    __syncthreads();
    if (threadIdx.x < kHot) {
        const unsigned long long b = best[threadIdx.x];
        hot_keys[(size_t)blockIdx.x * kHot + threadIdx.x] = b ? (long long)(b & ((1ull << 40) - 1)) : -1;
    }
}

// One update of row r by lane l of a bag group: into the CTA's hot-row copy if
// r is the table's hot row of its slot, else straight to the row (vector atomic).
__device__ __forceinline__ void hot_update(const long long* hk, float* hacc, float* W, int dim, int l, long long r,
                                           float4 gv) {
    const int h = hot_slot(r);
    if (hk[h] == r) {
        float* a = hacc + h * dim + 4 * l;
        atomicAdd(a, gv.x);
        atomicAdd(a + 1, gv.y);
        atomicAdd(a + 2, gv.z);
        atomicAdd(a + 3, gv.w);
    } else {
        atomicAdd(reinterpret_cast<float4*>(W + r * dim) + l, gv);   // red.global.add.v4.f32
    }
}

// Backward + SGD with the hot rows aggregated per CTA.  Each CTA works on a
// contiguous range of ONE table's warp items (table t owns CTAs
// [cta0_t, cta0_t + n_cta_t)), so its shared-memory accumulators hold only
// that table's kHot rows (kHot * dim floats <= 8 KB): occupancy stays at 8
// CTAs per SM, and no per-item table search.
__global__ void __launch_bounds__(256) k_bag_backward_sgd_hot(const BagTab* __restrict__ tabs, int n_tabs, int B,
                                                              int out_ld, const float* __restrict__ gout, float lr,
                                                              const long long* __restrict__ hot_keys,
                                                              int items_per_cta) {
    __shared__ __align__(16) float hacc[kHot * kMaxDim];
    __shared__ long long hk[kHot];
    int t = 0;
    while (t + 1 < n_tabs && tabs[t + 1].cta0 <= (int)blockIdx.x) ++t;   // few tables: linear scan
    const BagTab tb = tabs[t];
    for (int i = threadIdx.x; i < kHot * tb.dim; i += blockDim.x) hacc[i] = 0.f;
    if (threadIdx.x < kHot) hk[threadIdx.x] = __ldg(hot_keys + t * kHot + threadIdx.x);
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int g = lane / tb.lanes, l = lane % tb.lanes;
    const long long it0 = (long long)((int)blockIdx.x - tb.cta0) * items_per_cta;
    const long long it1 = std::min<long long>(it0 + items_per_cta, (B + tb.bpw - 1) / tb.bpw);
    for (long long it = it0 + w; it < it1; it += nw) {
        const long long b = it * tb.bpw + g;
        if (g >= tb.bpw || b >= B) continue;
        float4 gv = __ldg(reinterpret_cast<const float4*>(gout + (size_t)b * out_ld + tb.col) + l);
        gv.x *= -lr; gv.y *= -lr; gv.z *= -lr; gv.w *= -lr;
        const int i0 = tb.off[b], i1 = tb.off[b + 1];
        int i = i0;
        for (; i + 4 <= i1; i += 4) {   // 4 index loads in flight
            const long long r0 = __ldg(tb.idx + i), r1 = __ldg(tb.idx + i + 1), r2 = __ldg(tb.idx + i + 2),
                            r3 = __ldg(tb.idx + i + 3);
            hot_update(hk, hacc, tb.W, tb.dim, l, r0, gv);
            hot_update(hk, hacc, tb.W, tb.dim, l, r1, gv);
            hot_update(hk, hacc, tb.W, tb.dim, l, r2, gv);
            hot_update(hk, hacc, tb.W, tb.dim, l, r3, gv);
        }
        for (; i < i1; ++i) hot_update(hk, hacc, tb.W, tb.dim, l, __ldg(tb.idx + i), gv);
    }
    __syncthreads();
    // flush this CTA's hot-row sums: one vector atomic per non-zero 16-byte chunk
    const int q = tb.dim / 4;
    for (int i = threadIdx.x; i < kHot * q; i += blockDim.x) {
        const int h = i / q, c = i % q;
        const long long r = hk[h];
        if (r < 0) continue;
        const float4 v = *reinterpret_cast<const float4*>(hacc + h * tb.dim + 4 * c);
        if (v.x != 0.f || v.y != 0.f || v.z != 0.f || v.w != 0.f)
            atomicAdd(reinterpret_cast<float4*>(tb.W + r * tb.dim) + c, v);
    }
}

struct BagPlan {
    std::vector<BagTab> tabs;
    long long items = 0;
    int out_ld = 0;
};

ns_status plan_bags(ns_ctx* ctx, const ns_bag_table* t, int n, int B, BagPlan& p) {
    p.tabs.resize(n);
    int col = 0;
    for (int k = 0; k < n; ++k) {
        const ns_bag_table& s = t[k];
        if (!s.weights || !s.offsets || s.rows < 1 || s.dim < 4 || s.dim > kMaxDim || s.dim % 4 != 0)
            return set_err(ctx, NS_ERR_ARG, "ns_embedding_bag: table " + std::to_string(k) +
                                                " needs weights, offsets, rows >= 1, dim % 4 == 0 <= 128");
        // indices may be NULL when every bag of the table is empty
        if (!is_device_ptr(s.weights) || (s.indices && !is_device_ptr(s.indices)) || !is_device_ptr(s.offsets))
            return set_err(ctx, NS_ERR_ARG, "ns_embedding_bag: table buffers must be device memory");
        BagTab& b = p.tabs[k];
        b.W = s.weights;
        b.idx = s.indices;
        b.off = s.offsets;
        b.rows = s.rows;
        b.dim = s.dim;
        b.col = col;
        b.lanes = s.dim / 4;
        b.bpw = 32 / b.lanes;
        b.item0 = p.items;
        p.items += (B + b.bpw - 1) / b.bpw;
        col += s.dim;
    }
    p.out_ld = col;
    return NS_OK;
}

// descriptor array -> device (pageable source: the copy is staged before the call returns)
// (+ `extra` bytes of scratch after the descriptors, at *extra_out)
ns_status upload(ns_ctx* ctx, const BagPlan& p, BagTab** d, size_t extra = 0, void** extra_out = nullptr) {
    const size_t bytes = p.tabs.size() * sizeof(BagTab);
    const size_t off = (bytes + 255) & ~size_t(255);
    char* a = (char*)arena_get(ctx, off + extra + 256);
    if (!a) return arena_error(ctx, "ns_embedding_bag descriptors", off + extra + 256);
    NS_CUDA(ctx, cudaMemcpyAsync(a, p.tabs.data(), bytes, cudaMemcpyHostToDevice, ctx->stream));
    *d = (BagTab*)a;
    if (extra_out) *extra_out = a + off;
    return NS_OK;
}

}  // namespace
}  // namespace ns

using namespace ns;

extern "C" {

ns_status ns_embedding_bag_forward(ns_ctx* ctx, const ns_bag_table* tables, int32_t n_tables, int32_t batch,
                                   float* out) {
    if (!ctx) return NS_ERR_ARG;
    if (!tables || n_tables < 1 || batch < 1 || !out) return set_err(ctx, NS_ERR_ARG, "ns_embedding_bag_forward");
    if (!is_device_ptr(out)) return set_err(ctx, NS_ERR_ARG, "ns_embedding_bag_forward: out must be device memory");
    cudaSetDevice(ctx->device);
    BagPlan p;
    ns_status s = plan_bags(ctx, tables, n_tables, batch, p);
    if (s != NS_OK) return s;
    BagTab* d = nullptr;
    if ((s = upload(ctx, p, &d)) != NS_OK) return s;
    const unsigned blocks = (unsigned)std::min<long long>((p.items + 7) / 8, (long long)ctx->sm_count * 8);
    prof_begin(ctx, PK_OTHER);
    k_bag_forward<<<blocks, 256, 0, ctx->stream>>>(d, n_tables, p.items, batch, p.out_ld, out);
    prof_end(ctx);
    NS_LAUNCHED(ctx);
    return NS_OK;
}

ns_status ns_embedding_bag_backward_sgd(ns_ctx* ctx, const ns_bag_table* tables, int32_t n_tables, int32_t batch,
                                        const float* grad_out, float lr) {
    if (!ctx) return NS_ERR_ARG;
    if (!tables || n_tables < 1 || batch < 1 || !grad_out)
        return set_err(ctx, NS_ERR_ARG, "ns_embedding_bag_backward_sgd");
    if (!is_device_ptr(grad_out)) return set_err(ctx, NS_ERR_ARG, "ns_embedding_bag_backward_sgd: grad_out device");
    cudaSetDevice(ctx->device);
    BagPlan p;
    ns_status s = plan_bags(ctx, tables, n_tables, batch, p);
    if (s != NS_OK) return s;
    // hot-row aggregation: CTAs are assigned to tables in proportion to their
    // warp items (one table per CTA), items_per_cta chosen for ~4 waves of 8
    // CTAs per SM
    const bool hot = !getenv("NS_BAG_NO_HOT");
    int items_per_cta = 0, n_cta = 0;
    if (hot) {
        items_per_cta = (int)std::max<long long>(8, p.items / ((long long)ctx->sm_count * 8 * 4));
        for (int k = 0; k < n_tables; ++k) {
            const long long it_k = (batch + p.tabs[k].bpw - 1) / p.tabs[k].bpw;
            p.tabs[k].cta0 = n_cta;
            n_cta += (int)((it_k + items_per_cta - 1) / items_per_cta);
        }
    }
    BagTab* d = nullptr;
    void* kx = nullptr;
    if ((s = upload(ctx, p, &d, hot ? (size_t)n_tables * kHot * sizeof(long long) : 0, &kx)) != NS_OK) return s;
    prof_begin(ctx, PK_OTHER);
    if (hot) {
        long long* keys = reinterpret_cast<long long*>(kx);
        k_bag_hot_detect<<<n_tables, 256, 0, ctx->stream>>>(d, batch, keys);
        NS_LAUNCHED(ctx);
        k_bag_backward_sgd_hot<<<n_cta, 256, 0, ctx->stream>>>(d, n_tables, batch, p.out_ld, grad_out, lr, keys,
                                                               items_per_cta);
    } else {
        const unsigned blocks = (unsigned)std::min<long long>((p.items + 7) / 8, (long long)ctx->sm_count * 8);
        k_bag_backward_sgd<<<blocks, 256, 0, ctx->stream>>>(d, n_tables, p.items, batch, p.out_ld, grad_out, lr);
    }
    prof_end(ctx);
    NS_LAUNCHED(ctx);
    return NS_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- exchange
// The model-parallel embedding step of DLRM training: "each GPU
// queries the other GPUs with its sparse features to look up the embeddings
// from their tables (forward computation) and obtain the embeddings through an
// all-to-all communication (forward communication). In the backward pass, the
// gradients are sent back to the GPUs with another all-to-all communication
// (backward communication) and applied to the embeddings (backward
// computation)".  Layouts are chosen so that neither all-to-all needs a pack
// or unpack kernel: this shard's pooled rows [batch][cols[rank]] are already
// nranks contiguous per-destination blocks (sample block q goes to rank q),
// and the receive side is rank-blocked (block r = [Bl][cols[r]], Bl = batch /
// nranks), which is also the layout the backward sends from.
namespace {
ns_status exchange_sizes(ns_ctx* ctx, int batch, const int32_t* cols, int local_cols, std::vector<size_t>& mine,
                         std::vector<size_t>& theirs) {
    const int R = ctx->nranks;
    if (!cols) return set_err(ctx, NS_ERR_ARG, "exchange: cols[nranks] needed");
    if (batch % R != 0) return set_err(ctx, NS_ERR_ARG, "exchange: batch must be a multiple of nranks");
    if (cols[ctx->rank] != local_cols)
        return set_err(ctx, NS_ERR_ARG, "exchange: cols[rank] must equal the sum of this shard's dims");
    const size_t Bl = (size_t)(batch / R);
    mine.assign(R, Bl * (size_t)local_cols * sizeof(float));
    theirs.resize(R);
    for (int r = 0; r < R; ++r) {
        if (cols[r] < 0) return set_err(ctx, NS_ERR_ARG, "exchange: cols[r] < 0");
        theirs[r] = Bl * (size_t)cols[r] * sizeof(float);
    }
    return NS_OK;
}
}  // namespace

extern "C" {

ns_status ns_embedding_bag_forward_exchange(ns_ctx* ctx, const ns_bag_table* tables, int32_t n_tables, int32_t batch,
                                            const int32_t* cols, float* out, float* recv) {
    if (!ctx) return NS_ERR_ARG;
    if (!recv || !is_device_ptr(recv)) return set_err(ctx, NS_ERR_ARG, "ns_embedding_bag_forward_exchange: recv device");
    ns_status s = ns_embedding_bag_forward(ctx, tables, n_tables, batch, out);
    if (s != NS_OK) return s;
    int local = 0;
    for (int k = 0; k < n_tables; ++k) local += tables[k].dim;
    std::vector<size_t> send_b, recv_b;
    if ((s = exchange_sizes(ctx, batch, cols, local, send_b, recv_b)) != NS_OK) return s;
    return comm_alltoallv(ctx, out, send_b.data(), recv, recv_b.data());
}

ns_status ns_embedding_bag_backward_exchange_sgd(ns_ctx* ctx, const ns_bag_table* tables, int32_t n_tables,
                                                 int32_t batch, const int32_t* cols, const float* grad_recv,
                                                 float* grad_out, float lr) {
    if (!ctx) return NS_ERR_ARG;
    if (!tables || n_tables < 1 || !grad_recv || !grad_out || !is_device_ptr(grad_recv) || !is_device_ptr(grad_out))
        return set_err(ctx, NS_ERR_ARG, "ns_embedding_bag_backward_exchange_sgd: device grad_recv, grad_out");
    cudaSetDevice(ctx->device);
    int local = 0;
    for (int k = 0; k < n_tables; ++k) local += tables[k].dim;
    std::vector<size_t> mine, theirs;
    ns_status s = exchange_sizes(ctx, batch, cols, local, mine, theirs);
    if (s != NS_OK) return s;
    // the reverse exchange: block r of grad_recv goes back to rank r; rank q's
    // block lands at sample rows q * Bl ... of grad_out
    if ((s = comm_alltoallv(ctx, grad_recv, theirs.data(), grad_out, mine.data())) != NS_OK) return s;
    return ns_embedding_bag_backward_sgd(ctx, tables, n_tables, batch, grad_out, lr);
}

}  // extern "C"
