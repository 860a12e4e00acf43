// ns_internal.cuh -- internal data structures of the NeuroShard B200 library.
// Not part of the C ABI (include/neuroshard.h is).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <set>
#include <string>
#include <vector>

#include "../../include/neuroshard.h"
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3 (ranges show up in Nsight Systems; no-ops otherwise)

namespace ns {

// NVTX range for the lifetime of a scope (public entry points, beam levels)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

constexpr int kF = 5;        // table features (reading R1)
constexpr int kH = 128;      // encoder hidden width  ("128-32")
constexpr int kE = 32;       // table representation width
constexpr int kV = 64;       // head hidden width     ("32-64")
constexpr int kDepth = 6;    // variant slots per table: dim, dim/2, ..., dim/32 (128 -> 4)
// Largest accepted table dim: a split needs dim % 8 == 0 and leaves dim/2, so a
// table of dim <= 4 << (kDepth - 1) = 128 (the paper's maximum) never
// needs more than kDepth variant rows; larger dims are rejected at validation.
constexpr int kMaxDim = 4 << (kDepth - 1);
constexpr int kMaxD = 128;   // int8 device ids
constexpr int kStats = 6;    // device counters of ns_stats ([0] scores computed by the greedy kernels)
constexpr int kCommW[6] = {0, 128, 64, 32, 16, 0};   // comm widths "128-64-32-16"

// Head weights passed by value as a kernel parameter (lands in the constant
// bank, so the greedy's DFMA reads H2[k] as a constant operand).
struct HeadParams {
    double hb1[kV];
    double H2[kV];
    double hb2;
};

struct DevModel {
    bool loaded = false;
    // compute model, fp64, device
    double* enc1W = nullptr;   // [128][5]
    double* enc1b = nullptr;   // [128]
    double* enc2W = nullptr;   // [32][128]
    double* enc2b = nullptr;   // [32]
    double* H1 = nullptr;      // [64][32]
    HeadParams head{};
    // comm models: [dir][layer] W [out][in], b [out]
    int D = 0;
    int cin[5] = {0}, cout[5] = {0};
    double* cW[2][5] = {{nullptr}};
    double* cb[2][5] = {{nullptr}};
    double start_scale = 20.0, dim_scale = 1024.0;
    uint64_t fingerprint = 0;
};

// Comm model pointers passed to kernels.
struct CommParams {
    int D;
    const double* W[2][5];
    const double* b[2][5];
    double inv_start, inv_dim;   // 1/start_scale, 1/dim_scale
};

}  // namespace ns

namespace ns {
// Per-kernel-class timers (ns_profile): CUDA events around each launch on the
// ctx stream, resolved at the next synchronising call.
struct ProfEntry {
    double total_ms = 0.0;
    uint64_t launches = 0;
};
struct ProfPending {
    int kind;
    cudaEvent_t a, b;
};
enum ProfKind { PK_PRECOMPUTE = 0, PK_VALIDATE, PK_ORDER, PK_EXPAND, PK_GREEDY, PK_FINALIZE, PK_SELECT, PK_SCORE,
                PK_OTHER, PK_COUNT };
}  // namespace ns

struct ns_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    ns::DevModel model;
    uint64_t launches = 0;
    int sm_count = 148;
    // grow-only device arena for per-call scratch
    void* arena = nullptr;
    size_t arena_bytes = 0;
    bool arena_external = false;   // ns_set_workspace: caller-owned (never grown or freed here)
    // pinned host staging (results), and a second buffer for featurise inputs
    // guarded by an event so a new featurise call never waits for the stream
    void* pinned = nullptr;
    size_t pinned_bytes = 0;
    void* pinned_in = nullptr;
    size_t pinned_in_bytes = 0;
    cudaEvent_t pinned_in_done = nullptr;
    // pinned host descriptors: H2D on a copy stream into one of two device
    // staging buffers (overlaps the previous batch's kernels), then a D2D
    // copy on the ctx stream
    cudaStream_t copy_stream = nullptr;
    void* dstage[2] = {nullptr, nullptr};
    size_t dstage_bytes[2] = {0, 0};
    cudaEvent_t dstage_ready[2] = {nullptr, nullptr};
    cudaEvent_t dstage_free[2] = {nullptr, nullptr};
    int dstage_i = 0;
    // NS_SEARCH_ASYNC with host outputs: the result copies run on out_stream
    // after out_ready (search done) and record out_done; the next search
    // waits for out_done before its kernels rewrite the staging
    cudaStream_t out_stream = nullptr;   // device -> host result copies (separate from the H2D copies)
    cudaEvent_t out_ready = nullptr;
    cudaEvent_t out_done = nullptr;
    bool out_pending = false;
    // kernel timers
    bool prof = false;
    uint32_t prof_mask = 0;   // kernel classes timed (bit k = class k)
    bool prof_open = false;   // the last prof_begin recorded an event
    ns::ProfEntry prof_acc[ns::PK_COUNT];
    std::vector<ns::ProfPending> prof_pending;
    std::vector<cudaEvent_t> prof_free;
    // multi-GPU
    void* nccl = nullptr;    // ncclComm_t (also with nranks == 1: ns_comm_init with an id)
    int nranks = 1, rank = 0;
    bool emulated = false;   // ns_comm_init(id == NULL): all ranks' blocks computed in-process (test hook)
    uint32_t rflags = 0;                     // NS_R10/R11 readings of the current search / score call
    unsigned long long* d_stats = nullptr;   // [kStats] device counters (reset by ns_profile)
    uint64_t trajectories = 0;               // greedy trajectories launched (host count)
    bool host_comm_on = false;    // ns_comm_init_host: collectives through caller callbacks on host buffers
    ns_host_comm host_comm{};
    void* comm_stage = nullptr;   // pinned staging of the host-callback collectives
    size_t comm_stage_bytes = 0;
    std::set<ns_tables*> tables;   // live ns_tables of this ctx (freed by ns_destroy)
    // validation flags of NS_SEARCH_ASYNC searches, checked by ns_synchronize
    static constexpr int kAsyncFlags = 256;
    int32_t* d_async_flags = nullptr;   // [kAsyncFlags] device copies of the tables' flags
    int32_t* h_async_flags = nullptr;   // pinned
    int n_async_flags = 0;
};

struct ns_tables {
    ns_ctx* ctx = nullptr;
    int n_tasks = 0;
    int n_tables = 0;
    int T_max = 0;
    std::vector<int32_t> off;       // [n_tasks + 1]
    std::vector<int64_t> cap;       // [n_tasks]
    std::vector<int32_t> dims;      // [n_tables] host copy (host input, or fetched lazily)
    // device
    int32_t* d_off = nullptr;
    int64_t* d_cap = nullptr;
    int64_t* d_sumdim = nullptr;    // [n_tasks] sum of dims (grid)
    int32_t* d_flag = nullptr;      // device-side descriptor validation flag
    ns_table_desc* d_desc = nullptr;
    double* d_feat = nullptr;   // [rows][5]
    double* d_V = nullptr;      // [rows][64]  v = H1 e (hb1 excluded)
    double* d_C = nullptr;      // [rows]      single-table cost C({t})
    int32_t* d_vdim = nullptr;  // [rows]      0 = invalid variant
    int64_t* d_vbytes = nullptr;// [rows]
    int32_t* d_plist = nullptr; // [rows + 1] deep-variant precompute: count, then the valid rows
    bool deep_done = false;     // variants of depth >= 1 computed
};

namespace ns {

// ---------------------------------------------------------------- kernels
// N1: featurise + encoder + hoisted head projection + single cost for rows
// (table g, depth j), j in [jlo, jhi].
void launch_precompute(ns_ctx* ctx, const ns_tables* t, int jlo, int jhi);
// descriptor validation + per-task sum of dims (device side)
void launch_tables_validate(ns_ctx* ctx, const ns_tables* t);
ns_status ensure_host_dims(ns_ctx* ctx, const ns_tables* t);
ns_status check_async_flags(ns_ctx* ctx);   // syncs the stream
ns_status record_async_flag(ns_ctx* ctx, const int32_t* d_flag);
ns_status check_tables_flag(ns_ctx* ctx, const ns_tables* t, const int32_t* host_flag);

struct SearchBufs;   // defined in k_search.cu
ns_status run_tablewise(ns_ctx* ctx, const ns_tables* t, int D, const ns_search_params* p,
                        ns_plan_batch* out);
ns_status run_columnwise(ns_ctx* ctx, const ns_tables* t, int D, const ns_search_params* p,
                         ns_plan_batch* out);
ns_status run_score_plans(ns_ctx* ctx, const ns_tables* t, int task, int D,
                          const int32_t* col_plan, int n_col, const int8_t* assign, int64_t P,
                          int mode, double* cost_out, int64_t* best_index_out,
                          double* best_cost_out);

// kernel timers (ns_api.cu): prof_begin before a launch, prof_end after it;
// prof_collect after a stream synchronisation.
void prof_begin(ns_ctx* ctx, int kind);
void prof_end(ns_ctx* ctx);
void prof_collect(ns_ctx* ctx);

// N5 (k_mlp.cu): cost[r] = max_d(comp + fwd + bwd) for rows [rb, re) with the
// comm MLPs on the FP64 tensor cores; rows with feas[r] == 0 get +inf.  With a
// row list, the rows are list[rb .. rb + *list_n) (device count), re - rb is
// the list capacity (grid size).
ns_status launch_plan_cost(ns_ctx* ctx, long long rb, long long re, const uint8_t* feas, const double* comp,
                           const int32_t* devdim, double* cost, const int32_t* list = nullptr,
                           const int32_t* list_n = nullptr);

// N5 on tcgen05 (k_score_tc.cu, NS_SCORE_TF32X3): comm MLPs in split-TF32 x3
// with FP32 accumulation in TMEM; cost[p] = max_d(comp + fwd + bwd), NaN if !ok[p].
ns_status launch_plan_cost_tc(ns_ctx* ctx, long long pb, long long pe, const double* comp, const int32_t* devdim,
                              const uint8_t* ok, float* fbuf, float* bbuf, double* cost);

// N2 on tcgen05 (k_score_tc.cu, NS_SCORE_TF32X3): per-device pooling as a
// one-hot bf16 x3 contraction; writes comp / devdim / ok like k_pool_staged.
size_t pool_tc_smem(int Tp, int D);
ns_status launch_pool_tc(ns_ctx* ctx, long long pb, long long pe, int Tp, int D, const int8_t* assign,
                         const int32_t* rows, const ns_tables* t, double* comp, int32_t* devdim, uint8_t* ok);

// helpers (ns_api.cu)
ns_status set_err(ns_ctx* ctx, ns_status s, const std::string& msg);
ns_status cuda_check(ns_ctx* ctx, cudaError_t e, const char* what);
bool is_device_ptr(const void* p);
void* arena_get(ns_ctx* ctx, size_t bytes);   // nullptr on failure
ns_status arena_error(ns_ctx* ctx, const char* what, size_t bytes);   // NS_ERR_NOMEM with the size needed
// arena bytes a search / a score call of this shape needs (ns_*_workspace_bytes)
size_t search_workspace(const ns_ctx* ctx, int n_tasks, int T_max, int D, const ns_search_params* p, bool columnwise);
size_t score_workspace(const ns_ctx* ctx, int Tp, int D, long long P, bool dev_assign);
void* pinned_get(ns_ctx* ctx, size_t bytes);
void* pinned_in_get(ns_ctx* ctx, size_t bytes);      // waits only for the previous input copy
void pinned_in_release(ns_ctx* ctx);                  // record: copies out of it are enqueued
cudaError_t ensure_copy_stream(ns_ctx* ctx);          // lazily created copy stream + its events
CommParams comm_params(const ns_ctx* ctx);
ns_status comm_allgather(ns_ctx* ctx, const void* send, void* recv, size_t bytes_per_rank);
ns_status comm_allreduce_min_u64(ns_ctx* ctx, uint64_t* dev_buf, size_t count);
ns_status comm_allreduce_max_i8(ns_ctx* ctx, int8_t* dev_buf, size_t count);
ns_status comm_alltoallv(ns_ctx* ctx, const void* send, const size_t* send_bytes, void* recv, const size_t* recv_bytes);
// true when search / score calls are collective over ranks (any backend,
// including a 1-rank NCCL communicator and emulated ranks)
bool comm_collective(const ns_ctx* ctx);
void comm_destroy(ns_ctx* ctx);


}  // namespace ns

#define NS_CUDA(ctx, call)                                                   \
    do {                                                                     \
        cudaError_t _e = (call);                                             \
        if (_e != cudaSuccess) return ns::cuda_check((ctx), _e, #call);      \
    } while (0)

#define NS_LAUNCHED(ctx)                                                     \
    do {                                                                     \
        (ctx)->launches++;                                                   \
        cudaError_t _e = cudaGetLastError();                                 \
        if (_e != cudaSuccess) return ns::cuda_check((ctx), _e, "kernel launch"); \
    } while (0)

#define NS_CHECK_LAST(ctx)                                                   \
    do {                                                                     \
        cudaError_t _e = cudaGetLastError();                                 \
        if (_e != cudaSuccess) return ns::cuda_check((ctx), _e, "kernel launch"); \
    } while (0)
