/*
 * neuroshard.h -- C ABI of the B200-native NeuroShard plan-scoring hot path.
 *
 * NeuroShard ("Pre-train and Search: Efficient Embedding Table Sharding with
 * Pre-trained Neural Cost Models", arXiv 2305.01868) shards embedding tables
 * over D GPUs by searching column-wise splits (beam search, Alg. 1) and
 * table-wise placements (greedy grid search, Alg. 2) against pre-trained
 * neural cost models used as a simulator.  Citations "P:n" are lines of the
 * paper text; "Rk" are the readings of ambiguous passages listed
 * in DESIGN.md.
 *
 * Conventions (all calls)
 *  - Every call returns an ns_status.  Negative = error: outputs are left
 *    untouched and ns_last_error(ctx) holds a message (ctx-owned string, valid
 *    until the next call on that ctx).  NS_INFEASIBLE (> 0) is data, not an
 *    error ("-" = memory explosion).
 *  - Ownership: the caller owns every array it passes; the library copies
 *    what it keeps and never frees caller memory.  Handles (ns_ctx,
 *    ns_tables) are library-owned until their destroy/free call.
 *  - Pointers documented as "host or device" may point to host memory
 *    (pageable or pinned) or to device memory of the ctx's GPU; the library
 *    detects which with cudaPointerGetAttributes and copies accordingly.
 *  - All GPU work is enqueued on the ctx stream.  Calls return after the
 *    results they write to HOST memory are complete; results written to
 *    DEVICE memory are complete when the ctx stream reaches that point.
 *  - A ctx is bound to one GPU and is not thread-safe.  One process per GPU.
 *  - Arithmetic: cost-model forward passes, greedy scores and plan costs are
 *    computed in IEEE fp64 (the oracle's precision; dense MLP layers on the
 *    FP64 tensor cores), so decisions agree with the fp64 oracle except at
 *    relative top-2 margins ~1e-15.
 */
#ifndef NEUROSHARD_H
#define NEUROSHARD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    NS_OK = 0,
    NS_INFEASIBLE = 1,        /* at least one task has no feasible plan (cost = +inf) */
    NS_ERR_ARG = -1,          /* invalid argument (NULL, out of range, shape mismatch) */
    NS_ERR_STATE = -2,        /* call order violated (e.g. no models loaded) */
    NS_ERR_NOMEM = -3,        /* device or host allocation failed */
    NS_ERR_CUDA = -4,         /* CUDA runtime error (message has the CUDA string) */
    NS_ERR_NCCL = -5,         /* NCCL error */
    NS_ERR_INTERNAL = -6
} ns_status;

typedef struct ns_ctx ns_ctx;        /* opaque; one per (process, GPU) */
typedef struct ns_tables ns_tables;  /* opaque featurised batch of sharding tasks (device-resident) */

/* ------------------------------------------------------------------ lifecycle */
/* Create a context on CUDA device `cuda_device`.  `cuda_stream` is a
 * cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream) or NULL for the
 * legacy default stream.  *out receives the handle. */
ns_status ns_create(ns_ctx** out, int cuda_device, void* cuda_stream);
/* Frees the ctx and every ns_tables it still owns (their handles become invalid). */
ns_status ns_destroy(ns_ctx* ctx);
const char* ns_last_error(const ns_ctx* ctx);
ns_status ns_set_stream(ns_ctx* ctx, void* cuda_stream);
/* Block until all work enqueued by this ctx has finished; reports a pending
 * descriptor-validation error of an NS_SEARCH_ASYNC search (NS_ERR_ARG). */
ns_status ns_synchronize(ns_ctx* ctx);
/* Number of kernels this ctx has launched since creation (bench evidence). */
uint64_t ns_kernel_launches(const ns_ctx* ctx);
/* Kernel timers: with enable == 1 every launch is bracketed by CUDA events on
 * the ctx stream; enable > 1 is a class mask (bit k + 1 times kernel class k
 * of the list below, in order, e.g. 1 << 5 = "greedy" only); 0 turns them
 * off.  ns_profile resets the accumulators.  ns_profile_query
 * returns the summed device time (ms) and launch count of one kernel class:
 * "precompute" (N1), "validate", "order", "expand" (N3), "greedy" (N4),
 * "finalize" (N5), "select" (N6), "score" (N2), "other".  Both synchronise
 * the ctx stream. */
ns_status ns_profile(ns_ctx* ctx, int32_t enable);
/* Work counters since the last ns_profile call (synchronises the ctx
 * stream): scores_computed = candidate scores the greedy kernels evaluated
 * (the grouped kernels evaluate a score once for all identical trajectories,
 * so this is <= the algorithmic count W the plans report); trajectories =
 * greedy trajectories launched (column plans x grid points); group_steps =
 * steps run by k_greedy_wgrp88 and k_greedy_p2 (D > 16, grouped);
 * scores_linear = the part of scores_computed taken in the closed linear form
 * hb2 + (A_d + B_t) (2 flops instead of 256; DESIGN.md "linear-regime
 * certificate"); replay_rows / replay_reps = rows added and representatives
 * rebuilt by k_greedy_replay (phase 2). */
typedef struct {
    uint64_t scores_computed;
    uint64_t trajectories;
    uint64_t group_steps;   /* steps the large-D grouped greedy ran (one per group and table) */
    uint64_t scores_linear;
    uint64_t replay_rows;
    uint64_t replay_reps;
} ns_stats;
ns_status ns_stats_query(ns_ctx* ctx, ns_stats* out);
ns_status ns_profile_query(ns_ctx* ctx, const char* kernel, double* total_ms, uint64_t* launches);

/* ------------------------------------------------------------- cost models */
/* One dense layer y = W x + b, torch.nn.Linear layout: W is [out][in]
 * row-major fp64, b is [out] fp64.  Host pointers. */
typedef struct {
    int32_t in, out;
    const double* W;
    const double* b;
} ns_linear;

/* Computation cost model: shared table encoder "128-32"
 * (enc[0]: F=5 -> 128, enc[1]: 128 -> 32, ReLU after both, reading R2),
 * element-wise sum over the tables of a GPU, head "32-64" (head[0]: 32 -> 64,
 * ReLU; head[1]: 64 -> 1, no output activation, reading R3). */
typedef struct {
    ns_linear enc[2];
    ns_linear head[2];
} ns_compute_model;

/* Communication cost model: MLP "128-64-32-16",
 * layer[0]: 2D -> 128, layer[1]: 128 -> 64, layer[2]: 64 -> 32,
 * layer[3]: 32 -> 16, layer[4]: 16 -> D; ReLU on hidden layers.  Input is
 * [starts_ms / start_scale (D), device_dims / dim_scale (D)], output is the
 * per-GPU cost.  One model per direction ("two separate models"). */
typedef struct {
    int32_t D;
    ns_linear layer[5];
    double start_scale;   /* 20.0 (P:788 start range 0-20 ms) */
    double dim_scale;     /* 1024.0 */
} ns_comm_model;

/* Load (copy to the GPU) the three pre-trained cost models.  Shapes are
 * validated (NS_ERR_ARG on mismatch; fwd->D must equal bwd->D, 1 <= D <= 128).
 * *fingerprint_out (may be NULL) receives an FNV-1a-64 hash of every weight
 * byte, for the version control of P:226.  Replaces previously loaded models. */
ns_status ns_load_cost_models(ns_ctx* ctx, const ns_compute_model* compute,
                              const ns_comm_model* fwd, const ns_comm_model* bwd,
                              uint64_t* fingerprint_out);

/* ------------------------------------------------------------------ tables */
/* One embedding table (P:111 factors; reading R1): dimension (columns,
 * % 4 == 0, P:237, and 4 <= dim <= 128, the paper's maximum table dim P:368:
 * every dim reachable by halving then fits the library's 6 cached variants),
 * hash size (rows), mean pooling factor, indices-distribution skew scalar. */
typedef struct {
    int32_t dim;
    int32_t reserved;     /* must be 0 */
    int64_t hash_size;
    double  pooling_factor;
    double  skew;
} ns_table_desc;

/* Featurise a batch of n_tasks sharding tasks and run the cached per-table
 * cost-model precompute (kernel N1, P:219 + table augmentation): for
 * every table at its own dim (and, lazily on the first column-wise call, at
 * every dim reachable by halving) the encoder output e, the hoisted head
 * projection v = H1 e and the single-table cost C({t}).
 *   tables       host or device, [task_offsets[n_tasks]] descriptors,
 *                task i owns tables[task_offsets[i] .. task_offsets[i+1])
 *   task_offsets host, [n_tasks + 1], task_offsets[0] == 0, each task >= 1 table
 *   mem_cap      host, [n_tasks], per-GPU memory cap in bytes (P:368 4 GB;
 *                table bytes = hash * dim * 4, reading R7)
 * Descriptors in pageable host memory are validated before the call returns
 * (NS_ERR_ARG); device-resident or pinned descriptors are copied directly and
 * validated on the GPU, an invalid one making the next synchronising call
 * (ns_shard_*, ns_score_plans, ns_synchronize) return NS_ERR_ARG.  Device and
 * pinned descriptors are read asynchronously (pinned ones on a copy stream
 * that overlaps work already queued on the ctx stream): they must stay
 * unchanged until the ctx stream has passed this call (ns_synchronize).
 * Requires loaded models.  *out is freed with ns_tables_free. */
ns_status ns_featurize_tables(ns_ctx* ctx, const ns_table_desc* tables,
                              const int32_t* task_offsets, const int64_t* mem_cap,
                              int32_t n_tasks, ns_tables** out);
ns_status ns_tables_free(ns_tables* tables);

/* Copy the per-table single costs C({t}) (fp64, [task_offsets[n_tasks]]) and,
 * if features_out != NULL, the features x ([..][5] fp64) to host memory. */
ns_status ns_tables_single_costs(ns_ctx* ctx, const ns_tables* tables,
                                 double* cost_out, double* features_out);

/* ------------------------------------------------------------ plan scoring */
typedef enum {
    NS_SCORE_FP64 = 0,    /* fp64: pooling on the FP64 pipe, comm MLPs on the FP64 tensor cores */
    NS_SCORE_TF32X3 = 1   /* bulk mode (D <= 16): comm MLPs on the tcgen05 tensor cores in
                             split-TF32 (hi*hi + hi*lo + lo*hi), FP32 accumulation in TMEM;
                             the per-device pooling on tcgen05 as a one-hot bf16 contraction
                             (v split hi + mid + lo, FP32 accumulation; T' <= 111, else SIMT
                             fp32 pooling), head epilogue in fp32 partial dots summed in fp64;
                             ~1e-6 relative plan costs (north star tolerance 1e-3).  A device
                             `assign` is read in 16-byte aligned chunks: up to 15 bytes before
                             its first and after its last plan may be read (never written) */
} ns_score_mode;

/* Simulator f(c, t) as a service ("estimate the embedding cost of any
 * sharding plan"): score P explicit plans of task `task` of `tables`.
 *   col_plan  host, [n_col] column plan c: step i halves table c_i
 *             of the evolving list and appends the second half (n_col may be 0)
 *   assign    host or device, [P][T + n_col] int8 device ids in 0..D-1
 *   cost_out  host or device, [P] fp64 plan costs (may be NULL)
 *   best_index_out / best_cost_out  host, argmin over P (lowest index on ties)
 * f = max_d(comp_d + fwd_d + bwd_d) with comp_d = C(S_d) (0 if empty),
 * fwd starts = comp - min(comp), bwd starts = 0 (readings R4, R10, R11).
 * Memory and max_dim constraints are NOT applied (any plan can be scored).
 * mode may carry NS_R10_ABS_STARTS / NS_R11_SUM_OF_MAX (alternative readings).
 * After ns_comm_init the P plans are split over the ranks and the argmin is
 * an allreduce-min over packed (cost, index) keys; cost_out then holds only
 * this rank's slice [P_begin, P_end) at its global positions. */
ns_status ns_score_plans(ns_ctx* ctx, const ns_tables* tables, int32_t task, int32_t D,
                         const int32_t* col_plan, int32_t n_col,
                         const int8_t* assign, int64_t P, int32_t mode,
                         double* cost_out, int64_t* best_index_out, double* best_cost_out);

/* ------------------------------------------------------------------ search */
/* ns_search_params.flags: which greedy kernel (N4) runs.  All variants give
 * identical results; they differ in how the M grid trajectories of a column
 * plan are mapped to lanes. */
#define NS_GREEDY_AUTO 0u     /* grouped when there are many column plans, else per-lane */
#define NS_GREEDY_GROUPED 1u  /* one warp per column plan; trajectories with identical
                                 assignment history share their scores (the paper's
                                 life-long cache, as data parallelism) */
#define NS_GREEDY_LANES 2u    /* every trajectory in its own lane segment (latency mode) */
/* May be OR-ed with the greedy selector: enqueue the search on the ctx stream
 * and return without waiting (NS_OK unless an argument/launch error).  Device
 * outputs land in ctx-stream order; host outputs are copied by a library
 * output stream once the search is done (overlapping the caller's next
 * batch), so read them after ns_synchronize (or a device-wide sync).  The
 * next call that reuses the library's staging waits for those copies on the
 * device, never on the host.  Infeasible tasks are visible
 * as +inf costs (there is no NS_INFEASIBLE status); a descriptor-validation
 * error of device-resident featurise input is returned by the next
 * ns_synchronize.  Output pointers should be device or pinned host memory
 * (pageable host outputs make the copy, and so the call, blocking). */
#define NS_SEARCH_ASYNC 4u
/* "w/o greedy grid search" (Table 3: "not grid-searching the
 * table dimension threshold"; reading R8b): the greedy runs once per column
 * plan with NO dimension threshold -- only the memory cap constrains.  Needs
 * M == 1.  (M = 1 without this flag is the single tightest threshold M_s,
 * reading R8.) */
#define NS_NO_DIM_CAP 8u
/* Alternative readings of ambiguous passages, OR-ed into
 * ns_search_params.flags (all three) or into ns_score_plans' mode (R10, R11);
 * the oracle implements the same alternatives:
 *  NS_R10_ABS_STARTS  forward comm starts = the absolute compute costs, not
 *                     comp - min comp (reading R10)
 *  NS_R11_SUM_OF_MAX  f = max comp + max fwd + max bwd ("summing up")
 *                     instead of the maximum per-device sum (R11)
 *  NS_R14_SPLITTABLE  beam candidates: top N among the splittable tables only,
 *                     not top N of all then unsplittable dropped (R14) */
#define NS_R10_ABS_STARTS 16u
#define NS_R11_SUM_OF_MAX 32u
#define NS_R14_SPLITTABLE 64u

typedef struct {
    int32_t N;               /* candidate tables per kind, default 10 */
    int32_t K;               /* beam width, default 3 */
    int32_t L;               /* split steps, default 10; ignored by tablewise */
    int32_t M;               /* grid points, default 11 */
    double  grid_hi_factor;  /* M_e = factor * M_s, default 1.5 */
    uint32_t flags;          /* NS_GREEDY_* (0 = auto) | NS_SEARCH_ASYNC | NS_NO_DIM_CAP | NS_R1x_*; other bits 0 */
} ns_search_params;

/* Per-task results.  Every pointer is host or device; only `cost` is
 * required, others may be NULL. */
typedef struct {
    double*   cost;          /* [n_tasks] best simulated cost, +inf if infeasible */
    int32_t*  n_col;         /* [n_tasks] length of the best column plan */
    int32_t*  col_plan;      /* [n_tasks][L] best column plan, -1 padded */
    int8_t*   assign;        /* [n_tasks][assign_stride] device per table of the
                                post-split list (T_i + n_col entries), -1 padded */
    int32_t   assign_stride; /* >= max_i T_i + L (tablewise: max_i T_i) */
    int32_t*  grid_index;    /* [n_tasks] winning grid point m (0..M-1), -1 if infeasible */
    uint64_t* n_scores;      /* [n_tasks] candidate scores evaluated (work W, O12) */
} ns_plan_batch;

/* Table-wise sharding only: GreedyGridSearch (Alg. 2) of every
 * task with the empty column plan.  Tasks are independent (batch axis).
 * Returns NS_INFEASIBLE if some task has no feasible grid point. */
ns_status ns_shard_tablewise(ns_ctx* ctx, const ns_tables* tables, int32_t D,
                             const ns_search_params* params, ns_plan_batch* out);

/* Column-wise + table-wise sharding: BeamSearch (Alg. 1) over
 * column plans with GreedyGridSearch as the inner loop; the empty plan is
 * evaluated first (reading R15).  After ns_comm_init, each level's
 * trajectories are partitioned over the ranks and the per-trajectory results
 * (cost, feasibility, work, duplicate link, assignment) are exchanged with
 * in-place NCCL allgathers; every rank returns identical results. */
ns_status ns_shard_columnwise(ns_ctx* ctx, const ns_tables* tables, int32_t D,
                              const ns_search_params* params, ns_plan_batch* out);

/* ------------------------------------------------------------- workspace */
/* Caller-owned device scratch (e.g. a torch.uint8 CUDA tensor).
 * By default each ctx keeps a grow-only arena of its own (cudaMalloc).  After
 * ns_set_workspace(ctx, ptr, bytes) every call carves its scratch from
 * [ptr, ptr + bytes) instead and never allocates device memory: a call whose
 * scratch does not fit returns NS_ERR_NOMEM, ns_last_error naming the bytes
 * needed.  ptr must be 256-byte aligned device memory of the ctx's device;
 * the caller keeps it alive and unchanged while the ctx may use it (until
 * ns_set_workspace(ctx, NULL, 0), which returns to the internal arena, or
 * ns_destroy).  The call synchronises the ctx stream and frees the internal
 * arena.  Sizes: ns_search_workspace_bytes for ns_shard_* on a batch of
 * n_tasks tasks whose longest table list has T_max tables (columnwise = 0
 * for ns_shard_tablewise, 1 for ns_shard_columnwise; depends on the ctx's
 * ranks), ns_score_workspace_bytes for ns_score_plans with P plans of
 * T_prime = T + n_col tables (assign_on_device: the assignments are device
 * memory).  Other calls (pre-training, embedding bag) need a few KB to MB;
 * their error message names the size. */
ns_status ns_set_workspace(ns_ctx* ctx, void* device_ptr, size_t bytes);
ns_status ns_search_workspace_bytes(ns_ctx* ctx, int32_t n_tasks, int32_t T_max, int32_t D,
                                    const ns_search_params* params, int32_t columnwise, size_t* bytes_out);
ns_status ns_score_workspace_bytes(ns_ctx* ctx, int32_t T_prime, int32_t D, int64_t P, int32_t assign_on_device,
                                   size_t* bytes_out);

/* ------------------------------------------------------------ pre-training */
/* generate cost samples and train the cost models on
 * the GPU (§3.1-3.2, App. B Alg. 3-5, App. C, App. F).  Every
 * pointer is DEVICE memory (the datasets live in HBM; NS_ERR_ARG otherwise);
 * work is enqueued on the ctx stream.  Random numbers are inputs: the caller
 * draws Alg. 4's combinations, Alg. 5's subsets and its uniforms.
 *
 * Augmented tables (Alg. 3): augmented table a is pool table
 * a / n_dims with dimension aug_dims[a % n_dims] (App. F: {4,...,128}).
 * Labels: SPEC.md's analytic cost model stands in for the
 * paper's GPU micro-benchmarks (reading F2-L in DESIGN.md).
 *
 * ns_pretrain_compute_samples: combination s (Alg. 4) = augmented tables
 *   comb_idx[comb_off[s] .. comb_off[s+1]); writes the R1 features of every
 *   table ([rows][5]) and the label launch + sum_t(gamma*overhead + work(t))
 *   (one table: launch + overhead + work) ([n]).
 * ns_pretrain_comm_samples: placement s (Alg. 5) of the augmented tables
 *   idx[off[s] .. off[s+1]) (at most 256) on D devices with per-device memory
 *   cap mem_cap: tables sorted by descending dimension (stable); table k of
 *   that order goes, if u[off[s]+k] <= p[s], to the memory-feasible device with
 *   the lowest device dimension (lowest index on ties), else to the
 *   floor(r[off[s]+k] * |feasible|)-th feasible device; no feasible device ->
 *   valid_out[s] = 0 (reading F2-P).  assign_out [rows] (per sampled table),
 *   x_out [n][2D] = [starts/20, devdim/1024] (reading R10 scaling), yf_out /
 *   yb_out [n][D] = per-device forward / backward comm labels from the
 *   starts [n][D] (ms) and device dims.
 * ns_pretrain_compute_step / ns_pretrain_comm_step: one Adam step (torch
 *   defaults, lr as given: P:789) of the MSE loss (mean over the batch; comm:
 *   over batch x D) of the computation model (theta: 7073 fp64, per layer W
 *   [out][in] then b: enc 5->128, 128->32, head 32->64, 64->1) or a comm model
 *   (2D->128->64->32->16->D) on the samples batch[0..B) (indices into the
 *   sample arrays; max_rows = the largest combination, <= 64).  t is the
 *   1-based Adam step (bias correction).  theta, adam_m, adam_v are updated in
 *   place; *loss_out (device, may be NULL) receives the batch loss before the
 *   update.  Deterministic (fixed reduction order, no atomics). */
ns_status ns_pretrain_compute_samples(ns_ctx* ctx, const ns_table_desc* pool, int32_t n_pool,
                                      const int32_t* aug_dims, int32_t n_dims, const int32_t* comb_off,
                                      const int32_t* comb_idx, int32_t n, double* feats_out, double* labels_out);
ns_status ns_pretrain_comm_samples(ns_ctx* ctx, const ns_table_desc* pool, int32_t n_pool, const int32_t* aug_dims,
                                   int32_t n_dims, int32_t D, int64_t mem_cap, const int32_t* off, const int32_t* idx,
                                   const double* p, const double* u, const double* r, const double* starts,
                                   int32_t n, double* x_out, double* yf_out, double* yb_out, int8_t* assign_out,
                                   uint8_t* valid_out);
ns_status ns_pretrain_compute_step(ns_ctx* ctx, double* theta, double* adam_m, double* adam_v, int64_t t, double lr,
                                   const double* feats, const int32_t* off, const double* labels,
                                   const int32_t* batch, int32_t B, int32_t max_rows, double* loss_out);
ns_status ns_pretrain_comm_step(ns_ctx* ctx, int32_t D, double* theta, double* adam_m, double* adam_v, int64_t t,
                                double lr, const double* x, const double* y, const int32_t* batch, int32_t B,
                                double* loss_out);

/* ------------------------------------------------------------ real-cost evaluator */
/* SURVEY §8(f) row F3, single-GPU half: the computation cost of a device's
 * shard measured by running its fused embedding-bag operation (PAPER.md:391
 * "real costs", App. A.2: forward + backward, FBGEMM
 * table-batched embeddings).  One launch covers all n_tables tables of the
 * shard (table-batched).  Every buffer is DEVICE memory:
 *   weights  [rows][dim] fp32 (4 bytes per element, reading R7), dim % 4 == 0, <= 128
 *   offsets  [batch + 1] int32: bag b of this table = indices[offsets[b] .. offsets[b+1])
 *   indices  int64 row ids in [0, rows) (not checked on the device); may be NULL
 *            when every bag of the table is empty
 * ns_embedding_bag_forward: out[b][col_t + j] = sum_{i in bag(b, t)} W_t[i][j]
 *   (sum pooling, fp32 accumulation in index order), out [batch][sum_t dim_t],
 *   tables' columns in argument order.
 * ns_embedding_bag_backward_sgd: the SGD update fused into the backward
 *   (as FBGEMM fuses the optimizer): W_t[i] -= lr * grad_out[b][col_t ...] for
 *   every occurrence of row i in bag (b, t).  Repeated rows accumulate with
 *   fp32 atomics (order not fixed: last-bit nondeterminism). */
typedef struct {
    int32_t dim;
    int32_t reserved;
    int64_t rows;
    float* weights;
    const int64_t* indices;
    const int32_t* offsets;
} ns_bag_table;
ns_status ns_embedding_bag_forward(ns_ctx* ctx, const ns_bag_table* tables, int32_t n_tables, int32_t batch,
                                   float* out);
ns_status ns_embedding_bag_backward_sgd(ns_ctx* ctx, const ns_bag_table* tables, int32_t n_tables, int32_t batch,
                                        const float* grad_out, float lr);

/* SURVEY §8(f) row F3, multi-GPU half: the model-parallel embedding step of
 * DLRM training with its two all-to-alls (forward computation,
 * forward all-to-all, backward all-to-all, backward computation; the paper
 * times each and takes the max over GPUs, App. A.3).  Collective after
 * ns_comm_init / ns_comm_init_host (host transport: needs the alltoallv
 * callback); without a communicator it is the one-rank case (the exchange is
 * a copy).  R = nranks, batch % R == 0, Bl = batch / R; cols [R] HOST int32,
 * cols[r] = sum of the dims of rank r's tables (cols[rank] must equal this
 * shard's sum).  Rank q's samples are rows q*Bl .. (q+1)*Bl - 1 of the global
 * batch.  Every buffer is DEVICE memory.
 * forward_exchange: out [batch][cols[rank]] = ns_embedding_bag_forward of this
 *   shard for the whole batch (written, and it is the send buffer: sample
 *   block q is the contiguous block sent to rank q); recv [sum_r Bl*cols[r]]
 *   rank-blocked: block r (at float offset Bl * sum_{r'<r} cols[r']) is
 *   [Bl][cols[r]], the pooled rows of rank r's tables for this rank's samples.
 * backward_exchange_sgd: grad_recv has recv's layout (the gradient w.r.t. this
 *   rank's samples' pooled rows of every rank's tables); block r goes back to
 *   rank r, the blocks from all ranks land in grad_out [batch][cols[rank]]
 *   (device scratch, written), then ns_embedding_bag_backward_sgd(grad_out).
 * Errors: NS_ERR_ARG (layout), NS_ERR_STATE (emulated ranks or a host
 * transport without alltoallv), NS_ERR_NCCL; outputs undefined on error. */
ns_status ns_embedding_bag_forward_exchange(ns_ctx* ctx, const ns_bag_table* tables, int32_t n_tables, int32_t batch,
                                            const int32_t* cols, float* out, float* recv);
ns_status ns_embedding_bag_backward_exchange_sgd(ns_ctx* ctx, const ns_bag_table* tables, int32_t n_tables,
                                                 int32_t batch, const int32_t* cols, const float* grad_recv,
                                                 float* grad_out, float lr);

/* ------------------------------------------------------------ multi-GPU */
/* 128-byte NCCL unique id (call on rank 0, broadcast by any means). */
ns_status ns_comm_unique_id(unsigned char id_out[128]);
/* Make subsequent ns_score_plans / ns_shard_* calls collective over nranks
 * processes (one GPU each): each level's column plans are split
 * into equal contiguous blocks per rank; the per-trajectory keys (cost,
 * feasibility, work, duplicate link) are allgathered so every rank runs the
 * same grid argmin / top-K / global-best selection; the winning assignment
 * lives only on the rank that computed it and reaches the others through an
 * int8 allreduce-max (the others contribute -128); finally an allreduce-min
 * over the packed per-task keys (order-preserving cost bits, plan hash) and
 * their complements certifies that every rank selected the same plan
 * (NS_ERR_INTERNAL otherwise).  nranks == 1 with an id creates a real
 * one-rank NCCL communicator (the collectives then run through NCCL);
 * nranks == 1 with id == NULL is a no-op (plain single-GPU calls).
 * id == NULL with nranks > 1 is a test hook ("emulated ranks"): this process
 * computes every rank's block itself, exercising the partitioning without
 * NCCL. */
ns_status ns_comm_init(ns_ctx* ctx, int32_t nranks, int32_t rank, const unsigned char id[128]);

/* Caller-provided transport for the collectives (e.g. MPI or a
 * torch.distributed gloo group): the library stages the data in host memory
 * and calls these from the calling thread, in the same order on every rank.
 * Each returns 0 on success (anything else -> NS_ERR_NCCL).
 *   allgather: send = this rank's bytes_per_rank bytes; recv = nranks blocks in
 *              rank order (recv + rank * bytes_per_rank may alias send).
 *   allreduce: element-wise over count elements in place; op NS_COMM_MIN_U64
 *              (uint64 minimum) or NS_COMM_MAX_I8 (int8 maximum). */
#define NS_COMM_MIN_U64 0
#define NS_COMM_MAX_I8 1
typedef struct {
    void* user;
    int (*allgather)(void* user, const void* send, void* recv, size_t bytes_per_rank);
    int (*allreduce)(void* user, void* buf, size_t count, int op);
    /* all-to-all (ns_embedding_bag_*_exchange only; may be NULL otherwise):
     * send = nranks blocks in peer order, block q (send_bytes[q] bytes) goes to
     * rank q; recv = nranks blocks in peer order, block r (recv_bytes[r] bytes)
     * comes from rank r. */
    int (*alltoallv)(void* user, const void* send, const size_t* send_bytes, void* recv, const size_t* recv_bytes);
} ns_host_comm;
/* Like ns_comm_init, with the collectives going through `comm` (copied; the
 * function pointers and user data must stay valid until the ctx is destroyed
 * or re-initialised).  Several processes may share one GPU this way (NCCL
 * refuses two ranks on one device), which is how the multi-process path is
 * tested on a one-GPU box. */
ns_status ns_comm_init_host(ns_ctx* ctx, int32_t nranks, int32_t rank, const ns_host_comm* comm);

#ifdef __cplusplus
}
#endif
#endif /* NEUROSHARD_H */
