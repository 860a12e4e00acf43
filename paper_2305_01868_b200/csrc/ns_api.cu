// ns_api.cu -- C ABI entry points (include/neuroshard.h): context, device
// arena, cost-model loading, table featurisation, argument validation and
// dispatch to the search / scoring drivers.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "ns_internal.cuh"

namespace ns {

ns_status set_err(ns_ctx* ctx, ns_status s, const std::string& msg) {
    if (ctx) ctx->err = msg;
    return s;
}

ns_status cuda_check(ns_ctx* ctx, cudaError_t e, const char* what) {
    std::string m = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
    return set_err(ctx, NS_ERR_CUDA, m);
}

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

bool is_pinned_host_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

void* arena_get(ns_ctx* ctx, size_t bytes) {
    // a previous async search's result copies (copy stream) still read the
    // arena's output staging: work enqueued from here on waits for them
    if (ctx->out_pending) {
        cudaStreamWaitEvent(ctx->stream, ctx->out_done, 0);
        ctx->out_pending = false;
    }
    if (bytes <= ctx->arena_bytes) return ctx->arena;
    if (ctx->arena_external) return nullptr;   // the caller's workspace is too small (arena_error)
    if (ctx->arena) {
        cudaStreamSynchronize(ctx->stream);
        if (ctx->out_stream) cudaStreamSynchronize(ctx->out_stream);   // result copies read the arena
        cudaFree(ctx->arena);
        ctx->arena = nullptr;
        ctx->arena_bytes = 0;
    }
    size_t want = bytes + bytes / 4 + (1 << 20);
    if (cudaMalloc(&ctx->arena, want) != cudaSuccess) {
        cudaGetLastError();
        ctx->arena = nullptr;
        return nullptr;
    }
    ctx->arena_bytes = want;
    return ctx->arena;
}

ns_status arena_error(ns_ctx* ctx, const char* what, size_t bytes) {
    std::string m = std::string("device arena (") + what + "): need " + std::to_string(bytes) + " bytes";
    if (ctx->arena_external)
        m += ", the caller workspace (ns_set_workspace) holds " + std::to_string(ctx->arena_bytes);
    return set_err(ctx, NS_ERR_NOMEM, m);
}

void* pinned_get(ns_ctx* ctx, size_t bytes) {
    if (bytes <= ctx->pinned_bytes) return ctx->pinned;
    if (ctx->pinned) {
        cudaStreamSynchronize(ctx->stream);
        cudaFreeHost(ctx->pinned);
        ctx->pinned = nullptr;
        ctx->pinned_bytes = 0;
    }
    size_t want = bytes + bytes / 4 + 4096;
    if (cudaMallocHost(&ctx->pinned, want) != cudaSuccess) {
        cudaGetLastError();
        ctx->pinned = nullptr;
        return nullptr;
    }
    ctx->pinned_bytes = want;
    return ctx->pinned;
}

void* pinned_in_get(ns_ctx* ctx, size_t bytes) {
    if (ctx->pinned_in_done) cudaEventSynchronize(ctx->pinned_in_done);   // previous copy out of the buffer
    if (bytes <= ctx->pinned_in_bytes) return ctx->pinned_in;
    if (ctx->pinned_in) cudaFreeHost(ctx->pinned_in);
    ctx->pinned_in = nullptr;
    ctx->pinned_in_bytes = 0;
    const size_t want = bytes + bytes / 4 + 4096;
    if (cudaMallocHost(&ctx->pinned_in, want) != cudaSuccess) {
        cudaGetLastError();
        ctx->pinned_in = nullptr;
        return nullptr;
    }
    ctx->pinned_in_bytes = want;
    return ctx->pinned_in;
}

// Pinned host -> device copy that overlaps work already queued on the ctx
// stream: H2D on the ctx's copy stream into staging buffer i (double
// buffered), the ctx stream waits for it and copies D2D into dst.
cudaError_t ensure_copy_stream(ns_ctx* ctx) {
    cudaError_t e;
    if (!ctx->copy_stream) {
        if ((e = cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking)) != cudaSuccess) return e;
        for (int k = 0; k < 2; ++k) {
            if ((e = cudaEventCreateWithFlags(&ctx->dstage_ready[k], cudaEventDisableTiming)) != cudaSuccess) return e;
            if ((e = cudaEventCreateWithFlags(&ctx->dstage_free[k], cudaEventDisableTiming)) != cudaSuccess) return e;
        }
        if ((e = cudaStreamCreateWithFlags(&ctx->out_stream, cudaStreamNonBlocking)) != cudaSuccess) return e;
        if ((e = cudaEventCreateWithFlags(&ctx->out_ready, cudaEventDisableTiming)) != cudaSuccess) return e;
        if ((e = cudaEventCreateWithFlags(&ctx->out_done, cudaEventDisableTiming)) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

static cudaError_t stage_pinned_h2d(ns_ctx* ctx, void* dst, const void* host, size_t bytes) {
    cudaError_t e;
    if ((e = ensure_copy_stream(ctx)) != cudaSuccess) return e;
    const int i = ctx->dstage_i;
    ctx->dstage_i ^= 1;
    if (ctx->dstage_bytes[i] < bytes) {
        if (ctx->dstage[i]) {
            cudaEventSynchronize(ctx->dstage_free[i]);
            cudaFree(ctx->dstage[i]);
            ctx->dstage[i] = nullptr;
            ctx->dstage_bytes[i] = 0;
        }
        const size_t want = bytes + bytes / 4 + 4096;
        if ((e = cudaMalloc(&ctx->dstage[i], want)) != cudaSuccess) return e;
        ctx->dstage_bytes[i] = want;
    }
    if ((e = cudaStreamWaitEvent(ctx->copy_stream, ctx->dstage_free[i], 0)) != cudaSuccess) return e;
    if ((e = cudaMemcpyAsync(ctx->dstage[i], host, bytes, cudaMemcpyHostToDevice, ctx->copy_stream)) != cudaSuccess)
        return e;
    if ((e = cudaEventRecord(ctx->dstage_ready[i], ctx->copy_stream)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(ctx->stream, ctx->dstage_ready[i], 0)) != cudaSuccess) return e;
    if ((e = cudaMemcpyAsync(dst, ctx->dstage[i], bytes, cudaMemcpyDeviceToDevice, ctx->stream)) != cudaSuccess)
        return e;
    return cudaEventRecord(ctx->dstage_free[i], ctx->stream);
}

void pinned_in_release(ns_ctx* ctx) {
    if (!ctx->pinned_in_done) cudaEventCreateWithFlags(&ctx->pinned_in_done, cudaEventDisableTiming);
    cudaEventRecord(ctx->pinned_in_done, ctx->stream);
}

CommParams comm_params(const ns_ctx* ctx) {
    CommParams c{};
    c.D = ctx->model.D;
    for (int r = 0; r < 2; ++r)
        for (int l = 0; l < 5; ++l) {
            c.W[r][l] = ctx->model.cW[r][l];
            c.b[r][l] = ctx->model.cb[r][l];
        }
    c.inv_start = 1.0 / ctx->model.start_scale;
    c.inv_dim = 1.0 / ctx->model.dim_scale;
    return c;
}

static cudaEvent_t prof_event(ns_ctx* ctx) {
    if (!ctx->prof_free.empty()) {
        cudaEvent_t e = ctx->prof_free.back();
        ctx->prof_free.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

void prof_begin(ns_ctx* ctx, int kind) {
    ctx->prof_open = false;
    if (!ctx->prof || !((ctx->prof_mask >> kind) & 1u)) return;
    ctx->prof_open = true;
    ProfPending p;
    p.kind = kind;
    p.a = prof_event(ctx);
    p.b = nullptr;
    cudaEventRecord(p.a, ctx->stream);
    ctx->prof_pending.push_back(p);
}

void prof_end(ns_ctx* ctx) {
    if (!ctx->prof || !ctx->prof_open || ctx->prof_pending.empty()) return;
    ctx->prof_open = false;
    ProfPending& p = ctx->prof_pending.back();
    p.b = prof_event(ctx);
    cudaEventRecord(p.b, ctx->stream);
}

void prof_collect(ns_ctx* ctx) {
    for (ProfPending& p : ctx->prof_pending) {
        if (p.b) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
                ctx->prof_acc[p.kind].total_ms += ms;
                ctx->prof_acc[p.kind].launches += 1;
            } else {
                cudaGetLastError();
            }
            ctx->prof_free.push_back(p.b);
        }
        ctx->prof_free.push_back(p.a);
    }
    ctx->prof_pending.clear();
}

static void free_model(ns::DevModel& m) {
    double* ps[] = {m.enc1W, m.enc1b, m.enc2W, m.enc2b, m.H1};
    for (double* p : ps)
        if (p) cudaFree(p);
    for (int r = 0; r < 2; ++r)
        for (int l = 0; l < 5; ++l) {
            if (m.cW[r][l]) cudaFree(m.cW[r][l]);
            if (m.cb[r][l]) cudaFree(m.cb[r][l]);
        }
    m = ns::DevModel();
}

static uint64_t fnv1a(uint64_t h, const void* p, size_t n) {
    const unsigned char* c = (const unsigned char*)p;
    for (size_t i = 0; i < n; ++i) {
        h ^= c[i];
        h *= 1099511628211ull;
    }
    return h;
}

}  // namespace ns

using namespace ns;

extern "C" {

ns_status ns_create(ns_ctx** out, int cuda_device, void* cuda_stream) {
    if (!out) return NS_ERR_ARG;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return NS_ERR_CUDA;
    }
    if (cuda_device < 0 || cuda_device >= n) return NS_ERR_ARG;
    ns_ctx* c = new (std::nothrow) ns_ctx();
    if (!c) return NS_ERR_NOMEM;
    c->device = cuda_device;
    c->stream = (cudaStream_t)cuda_stream;
    if (cudaSetDevice(cuda_device) != cudaSuccess) {
        delete c;
        return NS_ERR_CUDA;
    }
    cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, cuda_device);
    if (cudaMalloc((void**)&c->d_stats, ns::kStats * sizeof(unsigned long long)) != cudaSuccess ||
        cudaMemset(c->d_stats, 0, ns::kStats * sizeof(unsigned long long)) != cudaSuccess) {
        delete c;
        return NS_ERR_NOMEM;
    }
    // keep stream-ordered allocations (ns_tables buffers) cached in the pool
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, cuda_device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    *out = c;
    return NS_OK;
}

ns_status ns_destroy(ns_ctx* ctx) {
    if (!ctx) return NS_ERR_ARG;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->out_stream) cudaStreamSynchronize(ctx->out_stream);   // result copies read the arena
    while (!ctx->tables.empty()) ns_tables_free(*ctx->tables.begin());
    cudaStreamSynchronize(ctx->stream);
    free_model(ctx->model);
    if (ctx->arena && !ctx->arena_external) cudaFree(ctx->arena);
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    if (ctx->pinned_in) cudaFreeHost(ctx->pinned_in);
    if (ctx->comm_stage) cudaFreeHost(ctx->comm_stage);
    if (ctx->d_stats) cudaFree(ctx->d_stats);
    if (ctx->pinned_in_done) cudaEventDestroy(ctx->pinned_in_done);
    if (ctx->d_async_flags) cudaFree(ctx->d_async_flags);
    if (ctx->copy_stream) {
        cudaStreamSynchronize(ctx->copy_stream);
        cudaStreamDestroy(ctx->copy_stream);
    }
    for (int k = 0; k < 2; ++k) {
        if (ctx->dstage[k]) cudaFree(ctx->dstage[k]);
        if (ctx->dstage_ready[k]) cudaEventDestroy(ctx->dstage_ready[k]);
        if (ctx->dstage_free[k]) cudaEventDestroy(ctx->dstage_free[k]);
    }
    {
        if (ctx->out_stream) cudaStreamDestroy(ctx->out_stream);
        if (ctx->out_ready) cudaEventDestroy(ctx->out_ready);
        if (ctx->out_done) cudaEventDestroy(ctx->out_done);
    }
    if (ctx->h_async_flags) cudaFreeHost(ctx->h_async_flags);
    prof_collect(ctx);
    for (cudaEvent_t e : ctx->prof_free) cudaEventDestroy(e);
    comm_destroy(ctx);
    delete ctx;
    return NS_OK;
}

const char* ns_last_error(const ns_ctx* ctx) { return ctx ? ctx->err.c_str() : "null ctx"; }

ns_status ns_set_stream(ns_ctx* ctx, void* s) {
    if (!ctx) return NS_ERR_ARG;
    ctx->stream = (cudaStream_t)s;
    return NS_OK;
}

ns_status ns_synchronize(ns_ctx* ctx) {
    if (!ctx) return NS_ERR_ARG;
    cudaSetDevice(ctx->device);
    NS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    if (ctx->out_stream) NS_CUDA(ctx, cudaStreamSynchronize(ctx->out_stream));   // result copies
    ctx->out_pending = false;
    prof_collect(ctx);
    return check_async_flags(ctx);
}

uint64_t ns_kernel_launches(const ns_ctx* ctx) { return ctx ? ctx->launches : 0; }

ns_status ns_stats_query(ns_ctx* ctx, ns_stats* out) {
    if (!ctx || !out) return NS_ERR_ARG;
    cudaSetDevice(ctx->device);
    unsigned long long h[kStats];
    NS_CUDA(ctx, cudaMemcpyAsync(h, ctx->d_stats, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    NS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    out->scores_computed = h[0];
    out->trajectories = ctx->trajectories;
    out->group_steps = h[1];
    out->scores_linear = h[2];
    out->replay_rows = h[3];
    out->replay_reps = h[4];
    return NS_OK;
}

static const char* kProfNames[PK_COUNT] = {"precompute", "validate", "order", "expand", "greedy",
                                            "finalize", "select", "score", "other"};

ns_status ns_profile(ns_ctx* ctx, int32_t enable) {
    if (!ctx) return NS_ERR_ARG;
    cudaSetDevice(ctx->device);
    NS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    prof_collect(ctx);
    for (int k = 0; k < PK_COUNT; ++k) ctx->prof_acc[k] = ProfEntry();
    NS_CUDA(ctx, cudaMemsetAsync(ctx->d_stats, 0, kStats * sizeof(unsigned long long), ctx->stream));
    ctx->trajectories = 0;
    // 1: every kernel class; > 1: bit (k + 1) times class k only (fewer
    // events inside a timed region)
    ctx->prof = enable != 0;
    ctx->prof_mask = enable == 1 ? 0xffffffffu : ((uint32_t)enable >> 1);
    return NS_OK;
}

ns_status ns_profile_query(ns_ctx* ctx, const char* kernel, double* total_ms, uint64_t* launches) {
    if (!ctx || !kernel) return NS_ERR_ARG;
    cudaSetDevice(ctx->device);
    NS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    prof_collect(ctx);
    for (int k = 0; k < PK_COUNT; ++k)
        if (std::strcmp(kernel, kProfNames[k]) == 0) {
            if (total_ms) *total_ms = ctx->prof_acc[k].total_ms;
            if (launches) *launches = ctx->prof_acc[k].launches;
            return NS_OK;
        }
    return set_err(ctx, NS_ERR_ARG, std::string("unknown kernel class ") + kernel);
}

static ns_status check_linear(ns_ctx* ctx, const ns_linear& l, int in, int out, const char* name) {
    if (l.in != in || l.out != out || !l.W || !l.b)
        return set_err(ctx, NS_ERR_ARG, std::string("bad layer shape/pointers: ") + name + " expects " +
                                            std::to_string(in) + "->" + std::to_string(out));
    return NS_OK;
}

static ns_status upload(ns_ctx* ctx, double** dst, const double* src, size_t n, uint64_t* fp) {
    NS_CUDA(ctx, cudaMalloc(dst, n * sizeof(double)));
    NS_CUDA(ctx, cudaMemcpy(*dst, src, n * sizeof(double), cudaMemcpyHostToDevice));
    *fp = fnv1a(*fp, src, n * sizeof(double));
    return NS_OK;
}

ns_status ns_load_cost_models(ns_ctx* ctx, const ns_compute_model* cm, const ns_comm_model* fwd,
                              const ns_comm_model* bwd, uint64_t* fingerprint_out) {
    if (!ctx) return NS_ERR_ARG;
    if (!cm || !fwd || !bwd) return set_err(ctx, NS_ERR_ARG, "null model");
    ns_status s;
    if ((s = check_linear(ctx, cm->enc[0], kF, kH, "enc[0]")) != NS_OK) return s;
    if ((s = check_linear(ctx, cm->enc[1], kH, kE, "enc[1]")) != NS_OK) return s;
    if ((s = check_linear(ctx, cm->head[0], kE, kV, "head[0]")) != NS_OK) return s;
    if ((s = check_linear(ctx, cm->head[1], kV, 1, "head[1]")) != NS_OK) return s;
    int D = fwd->D;
    if (D < 1 || D > kMaxD || bwd->D != D)
        return set_err(ctx, NS_ERR_ARG, "comm models: need 1 <= D <= 128 and fwd.D == bwd.D");
    const ns_comm_model* cms[2] = {fwd, bwd};
    int widths[6] = {2 * D, 128, 64, 32, 16, D};
    for (int r = 0; r < 2; ++r) {
        for (int l = 0; l < 5; ++l)
            if ((s = check_linear(ctx, cms[r]->layer[l], widths[l], widths[l + 1], "comm layer")) != NS_OK)
                return s;
        if (!(cms[r]->start_scale > 0) || !(cms[r]->dim_scale > 0))
            return set_err(ctx, NS_ERR_ARG, "comm scales must be > 0");
    }
    if (fwd->start_scale != bwd->start_scale || fwd->dim_scale != bwd->dim_scale)
        return set_err(ctx, NS_ERR_ARG, "fwd/bwd comm scales must match");
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    free_model(ctx->model);
    DevModel& m = ctx->model;
    uint64_t fp = 1469598103934665603ull;
    if ((s = upload(ctx, &m.enc1W, cm->enc[0].W, kH * kF, &fp)) != NS_OK) return s;
    if ((s = upload(ctx, &m.enc1b, cm->enc[0].b, kH, &fp)) != NS_OK) return s;
    if ((s = upload(ctx, &m.enc2W, cm->enc[1].W, kE * kH, &fp)) != NS_OK) return s;
    if ((s = upload(ctx, &m.enc2b, cm->enc[1].b, kE, &fp)) != NS_OK) return s;
    if ((s = upload(ctx, &m.H1, cm->head[0].W, kV * kE, &fp)) != NS_OK) return s;
    for (int k = 0; k < kV; ++k) {
        m.head.hb1[k] = cm->head[0].b[k];
        m.head.H2[k] = cm->head[1].W[k];
    }
    m.head.hb2 = cm->head[1].b[0];
    fp = fnv1a(fp, m.head.hb1, sizeof(m.head.hb1));
    fp = fnv1a(fp, m.head.H2, sizeof(m.head.H2));
    fp = fnv1a(fp, &m.head.hb2, sizeof(double));
    m.D = D;
    for (int l = 0; l < 5; ++l) {
        m.cin[l] = widths[l];
        m.cout[l] = widths[l + 1];
    }
    for (int r = 0; r < 2; ++r)
        for (int l = 0; l < 5; ++l) {
            size_t nw = (size_t)widths[l] * widths[l + 1];
            if ((s = upload(ctx, &m.cW[r][l], cms[r]->layer[l].W, nw, &fp)) != NS_OK) return s;
            if ((s = upload(ctx, &m.cb[r][l], cms[r]->layer[l].b, widths[l + 1], &fp)) != NS_OK) return s;
        }
    m.start_scale = fwd->start_scale;
    m.dim_scale = fwd->dim_scale;
    fp = fnv1a(fp, &m.start_scale, sizeof(double));
    fp = fnv1a(fp, &m.dim_scale, sizeof(double));
    m.fingerprint = fp;
    m.loaded = true;
    if (fingerprint_out) *fingerprint_out = fp;
    return NS_OK;
}

ns_status ns_featurize_tables(ns_ctx* ctx, const ns_table_desc* tables, const int32_t* task_offsets,
                              const int64_t* mem_cap, int32_t n_tasks, ns_tables** out) {
    NvtxRange nvtx_("ns_featurize_tables");
    if (!ctx) return NS_ERR_ARG;
    if (!out || !tables || !task_offsets || !mem_cap || n_tasks < 1)
        return set_err(ctx, NS_ERR_ARG, "ns_featurize_tables: null argument or n_tasks < 1");
    *out = nullptr;
    if (!ctx->model.loaded) return set_err(ctx, NS_ERR_STATE, "ns_featurize_tables: no cost models loaded");
    if (task_offsets[0] != 0) return set_err(ctx, NS_ERR_ARG, "task_offsets[0] must be 0");
    int T_max = 0;
    for (int i = 0; i < n_tasks; ++i) {
        int T = task_offsets[i + 1] - task_offsets[i];
        if (T < 1) return set_err(ctx, NS_ERR_ARG, "every task needs >= 1 table");
        if (mem_cap[i] <= 0) return set_err(ctx, NS_ERR_ARG, "mem_cap must be > 0");
        T_max = T > T_max ? T : T_max;
    }
    const int n = task_offsets[n_tasks];
    cudaSetDevice(ctx->device);
    const bool dev_in = is_device_ptr(tables);
    // pinned host descriptors are DMA'd directly and validated on the device
    // like device-resident ones (no host pass over the batch)
    const bool pinned_in = !dev_in && is_pinned_host_ptr(tables);
    const bool direct = dev_in || pinned_in;
    ns_tables* t = new (std::nothrow) ns_tables();
    if (!t) return set_err(ctx, NS_ERR_NOMEM, "host alloc");
    t->ctx = ctx;
    t->n_tasks = n_tasks;
    t->n_tables = n;
    t->T_max = T_max;
    t->off.assign(task_offsets, task_offsets + n_tasks + 1);
    t->cap.assign(mem_cap, mem_cap + n_tasks);
    if (!direct) {
        // pageable host descriptors: validate here; device / pinned descriptors
        // are validated by the k_tables_validate kernel and reported at the next
        // synchronising call
        t->dims.resize(n);
        for (int g = 0; g < n; ++g) {
            const ns_table_desc& d = tables[g];
            if (d.dim < 4 || d.dim % 4 != 0 || d.dim > kMaxDim || d.hash_size < 1 || !(d.pooling_factor > 0) ||
                !(d.skew >= 0) || d.reserved != 0) {
                delete t;
                return set_err(ctx, NS_ERR_ARG, "invalid table descriptor " + std::to_string(g) +
                                                    " (need dim%4==0, 4<=dim<=128, hash>=1, pooling>0, skew>=0)");
            }
            t->dims[g] = d.dim;
        }
    }
    size_t rows = (size_t)n * kDepth;
    cudaStream_t st = ctx->stream;
    auto fail = [&](cudaError_t e) {
        ns_tables_free(t);
        return cuda_check(ctx, e, "ns_featurize_tables alloc/copy");
    };
    cudaError_t e;
#define NS_TALLOC(ptr, bytes) \
    if ((e = cudaMallocAsync((void**)&(ptr), (bytes), st)) != cudaSuccess) return fail(e);
    NS_TALLOC(t->d_off, (n_tasks + 1) * sizeof(int32_t));
    NS_TALLOC(t->d_cap, n_tasks * sizeof(int64_t));
    NS_TALLOC(t->d_sumdim, n_tasks * sizeof(int64_t));
    NS_TALLOC(t->d_desc, n * sizeof(ns_table_desc));
    NS_TALLOC(t->d_feat, rows * kF * sizeof(double));
    NS_TALLOC(t->d_V, rows * kV * sizeof(double));
    NS_TALLOC(t->d_C, rows * sizeof(double));
    NS_TALLOC(t->d_vdim, rows * sizeof(int32_t));
    NS_TALLOC(t->d_vbytes, rows * sizeof(int64_t));
    NS_TALLOC(t->d_plist, (rows + 1) * sizeof(int32_t));
    NS_TALLOC(t->d_flag, sizeof(int32_t));
#undef NS_TALLOC
    // small host arrays go through pinned staging so the copies stay async
    const size_t meta = (n_tasks + 1) * sizeof(int32_t) + n_tasks * sizeof(int64_t);
    const size_t hbytes = meta + (direct ? 0 : (size_t)n * sizeof(ns_table_desc));
    char* pin = (char*)pinned_in_get(ctx, hbytes + 64);
    if (!pin) {
        ns_tables_free(t);
        return set_err(ctx, NS_ERR_NOMEM, "pinned staging");
    }
    std::memcpy(pin, task_offsets, (n_tasks + 1) * sizeof(int32_t));
    std::memcpy(pin + (n_tasks + 1) * sizeof(int32_t), mem_cap, n_tasks * sizeof(int64_t));
    if (!direct) std::memcpy(pin + meta, tables, (size_t)n * sizeof(ns_table_desc));
    if ((e = cudaMemcpyAsync(t->d_off, pin, (n_tasks + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, st)) !=
        cudaSuccess)
        return fail(e);
    if ((e = cudaMemcpyAsync(t->d_cap, pin + (n_tasks + 1) * sizeof(int32_t), n_tasks * sizeof(int64_t),
                             cudaMemcpyHostToDevice, st)) != cudaSuccess)
        return fail(e);
    if (pinned_in) {
        if ((e = stage_pinned_h2d(ctx, t->d_desc, tables, n * sizeof(ns_table_desc))) != cudaSuccess) return fail(e);
    } else if ((e = cudaMemcpyAsync(t->d_desc, dev_in ? (const void*)tables : (const void*)(pin + meta),
                                    n * sizeof(ns_table_desc),
                                    dev_in ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st)) != cudaSuccess) {
        return fail(e);
    }
    pinned_in_release(ctx);   // the staging buffer may be reused once these copies ran
    // (vdim of every row is written by the precompute of its depth before any read)
    if ((e = cudaMemsetAsync(t->d_flag, 0, sizeof(int32_t), st)) != cudaSuccess) return fail(e);
    launch_tables_validate(ctx, t);
    launch_precompute(ctx, t, 0, 0);
    if ((e = cudaGetLastError()) != cudaSuccess) return fail(e);
    ctx->tables.insert(t);
    *out = t;
    return NS_OK;
}

ns_status ns_tables_free(ns_tables* t) {
    if (!t) return NS_ERR_ARG;
    if (t->ctx) t->ctx->tables.erase(t);
    cudaStream_t st = t->ctx ? t->ctx->stream : nullptr;
    if (t->ctx) cudaSetDevice(t->ctx->device);
    void* ps[] = {t->d_off, t->d_cap, t->d_sumdim, t->d_desc, t->d_feat, t->d_V, t->d_C, t->d_vdim, t->d_vbytes,
                  t->d_flag, t->d_plist};
    for (void* p : ps)
        if (p) cudaFreeAsync(p, st);
    delete t;
    return NS_OK;
}

}  // extern "C"

namespace ns {
// Host copy of the table dims (validation of column plans); fetched lazily
// when the descriptors were device-resident.
ns_status ensure_host_dims(ns_ctx* ctx, const ns_tables* t) {
    if ((int)t->dims.size() == t->n_tables) return NS_OK;
    std::vector<ns_table_desc> h(t->n_tables);
    NS_CUDA(ctx, cudaMemcpyAsync(h.data(), t->d_desc, h.size() * sizeof(ns_table_desc), cudaMemcpyDeviceToHost,
                                 ctx->stream));
    NS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    ns_tables* m = const_cast<ns_tables*>(t);
    m->dims.resize(t->n_tables);
    for (int g = 0; g < t->n_tables; ++g) m->dims[g] = h[g].dim;
    return NS_OK;
}

// NS_SEARCH_ASYNC: the tables' validation flag is copied (stream-ordered) into
// a ctx slot; ns_synchronize checks every recorded slot.
ns_status record_async_flag(ns_ctx* ctx, const int32_t* d_flag) {
    if (!ctx->d_async_flags) {
        NS_CUDA(ctx, cudaMalloc(&ctx->d_async_flags, ns_ctx::kAsyncFlags * sizeof(int32_t)));
        NS_CUDA(ctx, cudaMallocHost(&ctx->h_async_flags, ns_ctx::kAsyncFlags * sizeof(int32_t)));
    }
    if (ctx->n_async_flags == ns_ctx::kAsyncFlags) {   // full: check (and empty) now
        ns_status s = check_async_flags(ctx);
        if (s != NS_OK) return s;
    }
    NS_CUDA(ctx, cudaMemcpyAsync(ctx->d_async_flags + ctx->n_async_flags++, d_flag, sizeof(int32_t),
                                 cudaMemcpyDeviceToDevice, ctx->stream));
    return NS_OK;
}

ns_status check_async_flags(ns_ctx* ctx) {
    const int n = ctx->n_async_flags;
    if (n == 0) return NS_OK;
    ctx->n_async_flags = 0;
    NS_CUDA(ctx, cudaMemcpyAsync(ctx->h_async_flags, ctx->d_async_flags, n * sizeof(int32_t), cudaMemcpyDeviceToHost,
                                 ctx->stream));
    NS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    for (int i = 0; i < n; ++i) {
        ns_status s = check_tables_flag(ctx, nullptr, ctx->h_async_flags + i);
        if (s != NS_OK) return s;
    }
    return NS_OK;
}

// Device-side validation flag of the descriptors (set by k_tables_validate).
ns_status check_tables_flag(ns_ctx* ctx, const ns_tables* t, const int32_t* host_flag) {
    (void)t;
    if (*host_flag & 2)   // set by the multi-rank consistency check (k_search.cu, k_rank_check)
        return set_err(ctx, NS_ERR_INTERNAL, "ranks selected different plans (multi-rank consistency check)");
    if (*host_flag != 0)
        return set_err(ctx, NS_ERR_ARG,
                       "invalid table descriptor in device-resident input (need dim%4==0, dim>=4, hash>=1, "
                       "pooling>0, skew>=0, reserved==0)");
    return NS_OK;
}
}  // namespace ns

extern "C" {

ns_status ns_tables_single_costs(ns_ctx* ctx, const ns_tables* t, double* cost_out, double* features_out) {
    if (!ctx || !t || !cost_out) return set_err(ctx, NS_ERR_ARG, "null argument");
    cudaSetDevice(ctx->device);
    // depth-0 rows are g*kDepth
    NS_CUDA(ctx, cudaMemcpy2DAsync(cost_out, sizeof(double), t->d_C, kDepth * sizeof(double), sizeof(double),
                                   t->n_tables, cudaMemcpyDeviceToHost, ctx->stream));
    if (features_out)
        NS_CUDA(ctx, cudaMemcpy2DAsync(features_out, kF * sizeof(double), t->d_feat, kDepth * kF * sizeof(double),
                                       kF * sizeof(double), t->n_tables, cudaMemcpyDeviceToHost, ctx->stream));
    NS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return NS_OK;
}

static ns_status check_search(ns_ctx* ctx, const ns_tables* t, int D, const ns_search_params* p,
                              ns_plan_batch* out, bool columnwise) {
    if (!ctx) return NS_ERR_ARG;
    if (!t || !p || !out || !out->cost) return set_err(ctx, NS_ERR_ARG, "null argument (tables/params/out/cost)");
    if (t->ctx != ctx) return set_err(ctx, NS_ERR_ARG, "tables belong to another ctx");
    if (!ctx->model.loaded) return set_err(ctx, NS_ERR_STATE, "no cost models loaded");
    if (D != ctx->model.D) return set_err(ctx, NS_ERR_ARG, "D differs from the loaded comm models' D");
    if (p->M < 1 || p->M > 4096) return set_err(ctx, NS_ERR_ARG, "need 1 <= M <= 4096");
    if (!(p->grid_hi_factor >= 1.0) ||
        (p->flags & ~(NS_SEARCH_ASYNC | NS_NO_DIM_CAP | NS_R10_ABS_STARTS | NS_R11_SUM_OF_MAX | NS_R14_SPLITTABLE)) >
            NS_GREEDY_LANES)
        return set_err(ctx, NS_ERR_ARG, "bad grid_hi_factor/flags");
    if ((p->flags & NS_NO_DIM_CAP) && p->M != 1) return set_err(ctx, NS_ERR_ARG, "NS_NO_DIM_CAP needs M == 1");
    if (columnwise) {
        if (p->N < 1 || p->K < 1 || p->L < 0 || p->L > 64 || p->N > 512 || p->K > 512)
            return set_err(ctx, NS_ERR_ARG, "need N,K in [1,512], L in [0,64]");
    }
    int L = columnwise ? p->L : 0;
    if (out->assign && out->assign_stride < t->T_max + L)
        return set_err(ctx, NS_ERR_ARG, "assign_stride < T_max + L");
    if (t->T_max + L > 8192) return set_err(ctx, NS_ERR_ARG, "T + L > 8192 not supported");
    return NS_OK;
}

ns_status ns_shard_tablewise(ns_ctx* ctx, const ns_tables* t, int32_t D, const ns_search_params* p,
                             ns_plan_batch* out) {
    NvtxRange nvtx_("ns_shard_tablewise");
    ns_status s = check_search(ctx, t, D, p, out, false);
    if (s != NS_OK) return s;
    cudaSetDevice(ctx->device);
    return run_tablewise(ctx, t, D, p, out);
}

ns_status ns_shard_columnwise(ns_ctx* ctx, const ns_tables* t, int32_t D, const ns_search_params* p,
                              ns_plan_batch* out) {
    NvtxRange nvtx_("ns_shard_columnwise");
    ns_status s = check_search(ctx, t, D, p, out, true);
    if (s != NS_OK) return s;
    cudaSetDevice(ctx->device);
    if (!t->deep_done) {
        launch_precompute(ctx, t, 1, kDepth - 1);
        NS_CHECK_LAST(ctx);
        const_cast<ns_tables*>(t)->deep_done = true;
    }
    return run_columnwise(ctx, t, D, p, out);
}

ns_status ns_score_plans(ns_ctx* ctx, const ns_tables* t, int32_t task, int32_t D, const int32_t* col_plan,
                         int32_t n_col, const int8_t* assign, int64_t P, int32_t mode, double* cost_out,
                         int64_t* best_index_out, double* best_cost_out) {
    NvtxRange nvtx_("ns_score_plans");
    if (!ctx) return NS_ERR_ARG;
    if (!t || !assign || P < 1 || (n_col > 0 && !col_plan) || n_col < 0)
        return set_err(ctx, NS_ERR_ARG, "ns_score_plans: null argument or P < 1");
    if (t->ctx != ctx) return set_err(ctx, NS_ERR_ARG, "tables belong to another ctx");
    if (!ctx->model.loaded) return set_err(ctx, NS_ERR_STATE, "no cost models loaded");
    if (D != ctx->model.D) return set_err(ctx, NS_ERR_ARG, "D differs from the loaded comm models' D");
    if (task < 0 || task >= t->n_tasks) return set_err(ctx, NS_ERR_ARG, "task out of range");
    const uint32_t readings = (uint32_t)mode & (NS_R10_ABS_STARTS | NS_R11_SUM_OF_MAX);
    mode &= ~(int32_t)(NS_R10_ABS_STARTS | NS_R11_SUM_OF_MAX);
    if (mode != NS_SCORE_FP64 && mode != NS_SCORE_TF32X3) return set_err(ctx, NS_ERR_ARG, "bad mode");
    ctx->rflags = readings;
    if (mode == NS_SCORE_TF32X3 && D > 16) return set_err(ctx, NS_ERR_ARG, "NS_SCORE_TF32X3 needs D <= 16");
    // validate the column plan against the evolving dims
    if (n_col > 0) {
        ns_status ds = ensure_host_dims(ctx, t);
        if (ds != NS_OK) return ds;
    }
    std::vector<int32_t> dims;
    if (n_col > 0) dims.assign(t->dims.begin() + t->off[task], t->dims.begin() + t->off[task + 1]);
    std::vector<int> depth(dims.size(), 0);   // variant row depth of each list entry (< kDepth)
    for (int i = 0; i < n_col; ++i) {
        int c = col_plan[i];
        if (c < 0 || c >= (int)dims.size() || dims[c] % 8 != 0 || depth[c] >= kDepth - 1)
            return set_err(ctx, NS_ERR_ARG, "col_plan step " + std::to_string(i) + " is not a legal split");
        dims[c] /= 2;
        dims.push_back(dims[c]);
        depth[c] += 1;
        depth.push_back(depth[c]);
    }
    cudaSetDevice(ctx->device);
    if (n_col > 0 && !t->deep_done) {
        launch_precompute(ctx, t, 1, kDepth - 1);
        NS_CHECK_LAST(ctx);
        const_cast<ns_tables*>(t)->deep_done = true;
    }
    return run_score_plans(ctx, t, task, D, col_plan, n_col, assign, P, mode, cost_out, best_index_out,
                           best_cost_out);
}

ns_status ns_set_workspace(ns_ctx* ctx, void* device_ptr, size_t bytes) {
    if (!ctx) return NS_ERR_ARG;
    if (device_ptr && (!is_device_ptr(device_ptr) || ((uintptr_t)device_ptr & 255) != 0))
        return set_err(ctx, NS_ERR_ARG, "ns_set_workspace: need 256-byte aligned device memory");
    cudaSetDevice(ctx->device);
    // work in flight (and async result copies) may still use the current arena
    NS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    if (ctx->out_stream) NS_CUDA(ctx, cudaStreamSynchronize(ctx->out_stream));
    ctx->out_pending = false;
    if (ctx->arena && !ctx->arena_external) cudaFree(ctx->arena);
    ctx->arena = device_ptr;
    ctx->arena_bytes = device_ptr ? bytes : 0;
    ctx->arena_external = device_ptr != nullptr;
    return NS_OK;
}

ns_status ns_search_workspace_bytes(ns_ctx* ctx, int32_t n_tasks, int32_t T_max, int32_t D,
                                    const ns_search_params* p, int32_t columnwise, size_t* bytes_out) {
    if (!ctx) return NS_ERR_ARG;
    if (!p || !bytes_out || n_tasks < 1 || T_max < 1 || D < 1 || D > kMaxD || p->M < 1 ||
        (columnwise && (p->N < 1 || p->K < 1 || p->L < 0 || p->L > 64)))
        return set_err(ctx, NS_ERR_ARG, "ns_search_workspace_bytes: bad shape or parameters");
    *bytes_out = search_workspace(ctx, n_tasks, T_max, D, p, columnwise != 0);
    return NS_OK;
}

ns_status ns_score_workspace_bytes(ns_ctx* ctx, int32_t T_prime, int32_t D, int64_t P, int32_t assign_on_device,
                                   size_t* bytes_out) {
    if (!ctx) return NS_ERR_ARG;
    if (!bytes_out || T_prime < 1 || D < 1 || D > kMaxD || P < 1)
        return set_err(ctx, NS_ERR_ARG, "ns_score_workspace_bytes: bad shape");
    *bytes_out = score_workspace(ctx, T_prime, D, P, assign_on_device != 0);
    return NS_OK;
}

}  // extern "C"
