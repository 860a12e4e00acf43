// comm.cu -- NCCL layer (N7): communicator bootstrap and the two collectives
// the search needs (allgather of per-trajectory results, allreduce-min of
// packed (cost, index) keys).  NCCL is resolved at run time with dlopen so
// the library shares the single libnccl.so.2 that torch already loaded
// (NCCL 2.28 from the nvidia-nccl pip package) instead of linking a second
// copy.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <string>
#include <vector>

#include "ns_internal.cuh"

namespace {

struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& api() {
    static NcclApi a;
    static bool tried = false;
    if (tried) return a;
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        const char* site = getenv("NS_NCCL_LIB");
        if (site) h = dlopen(site, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) {
        a.why = std::string("dlopen libnccl.so.2 failed: ") + (dlerror() ? dlerror() : "?");
        return a;
    }
    a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))dlsym(h, "ncclCommInitRank");
    a.CommDestroy = (decltype(a.CommDestroy))dlsym(h, "ncclCommDestroy");
    a.AllGather = (decltype(a.AllGather))dlsym(h, "ncclAllGather");
    a.AllReduce = (decltype(a.AllReduce))dlsym(h, "ncclAllReduce");
    a.GetErrorString = (decltype(a.GetErrorString))dlsym(h, "ncclGetErrorString");
    a.GroupStart = (decltype(a.GroupStart))dlsym(h, "ncclGroupStart");
    a.GroupEnd = (decltype(a.GroupEnd))dlsym(h, "ncclGroupEnd");
    a.Send = (decltype(a.Send))dlsym(h, "ncclSend");
    a.Recv = (decltype(a.Recv))dlsym(h, "ncclRecv");
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllGather && a.AllReduce && a.GetErrorString &&
           a.GroupStart && a.GroupEnd && a.Send && a.Recv;
    if (!a.ok) a.why = "libnccl.so.2 lacks required symbols";
    return a;
}

ns_status nccl_err(ns_ctx* ctx, ncclResult_t r, const char* what) {
    return ns::set_err(ctx, NS_ERR_NCCL, std::string("NCCL error in ") + what + ": " + api().GetErrorString(r));
}

}  // namespace

namespace ns {
void comm_destroy(ns_ctx* ctx) {
    if (ctx && ctx->nccl && api().ok) api().CommDestroy((ncclComm_t)ctx->nccl);
    if (ctx) {
        ctx->nccl = nullptr;
        ctx->nranks = 1;
        ctx->rank = 0;
        ctx->emulated = false;
        ctx->host_comm_on = false;
        ctx->host_comm = ns_host_comm{};
    }
}

bool comm_collective(const ns_ctx* ctx) {
    return ctx->nranks > 1 || ctx->nccl != nullptr || ctx->host_comm_on || ctx->emulated;
}

namespace {
// host-callback backend: stage through pinned memory on the ctx stream
char* host_stage(ns_ctx* ctx, size_t bytes) {
    if (ctx->comm_stage_bytes < bytes) {
        if (ctx->comm_stage) cudaFreeHost(ctx->comm_stage);
        ctx->comm_stage = nullptr;
        ctx->comm_stage_bytes = 0;
        if (cudaMallocHost(&ctx->comm_stage, bytes) != cudaSuccess) return nullptr;
        ctx->comm_stage_bytes = bytes;
    }
    return (char*)ctx->comm_stage;
}
}  // namespace

ns_status comm_allgather(ns_ctx* ctx, const void* send, void* recv, size_t bytes_per_rank) {
    if (ctx->emulated || (!ctx->nccl && !ctx->host_comm_on)) {
        if (send != recv)
            NS_CUDA(ctx, cudaMemcpyAsync(recv, send, bytes_per_rank, cudaMemcpyDeviceToDevice, ctx->stream));
        return NS_OK;
    }
    if (ctx->nccl) {
        ncclResult_t r = api().AllGather(send, recv, bytes_per_rank, ncclUint8, (ncclComm_t)ctx->nccl, ctx->stream);
        if (r != ncclSuccess) return nccl_err(ctx, r, "ncclAllGather");
        return NS_OK;
    }
    const size_t total = bytes_per_rank * (size_t)ctx->nranks;
    char* h = host_stage(ctx, total);
    if (!h) return set_err(ctx, NS_ERR_NOMEM, "pinned comm staging");
    char* mine = h + (size_t)ctx->rank * bytes_per_rank;
    NS_CUDA(ctx, cudaMemcpyAsync(mine, send, bytes_per_rank, cudaMemcpyDeviceToHost, ctx->stream));
    NS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    if (ctx->host_comm.allgather(ctx->host_comm.user, mine, h, bytes_per_rank) != 0)
        return set_err(ctx, NS_ERR_NCCL, "host allgather callback failed");
    NS_CUDA(ctx, cudaMemcpyAsync(recv, h, total, cudaMemcpyHostToDevice, ctx->stream));
    NS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));   // the staging is reused by the next collective
    return NS_OK;
}

namespace {
ns_status allreduce(ns_ctx* ctx, void* buf, size_t count, int op) {
    if (ctx->emulated || (!ctx->nccl && !ctx->host_comm_on)) return NS_OK;
    if (ctx->nccl) {
        ncclResult_t r = op == NS_COMM_MIN_U64
                             ? api().AllReduce(buf, buf, count, ncclUint64, ncclMin, (ncclComm_t)ctx->nccl, ctx->stream)
                             : api().AllReduce(buf, buf, count, ncclInt8, ncclMax, (ncclComm_t)ctx->nccl, ctx->stream);
        if (r != ncclSuccess) return nccl_err(ctx, r, op == NS_COMM_MIN_U64 ? "ncclAllReduce(min)" : "ncclAllReduce(max)");
        return NS_OK;
    }
    const size_t bytes = count * (op == NS_COMM_MIN_U64 ? 8 : 1);
    char* h = host_stage(ctx, bytes);
    if (!h) return set_err(ctx, NS_ERR_NOMEM, "pinned comm staging");
    NS_CUDA(ctx, cudaMemcpyAsync(h, buf, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    NS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    if (ctx->host_comm.allreduce(ctx->host_comm.user, h, count, op) != 0)
        return set_err(ctx, NS_ERR_NCCL, "host allreduce callback failed");
    NS_CUDA(ctx, cudaMemcpyAsync(buf, h, bytes, cudaMemcpyHostToDevice, ctx->stream));
    NS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return NS_OK;
}
}  // namespace

ns_status comm_allreduce_min_u64(ns_ctx* ctx, uint64_t* buf, size_t count) {
    return allreduce(ctx, buf, count, NS_COMM_MIN_U64);
}

ns_status comm_allreduce_max_i8(ns_ctx* ctx, int8_t* buf, size_t count) {
    return allreduce(ctx, buf, count, NS_COMM_MAX_I8);
}

// All-to-all with per-peer sizes: send block q (send_bytes[q] bytes, blocks
// contiguous in peer order) goes to rank q; the block from rank r lands at
// recv + sum_{r' < r} recv_bytes[r'].  NCCL: one group of ncclSend/ncclRecv
// pairs (the self pair included), so every transfer is in flight at once.
ns_status comm_alltoallv(ns_ctx* ctx, const void* send, const size_t* send_bytes, void* recv,
                         const size_t* recv_bytes) {
    const int R = ctx->nranks;
    if (ctx->emulated) return set_err(ctx, NS_ERR_STATE, "all-to-all needs real ranks (not emulated)");
    std::vector<size_t> so(R + 1, 0), ro(R + 1, 0);
    for (int q = 0; q < R; ++q) {
        so[q + 1] = so[q] + send_bytes[q];
        ro[q + 1] = ro[q] + recv_bytes[q];
    }
    if (!ctx->nccl && !ctx->host_comm_on) {   // one rank: the block to self
        if (send_bytes[0] != recv_bytes[0]) return set_err(ctx, NS_ERR_ARG, "all-to-all: self block sizes differ");
        if (send_bytes[0])
            NS_CUDA(ctx, cudaMemcpyAsync(recv, send, send_bytes[0], cudaMemcpyDeviceToDevice, ctx->stream));
        return NS_OK;
    }
    if (ctx->nccl) {
        ncclResult_t r = api().GroupStart();
        for (int q = 0; q < R && r == ncclSuccess; ++q) {
            if (send_bytes[q]) r = api().Send((const char*)send + so[q], send_bytes[q], ncclUint8, q, (ncclComm_t)ctx->nccl, ctx->stream);
            if (r == ncclSuccess && recv_bytes[q])
                r = api().Recv((char*)recv + ro[q], recv_bytes[q], ncclUint8, q, (ncclComm_t)ctx->nccl, ctx->stream);
        }
        const ncclResult_t e = api().GroupEnd();
        if (r != ncclSuccess) return nccl_err(ctx, r, "ncclSend/ncclRecv");
        if (e != ncclSuccess) return nccl_err(ctx, e, "ncclGroupEnd");
        return NS_OK;
    }
    if (!ctx->host_comm.alltoallv) return set_err(ctx, NS_ERR_STATE, "host transport without an alltoallv callback");
    char* h = host_stage(ctx, so[R] + ro[R]);
    if (!h) return set_err(ctx, NS_ERR_NOMEM, "pinned comm staging");
    if (so[R]) NS_CUDA(ctx, cudaMemcpyAsync(h, send, so[R], cudaMemcpyDeviceToHost, ctx->stream));
    NS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    if (ctx->host_comm.alltoallv(ctx->host_comm.user, h, send_bytes, h + so[R], recv_bytes) != 0)
        return set_err(ctx, NS_ERR_NCCL, "host alltoallv callback failed");
    if (ro[R]) NS_CUDA(ctx, cudaMemcpyAsync(recv, h + so[R], ro[R], cudaMemcpyHostToDevice, ctx->stream));
    NS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return NS_OK;
}

}  // namespace ns

extern "C" {

ns_status ns_comm_unique_id(unsigned char id_out[128]) {
    if (!id_out) return NS_ERR_ARG;
    if (!api().ok) return NS_ERR_NCCL;
    ncclUniqueId id;
    if (api().GetUniqueId(&id) != ncclSuccess) return NS_ERR_NCCL;
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id_out, &id, 128);
    return NS_OK;
}

ns_status ns_comm_init(ns_ctx* ctx, int32_t nranks, int32_t rank, const unsigned char id[128]) {
    if (!ctx) return NS_ERR_ARG;
    if (nranks < 1 || rank < 0 || rank >= nranks) return ns::set_err(ctx, NS_ERR_ARG, "ns_comm_init: bad nranks/rank");
    ns::comm_destroy(ctx);
    if (nranks == 1 && !id) return NS_OK;
    if (!id) {   // emulated ranks: partitioning exercised in one process, no NCCL
        ctx->nranks = nranks;
        ctx->rank = 0;
        ctx->emulated = true;
        return NS_OK;
    }
    if (!api().ok) return ns::set_err(ctx, NS_ERR_NCCL, api().why);
    cudaSetDevice(ctx->device);
    ncclUniqueId uid;
    std::memcpy(&uid, id, 128);
    ncclComm_t comm;
    ncclResult_t r = api().CommInitRank(&comm, nranks, uid, rank);
    if (r != ncclSuccess) return nccl_err(ctx, r, "ncclCommInitRank");
    ctx->nccl = comm;
    ctx->nranks = nranks;
    ctx->rank = rank;
    return NS_OK;
}

ns_status ns_comm_init_host(ns_ctx* ctx, int32_t nranks, int32_t rank, const ns_host_comm* comm) {
    if (!ctx) return NS_ERR_ARG;
    if (nranks < 1 || rank < 0 || rank >= nranks || !comm || !comm->allgather || !comm->allreduce)
        return ns::set_err(ctx, NS_ERR_ARG, "ns_comm_init_host: bad nranks/rank or missing callbacks");
    ns::comm_destroy(ctx);
    ctx->host_comm = *comm;
    ctx->host_comm_on = true;
    ctx->nranks = nranks;
    ctx->rank = rank;
    return NS_OK;
}

}  // extern "C"
