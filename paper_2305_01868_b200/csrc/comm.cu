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
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllGather && a.AllReduce && a.GetErrorString;
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
    }
}

ns_status comm_allgather(ns_ctx* ctx, const void* send, void* recv, size_t bytes_per_rank) {
    if (ctx->nranks == 1 || ctx->emulated) {
        if (send != recv)
            NS_CUDA(ctx, cudaMemcpyAsync(recv, send, bytes_per_rank, cudaMemcpyDeviceToDevice, ctx->stream));
        return NS_OK;
    }
    ncclResult_t r = api().AllGather(send, recv, bytes_per_rank, ncclUint8, (ncclComm_t)ctx->nccl, ctx->stream);
    if (r != ncclSuccess) return nccl_err(ctx, r, "ncclAllGather");
    return NS_OK;
}

ns_status comm_allreduce_min_u64(ns_ctx* ctx, uint64_t* buf, size_t count) {
    if (ctx->nranks == 1 || ctx->emulated) return NS_OK;
    ncclResult_t r = api().AllReduce(buf, buf, count, ncclUint64, ncclMin, (ncclComm_t)ctx->nccl, ctx->stream);
    if (r != ncclSuccess) return nccl_err(ctx, r, "ncclAllReduce(min)");
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
    if (nranks == 1) return NS_OK;
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

}  // extern "C"
