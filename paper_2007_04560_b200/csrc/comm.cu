// In-library multi-GPU data plane: NCCL on the context's stream.
//
// The z-slab decomposition (slab.py) needs two things per
// stencil application and per Krylov step: ghost planes from the z-neighbour
// ranks, and sums / minima combined across ranks.  With an NCCL communicator
// bound to the context (acch_set_nccl) both are device-side:
//   * comm_halo  -- one grouped ncclSend / ncclRecv per neighbour of the
//                   `depth` boundary planes straight out of / into the
//                   caller's vector, enqueued on ctx->stream (no host sync;
//                   the kernels that read the ghosts follow on the stream);
//   * comm_allreduce_dev -- ncclAllReduce in place on device scratch (the
//                   device-resident GMRES multi-dots, lagged-pass
//                   projections and the lost-orthogonality norm);
//   * comm_allreduce -- host values: staged through device scratch, reduced,
//                   read back by the caller's own synchronisation point.
// Without NCCL the host hooks of acch_set_comm are used (ThreadComm /
// TorchDistComm in slab.py).  Left-RAS only needs the forward exchange (its
// apply scatters owned cells), the property the paper uses to halve RAS
// communication.
//
// libnccl is loaded at run time (dlopen of the path the caller gives -- the
// one torch.distributed already loaded -- or "libnccl.so.2"), so the library
// neither links a second NCCL into the process nor needs one to load.
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include <mutex>
#include <string>

#include "acch_internal.cuh"

namespace {

struct NcclApi {
    void *handle = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi g_api;
std::mutex g_api_mu;

acch_status load_nccl(const char *path)
{
    std::lock_guard<std::mutex> lk(g_api_mu);
    if (g_api.handle) return ACCH_OK;
    const char *p = (path && path[0]) ? path : "libnccl.so.2";
    void *h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        acch_set_error(std::string("cannot load NCCL (") + p + "): " + dlerror());
        return ACCH_ERR_INVALID_ARG;
    }
    NcclApi a;
    a.handle = h;
#define SYM(field, name)                                                          \
    a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name));                \
    if (!a.field) {                                                               \
        acch_set_error(std::string("NCCL library lacks ") + name);                \
        return ACCH_ERR_INVALID_ARG;                                              \
    }
    SYM(GetUniqueId, "ncclGetUniqueId")
    SYM(CommInitRank, "ncclCommInitRank")
    SYM(CommDestroy, "ncclCommDestroy")
    SYM(AllReduce, "ncclAllReduce")
    SYM(Send, "ncclSend")
    SYM(Recv, "ncclRecv")
    SYM(GroupStart, "ncclGroupStart")
    SYM(GroupEnd, "ncclGroupEnd")
    SYM(GetErrorString, "ncclGetErrorString")
#undef SYM
    g_api = a;
    return ACCH_OK;
}

acch_status nccl_fail(ncclResult_t r, const char *what)
{
    acch_set_error(std::string("NCCL error in ") + what + ": " +
                   (g_api.GetErrorString ? g_api.GetErrorString(r) : "?"));
    return ACCH_ERR_CUDA;
}

#define NCCL_TRY(call, what)                              \
    do {                                                  \
        ncclResult_t _r = (call);                         \
        if (_r != ncclSuccess) return nccl_fail(_r, what); \
    } while (0)

ncclRedOp_t red_op(int op) { return op == 0 ? ncclSum : (op == 1 ? ncclMin : ncclMax); }

int lower_rank(const acch_ctx *ctx)
{
    if (ctx->rank > 0) return ctx->rank - 1;
    return ctx->g.periodic ? ctx->nranks - 1 : -1;
}
int upper_rank(const acch_ctx *ctx)
{
    if (ctx->rank < ctx->nranks - 1) return ctx->rank + 1;
    return ctx->g.periodic ? 0 : -1;
}

}  // namespace

bool comm_has_nccl(const acch_ctx *ctx) { return ctx->nccl_comm != nullptr; }

acch_status nccl_halo(acch_ctx *ctx, double *vec, long long plane, int depth)
{
    const GridDev &g = ctx->g;
    const int lo = lower_rank(ctx), hi = upper_rank(ctx);
    const size_t count = (size_t)depth * plane;
    double *bot_g = vec + (long long)(g.zg - depth) * plane, *top_g = vec + (long long)(g.zg + g.nz) * plane;
    const double *bot_i = vec + (long long)g.zg * plane, *top_i = vec + (long long)(g.zg + g.nz - depth) * plane;
    ncclComm_t comm = reinterpret_cast<ncclComm_t>(ctx->nccl_comm);
    // per peer pair: the sends go "up" first, the receives come "from below"
    // first, so two ranks that are each other's upper and lower neighbour
    // (2 periodic ranks, or 1 rank exchanging with itself) still pair the
    // messages correctly (NCCL matches sends / receives per peer in order)
    NCCL_TRY(g_api.GroupStart(), "ncclGroupStart");
    if (hi >= 0) NCCL_TRY(g_api.Send(top_i, count, ncclFloat64, hi, comm, ctx->stream), "ncclSend");
    if (lo >= 0) NCCL_TRY(g_api.Send(bot_i, count, ncclFloat64, lo, comm, ctx->stream), "ncclSend");
    if (lo >= 0) NCCL_TRY(g_api.Recv(bot_g, count, ncclFloat64, lo, comm, ctx->stream), "ncclRecv");
    if (hi >= 0) NCCL_TRY(g_api.Recv(top_g, count, ncclFloat64, hi, comm, ctx->stream), "ncclRecv");
    NCCL_TRY(g_api.GroupEnd(), "ncclGroupEnd");
    ctx->comm_bytes += (double)count * sizeof(double) * ((lo >= 0) + (hi >= 0));
    ctx->comm_calls += 1;
    return ACCH_OK;
}

acch_status comm_allreduce_dev(acch_ctx *ctx, double *dev, int n, int op)
{
    if (ctx->nranks <= 1 && !ctx->nccl_comm) return ACCH_OK;
    if (!ctx->nccl_comm) {
        acch_set_error("device allreduce needs an NCCL communicator (acch_set_nccl)");
        return ACCH_ERR_INVALID_ARG;
    }
    NCCL_TRY(g_api.AllReduce(dev, dev, (size_t)n, ncclFloat64, red_op(op),
                             reinterpret_cast<ncclComm_t>(ctx->nccl_comm), ctx->stream),
             "ncclAllReduce");
    ctx->comm_calls += 1;
    return ACCH_OK;
}

acch_status nccl_allreduce_host(acch_ctx *ctx, double *vals, int n, int op)
{
    if (n > 64) {
        acch_set_error("allreduce: at most 64 values");
        return ACCH_ERR_INVALID_ARG;
    }
    double *d = ctx->d_comm;
    ACCH_CUDA(cudaMemcpyAsync(d, vals, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    acch_status st = comm_allreduce_dev(ctx, d, n, op);
    if (st != ACCH_OK) return st;
    ACCH_CUDA(cudaMemcpyAsync(vals, d, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
    ACCH_CUDA(cudaStreamSynchronize(ctx->stream));
    return ACCH_OK;
}

void comm_release(acch_ctx *ctx)
{
    if (ctx->nccl_comm && g_api.CommDestroy) g_api.CommDestroy(reinterpret_cast<ncclComm_t>(ctx->nccl_comm));
    ctx->nccl_comm = nullptr;
    if (ctx->d_comm) cudaFree(ctx->d_comm);
    ctx->d_comm = nullptr;
}

extern "C" {

acch_status acch_nccl_unique_id(const char *nccl_path, void *id_out)
{
    if (!id_out) {
        acch_set_error("acch_nccl_unique_id: null output");
        return ACCH_ERR_INVALID_ARG;
    }
    acch_status st = load_nccl(nccl_path);
    if (st != ACCH_OK) return st;
    ncclUniqueId id;
    NCCL_TRY(g_api.GetUniqueId(&id), "ncclGetUniqueId");
    memcpy(id_out, &id, sizeof(id));
    return ACCH_OK;
}

int32_t acch_nccl_id_bytes(void) { return (int32_t)sizeof(ncclUniqueId); }

acch_status acch_set_nccl(acch_ctx *ctx, const char *nccl_path, const void *id, int32_t nranks, int32_t rank)
{
    if (!ctx || !id) {
        acch_set_error("acch_set_nccl: null argument");
        return ACCH_ERR_INVALID_ARG;
    }
    if (nranks != ctx->nranks || rank != ctx->rank) {
        acch_set_error("acch_set_nccl: rank / size differ from the slab (acch_ctx_set_slab first)");
        return ACCH_ERR_INVALID_ARG;
    }
    ACCH_CUDA(cudaSetDevice(ctx->device));
    acch_status st = load_nccl(nccl_path);
    if (st != ACCH_OK) return st;
    comm_release(ctx);
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    ncclComm_t comm = nullptr;
    NCCL_TRY(g_api.CommInitRank(&comm, nranks, uid, rank), "ncclCommInitRank");
    ctx->nccl_comm = comm;
    ACCH_CUDA(cudaMalloc(&ctx->d_comm, sizeof(double) * 64));
    return ACCH_OK;
}

acch_status acch_comm_stats(acch_ctx *ctx, double *bytes, int64_t *calls)
{
    if (!ctx) {
        acch_set_error("null context");
        return ACCH_ERR_INVALID_ARG;
    }
    if (bytes) *bytes = ctx->comm_bytes;
    if (calls) *calls = ctx->comm_calls;
    return ACCH_OK;
}

}  // extern "C"
