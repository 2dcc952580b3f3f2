// collective.cu -- multi-GPU decode: (request, layer, kv_head)
// units shard across GPUs with no exchange inside the path; the one
// collective is the all-gather of the per-unit attention outputs, batched
// over the layers of a call, on NCCL (NVLink / NVSwitch inside a box).
//
// NCCL is loaded at run time (dlopen of libnccl.so.2 -- the process's
// already-loaded NCCL when torch or the host application brought one), so
// libpqkv.so itself has no link-time NCCL dependency and the single-GPU API
// works without it.  A communicator is created from an ncclUniqueId the host
// exchanges out of band (pqkv_comm_unique_id on rank 0, broadcast, then
// pqkv_comm_init on every rank) -- the ncclCommInitRank protocol.
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <nccl.h>

#include "internal.cuh"

using namespace pqkv_dev;

struct pqkv_comm {
    ncclComm_t nccl = nullptr;
    int n_ranks = 0, rank = 0, device = 0;
    cudaStream_t stream = nullptr;   // collective stream (ordered after the decode by an event)
    cudaEvent_t decoded = nullptr;   // decode done on the caller's stream
    cudaEvent_t gathered = nullptr;  // all-gather done on the collective stream
    void* send = nullptr;
    size_t send_bytes = 0;
};

namespace {

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    bool ok = false;
    std::string why;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);  // the process's NCCL first
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = std::string("pqkv: libnccl.so.2 not found (") + dlerror() + ")";
            return;
        }
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
        api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_gather && api.error_string;
        if (!api.ok) api.why = "pqkv: libnccl.so.2 lacks the collective entry points";
    });
    if (!api.ok) fail(PQKV_ERUNTIME, api.why);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(PQKV_ERUNTIME, std::string(what) + ": " + nccl().error_string(r));
}

}  // namespace

extern "C" {

int pqkv_comm_unique_id(uint8_t out[128]) {
    return guard([&] {
        if (!out) fail(PQKV_EINVAL, "pqkv_comm_unique_id: out is NULL");
        ncclUniqueId id;
        nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
        std::memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
    });
}

int pqkv_comm_init(pqkv_ctx* ctx, const uint8_t id[128], int n_ranks, int rank, pqkv_comm** out) {
    return guard([&] {
        if (!ctx || !id || !out) fail(PQKV_EINVAL, "pqkv_comm_init: NULL argument");
        if (n_ranks < 1 || rank < 0 || rank >= n_ranks) fail(PQKV_EINVAL, "pqkv_comm_init: bad rank / size");
        bind_device(ctx);
        ncclUniqueId uid;
        std::memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
        auto* c = new pqkv_comm();
        c->n_ranks = n_ranks;
        c->rank = rank;
        c->device = ctx->device;
        try {
            nccl_check(nccl().comm_init_rank(&c->nccl, n_ranks, uid, rank), "ncclCommInitRank");
            PQKV_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
            PQKV_CUDA(cudaEventCreateWithFlags(&c->decoded, cudaEventDisableTiming));
            PQKV_CUDA(cudaEventCreateWithFlags(&c->gathered, cudaEventDisableTiming));
        } catch (...) {
            if (c->nccl) nccl().comm_destroy(c->nccl);
            delete c;
            throw;
        }
        *out = c;
    });
}

int pqkv_comm_destroy(pqkv_comm* comm) {
    return guard([&] {
        if (!comm) return;
        cudaSetDevice(comm->device);
        if (comm->stream) cudaStreamSynchronize(comm->stream);
        if (comm->send) cudaFree(comm->send);
        if (comm->decoded) cudaEventDestroy(comm->decoded);
        if (comm->gathered) cudaEventDestroy(comm->gathered);
        if (comm->stream) cudaStreamDestroy(comm->stream);
        if (comm->nccl) nccl().comm_destroy(comm->nccl);
        delete comm;
    });
}

// Sharded decode of n_layers layers: this rank decodes its units of every
// layer (layers[l], units_per_rank units each -- ranks with fewer units pad:
// their extra rows are zero) into a send buffer [n_layers][units_per_rank]
// [g][d_h], and ONE all-gather (on the communicator's stream, ordered after
// the decodes by an event; the caller's stream waits for it) fills
// d_out_all [n_ranks][n_layers][units_per_rank][g][d_h].
int pqkv_decode_sharded(pqkv_ctx* ctx, pqkv_comm* comm, const pqkv_layer* layers, size_t n_layers,
                        size_t units_per_rank, const float* const* d_queries, size_t g, size_t k, float* d_out_all,
                        void* stream) {
    return guard([&] {
        if (!ctx || !comm || !layers || !d_queries || !d_out_all) fail(PQKV_EINVAL, "decode_sharded: NULL argument");
        if (comm->device != ctx->device) fail(PQKV_EINVAL, "decode_sharded: context and communicator devices differ");
        bind_device(ctx);
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        size_t d_h = 0;
        for (size_t l = 0; l < n_layers; ++l) {
            if (layers[l].n_heads > units_per_rank) fail(PQKV_EINVAL, "decode_sharded: layer has more units than units_per_rank");
            if (l && layers[l].d_h != d_h) fail(PQKV_EINVAL, "decode_sharded: layers differ in d_h");
            d_h = layers[l].d_h;
        }
        if (!n_layers) return;
        const size_t per_layer = units_per_rank * g * d_h, bytes = n_layers * per_layer * sizeof(float);
        if (bytes > comm->send_bytes) {
            if (comm->send) {
                PQKV_CUDA(cudaStreamSynchronize(comm->stream));
                PQKV_CUDA(cudaFree(comm->send));
                comm->send = nullptr;
            }
            PQKV_CUDA(cudaMalloc(&comm->send, bytes));
            comm->send_bytes = bytes;
        }
        float* send = static_cast<float*>(comm->send);
        // the previous call's all-gather may still read the send buffer
        PQKV_CUDA(cudaStreamWaitEvent(st, comm->gathered, 0));
        for (size_t l = 0; l < n_layers; ++l) {
            float* o = send + l * per_layer;
            const size_t used = layers[l].n_heads * g * d_h;
            if (used < per_layer) PQKV_CUDA(cudaMemsetAsync(o + used, 0, (per_layer - used) * sizeof(float), st));
            if (!layers[l].n_heads) continue;
            const int rc = pqkv_decode(ctx, &layers[l], d_queries[l], g, k, o, nullptr, stream);
            if (rc != PQKV_OK) fail(rc, pqkv_last_error());
        }
        PQKV_CUDA(cudaEventRecord(comm->decoded, st));
        PQKV_CUDA(cudaStreamWaitEvent(comm->stream, comm->decoded, 0));
        nccl_check(nccl().all_gather(send, d_out_all, n_layers * per_layer, ncclFloat32, comm->nccl, comm->stream),
                   "ncclAllGather");
        PQKV_CUDA(cudaEventRecord(comm->gathered, comm->stream));
        PQKV_CUDA(cudaStreamWaitEvent(st, comm->gathered, 0));
    });
}

}  // extern "C"
