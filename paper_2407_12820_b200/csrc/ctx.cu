// ctx.cu -- context, scratch arena, status plumbing and the geometry entry
// points of the C ABI (include/pqkv_c.h).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <new>
#include <vector>
#include <string>

#include "internal.cuh"

namespace {
thread_local std::string g_last_error;
}  // namespace

namespace pqkv_dev {

void set_last_error(const std::string& msg) { g_last_error = msg; }

void bind_device(pqkv_ctx* ctx) {
    int cur = -1;
    PQKV_CUDA(cudaGetDevice(&cur));
    if (cur != ctx->device) PQKV_CUDA(cudaSetDevice(ctx->device));
}

void Scratch::commit() {
    if (total_ > ctx_->arena_bytes) {
        size_t want = round_up(total_ + total_ / 4, size_t(1) << 20);
        if (ctx_->arena) {
            PQKV_CUDA(cudaDeviceSynchronize());
            PQKV_CUDA(cudaFree(ctx_->arena));
            ctx_->arena = nullptr;
            ctx_->arena_bytes = 0;
        }
        PQKV_CUDA(cudaMalloc(&ctx_->arena, want));
        ctx_->arena_bytes = want;
    }
}

void* pinned_staging(pqkv_ctx* ctx, size_t bytes) {
    if (bytes > ctx->pinned_bytes) {
        if (ctx->pinned) {
            PQKV_CUDA(cudaDeviceSynchronize());
            PQKV_CUDA(cudaFreeHost(ctx->pinned));
        }
        ctx->pinned = nullptr;
        PQKV_CUDA(cudaMallocHost(&ctx->pinned, bytes));
        ctx->pinned_bytes = bytes;
    }
    return ctx->pinned;
}

void* decode_workspace(pqkv_ctx* ctx, size_t bytes) {
    if (bytes > ctx->ws_bytes) {
        if (ctx->ws) {
            PQKV_CUDA(cudaDeviceSynchronize());
            PQKV_CUDA(cudaFree(ctx->ws));
            ctx->ws = nullptr;
        }
        size_t want = round_up(bytes + bytes / 4, size_t(1) << 16);
        PQKV_CUDA(cudaMalloc(&ctx->ws, want));
        ctx->ws_bytes = want;
    }
    return ctx->ws;
}

void* host_io_staging(pqkv_ctx* ctx, size_t bytes) {
    if (bytes > ctx->io_bytes) {
        if (ctx->io) {
            PQKV_CUDA(cudaDeviceSynchronize());
            PQKV_CUDA(cudaFree(ctx->io));
            ctx->io = nullptr;
            ctx->io_bytes = 0;
        }
        size_t want = round_up(bytes, size_t(1) << 12);
        PQKV_CUDA(cudaMalloc(&ctx->io, want));
        ctx->io_bytes = want;
    }
    return ctx->io;
}

int current_sm_count() {
    static std::atomic<int> cache[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    std::atomic<int>& slot = cache[dev & 63];
    int v = slot.load(std::memory_order_relaxed);
    if (v <= 0) {
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        slot.store(v, std::memory_order_relaxed);
    }
    return v;
}

unsigned* arrival_counters(pqkv_ctx* ctx, size_t n, cudaStream_t st) {
    if (n > ctx->n_arrivals) {
        if (ctx->d_arrivals) {
            PQKV_CUDA(cudaDeviceSynchronize());
            PQKV_CUDA(cudaFree(ctx->d_arrivals));
        }
        size_t want = std::max<size_t>(n, 1024);
        PQKV_CUDA(cudaMalloc(&ctx->d_arrivals, want * sizeof(unsigned)));
        PQKV_CUDA(cudaMemsetAsync(ctx->d_arrivals, 0, want * sizeof(unsigned), st));
        ctx->n_arrivals = want;
    }
    return ctx->d_arrivals;
}

unsigned* ready_counters(pqkv_ctx* ctx, size_t n, cudaStream_t st) {
    if (n > ctx->n_ready) {
        if (ctx->d_ready) {
            PQKV_CUDA(cudaDeviceSynchronize());
            PQKV_CUDA(cudaFree(ctx->d_ready));
        }
        size_t want = std::max<size_t>(n, 256);
        PQKV_CUDA(cudaMalloc(&ctx->d_ready, want * sizeof(unsigned)));
        PQKV_CUDA(cudaMemsetAsync(ctx->d_ready, 0, want * sizeof(unsigned), st));
        ctx->n_ready = want;
    }
    return ctx->d_ready;
}

namespace {

__global__ void scatter_rows_kernel(const float* src_k, const float* src_v, const int64_t* rows, long long n, int d_h,
                                    float* dst_k, float* dst_v) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n * d_h;
         e += (long long)gridDim.x * blockDim.x) {
        const long long i = e / d_h, j = e % d_h, r = rows[i];
        dst_k[r * d_h + j] = src_k[e];
        dst_v[r * d_h + j] = src_v[e];
    }
}

}  // namespace

}  // namespace pqkv_dev

using namespace pqkv_dev;

extern "C" {

int pqkv_abi_version(void) { return PQKV_ABI_VERSION; }

const char* pqkv_last_error(void) { return g_last_error.c_str(); }

int pqkv_ctx_create(int device, pqkv_ctx** out) {
    return guard([&] {
        if (!out) fail(PQKV_EINVAL, "pqkv_ctx_create: out is NULL");
        int n = 0;
        PQKV_CUDA(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n) fail(PQKV_EINVAL, "pqkv_ctx_create: bad device");
        auto* c = new pqkv_ctx();
        c->device = device;
        bind_device(c);
        PQKV_CUDA(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
        PQKV_CUDA(cudaMalloc(&c->d_stats, 4 * sizeof(unsigned long long)));
        *out = c;
    });
}

int pqkv_ctx_destroy(pqkv_ctx* ctx) {
    return guard([&] {
        if (!ctx) return;
        bind_device(ctx);
        cudaDeviceSynchronize();
        if (ctx->arena) cudaFree(ctx->arena);
        if (ctx->pinned) cudaFreeHost(ctx->pinned);
        if (ctx->d_stats) cudaFree(ctx->d_stats);
        if (ctx->d_arrivals) cudaFree(ctx->d_arrivals);
        if (ctx->d_ready) cudaFree(ctx->d_ready);
        if (ctx->ws) cudaFree(ctx->ws);
        if (ctx->io) cudaFree(ctx->io);
        if (ctx->d_prof) cudaFree(ctx->d_prof);
        for (auto& hg : ctx->host_graphs)
            if (hg.exec) cudaGraphExecDestroy(hg.exec);
        if (ctx->capture_stream) cudaStreamDestroy(ctx->capture_stream);
        delete ctx;
    });
}

int pqkv_ctx_set_assign_mode(pqkv_ctx* ctx, int mode) {
    return guard([&] {
        if (!ctx) fail(PQKV_EINVAL, "ctx is NULL");
        if (mode != PQKV_ASSIGN_FILTERED && mode != PQKV_ASSIGN_EXACT)
            fail(PQKV_EINVAL, "unknown assign mode");
        ctx->assign_mode = mode;
    });
}

int pqkv_ctx_last_build_stats(pqkv_ctx* ctx, uint64_t* rechecked, uint64_t* total) {
    return guard([&] {
        if (!ctx) fail(PQKV_EINVAL, "ctx is NULL");
        if (rechecked) *rechecked = ctx->last_rechecked;
        if (total) *total = ctx->last_total;
    });
}

int pqkv_device_alloc(pqkv_ctx* ctx, size_t bytes, void** out) {
    return guard([&] {
        if (!ctx || !out) fail(PQKV_EINVAL, "pqkv_device_alloc: NULL argument");
        bind_device(ctx);
        *out = nullptr;
        if (bytes) PQKV_CUDA(cudaMalloc(out, bytes));
    });
}

int pqkv_device_free(pqkv_ctx* ctx, void* ptr) {
    return guard([&] {
        if (!ctx) fail(PQKV_EINVAL, "pqkv_device_free: NULL context");
        bind_device(ctx);
        if (ptr) PQKV_CUDA(cudaFree(ptr));
    });
}

int pqkv_copy(pqkv_ctx* ctx, void* dst, const void* src, size_t bytes, int kind) {
    return guard([&] {
        if (!ctx) fail(PQKV_EINVAL, "pqkv_copy: NULL context");
        bind_device(ctx);
        if (!bytes) return;
        cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice
                           : kind == 1 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
        PQKV_CUDA(cudaMemcpy(dst, src, bytes, k));
    });
}

int pqkv_stream_sync(pqkv_ctx* ctx, void* stream) {
    return guard([&] {
        if (!ctx) fail(PQKV_EINVAL, "pqkv_stream_sync: NULL context");
        bind_device(ctx);
        PQKV_CUDA(cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream)));
    });
}

int pqkv_scatter_rows(pqkv_ctx* ctx, const float* d_src_k, const float* d_src_v, const int64_t* d_rows, size_t n,
                      size_t d_h, float* d_dst_k, float* d_dst_v, void* stream) {
    return guard([&] {
        if (!ctx) fail(PQKV_EINVAL, "pqkv_scatter_rows: NULL context");
        bind_device(ctx);
        if (!n || !d_h) return;
        if (!d_src_k || !d_src_v || !d_rows || !d_dst_k || !d_dst_v) fail(PQKV_EINVAL, "pqkv_scatter_rows: NULL buffer");
        const size_t total = n * d_h;
        const unsigned blocks = (unsigned)std::min<size_t>(ceil_div(total, 256), 4 * (size_t)ctx->sm_count);
        scatter_rows_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
            d_src_k, d_src_v, d_rows, (long long)n, (int)d_h, d_dst_k, d_dst_v);
        PQKV_LAUNCHED("scatter_rows_kernel");
    });
}

int pqkv_ctx_set_selection_dump(pqkv_ctx* ctx, uint32_t* d_bitmap) {
    return guard([&] {
        if (!ctx) fail(PQKV_EINVAL, "NULL context");
        ctx->sel_dump = d_bitmap;
    });
}

int pqkv_ctx_set_profiling(pqkv_ctx* ctx, int on) {
    return guard([&] {
        if (!ctx) fail(PQKV_EINVAL, "NULL context");
        ctx->profiling = on ? 1 : 0;
    });
}

// Mean SM cycles per CTA of the last attention launch (profiling mode):
// [0] row-list prologue incl. pair select, [1] of which pair select + DSMEM,
// [2] gather + softmax, [3] CTAs measured.
int pqkv_ctx_last_decode_profile(pqkv_ctx* ctx, double out[4]) {
    return guard([&] {
        if (!ctx || !out) fail(PQKV_EINVAL, "NULL argument");
        for (int i = 0; i < 4; ++i) out[i] = 0.0;
        if (!ctx->d_prof || !ctx->n_prof) return;
        bind_device(ctx);
        std::vector<unsigned long long> h(ctx->n_prof * PQKV_PROF_SLOTS);
        PQKV_CUDA(cudaDeviceSynchronize());
        PQKV_CUDA(cudaMemcpy(h.data(), ctx->d_prof, h.size() * 8, cudaMemcpyDeviceToHost));
        double n = 0;
        for (size_t c = 0; c < ctx->n_prof; ++c) {
            const unsigned long long* t = &h[c * PQKV_PROF_SLOTS];
            if (!t[0] || !t[2] || !t[3]) continue;
            out[0] += (double)(t[2] - t[0]);
            out[1] += t[1] ? (double)(t[1] - t[0]) : 0.0;
            out[2] += (double)(t[3] - t[2]);
            n += 1;
        }
        if (n > 0) for (int i = 0; i < 3; ++i) out[i] /= n;
        out[3] = n;
    });
}

// Raw per-CTA timestamps of the last attention launch (profiling mode):
// 16 u64 per CTA (clock64 at start / after pair select / after the row list /
// after the gather; globaltimer ns at start / after the row list / after the
// gather / at exit; clock64 at the pair_select phase marks 0..6 (rank 0) and
// after the first cluster barrier).  *n_ctas = CTAs; copies min(cap, 16 n).
int pqkv_ctx_decode_profile_raw(pqkv_ctx* ctx, uint64_t* out, size_t cap, size_t* n_ctas) {
    return guard([&] {
        if (!ctx || !n_ctas) fail(PQKV_EINVAL, "NULL argument");
        *n_ctas = ctx->d_prof ? ctx->n_prof : 0;
        if (!ctx->d_prof || !out) return;
        bind_device(ctx);
        PQKV_CUDA(cudaDeviceSynchronize());
        PQKV_CUDA(cudaMemcpy(out, ctx->d_prof, std::min(cap, ctx->n_prof * PQKV_PROF_SLOTS) * 8, cudaMemcpyDeviceToHost));
    });
}

int pqkv_ctx_last_build_profile(pqkv_ctx* ctx, uint64_t cycles[8]) {
    return guard([&] {
        if (!ctx || !cycles) fail(PQKV_EINVAL, "NULL argument");
        for (int i = 0; i < 8; ++i) cycles[i] = ctx->last_phase_cycles[i];
    });
}

// PqConfig::create (pq.cpp:13-25): same rejection rules and messages.
int pqkv_pq_config(size_t m, size_t b, size_t d_h, size_t* d_m, size_t* n_clusters) {
    return guard([&] {
        if (m < 1) fail(PQKV_EINVAL, "pq: m must be >= 1");
        if (b < 1 || b > 16) fail(PQKV_EINVAL, "pq: b must be in [1, 16]");
        if (d_h < 1 || d_h % m != 0)
            fail(PQKV_EINVAL, "pq: head_dim must be a positive multiple of m");
        if (d_m) *d_m = d_h / m;
        if (n_clusters) *n_clusters = size_t{1} << b;
    });
}

// codes_memory_ratio (pq.cpp:179-182): bytes of codes per token over an fp16 key.
int pqkv_codes_memory_ratio(size_t m, size_t b, size_t d_h, double* ratio) {
    return guard([&] {
        if (d_h < 1) fail(PQKV_EINVAL, "pq: head_dim must be >= 1");
        if (!ratio) fail(PQKV_EINVAL, "ratio is NULL");
        *ratio = static_cast<double>(m * b) / (16.0 * static_cast<double>(d_h));
    });
}

}  // extern "C"
