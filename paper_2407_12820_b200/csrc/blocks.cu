// blocks.cu -- block-cache accounting of a fetch.
//
// KvStore::fetch_topk (kv_store.cpp:115-191) counts one lookup per distinct
// block of the requested tokens and then refreshes its fast-tier cache with
// the top-k_cache blocks of the request ranked by requested-token count, ties
// toward the lower block id (kv_store.cpp:158-166).  The per-request part --
// distinct tokens, per-block counts and that ranking -- runs here, one CTA
// per (layer, kv_head) unit, on the device-resident selection; the small
// sequential LRU/LFU state machine stays on the host (api.cpp).
#include <algorithm>

#include "internal.cuh"

namespace pqkv_dev {
namespace {

constexpr int BR_THREADS = 1024;

__global__ void __launch_bounds__(BR_THREADS) block_rank_kernel(const int64_t* ids, long long ids_stride, int n_ids,
                                                                int n_tokens, int block_size, int n_blocks,
                                                                int n_pow2, int k_cache, uint32_t* bitmap_out,
                                                                uint32_t* counts, int64_t* ranked,
                                                                uint32_t* touched) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int p = blockIdx.x, tid = threadIdx.x;
    const int words = (n_tokens + 31) / 32;
    unsigned long long* key = reinterpret_cast<unsigned long long*>(smem);  // [n_pow2]
    uint32_t* bits = reinterpret_cast<uint32_t*>(key + n_pow2);            // [words]
    __shared__ uint32_t n_touch;
    for (int w = tid; w < words; w += BR_THREADS) bits[w] = 0u;
    if (tid == 0) n_touch = 0;
    __syncthreads();
    // distinct requested tokens (a repeated id counts once, kv_store.cpp:127-128)
    const int64_t* ip = ids + p * ids_stride;
    for (int i = tid; i < n_ids; i += BR_THREADS) {
        const int64_t id = ip[i];
        if (id >= 0 && id < n_tokens) atomicOr(&bits[id >> 5], 1u << (id & 31));
    }
    __syncthreads();
    if (bitmap_out)
        for (int w = tid; w < words; w += BR_THREADS) bitmap_out[(long long)p * words + w] = bits[w];
    // distinct tokens per block; sort key (count desc, block asc)
    for (int b = tid; b < n_pow2; b += BR_THREADS) {
        uint32_t cnt = 0;
        if (b < n_blocks) {
            const int lo = b * block_size, hi = min(n_tokens, lo + block_size);
            for (int t = lo; t < hi;) {
                const int w = t >> 5, off = t & 31;
                const int take = min(32 - off, hi - t);
                const uint32_t m = (take == 32 ? 0xffffffffu : ((1u << take) - 1u)) << off;
                cnt += __popc(bits[w] & m);
                t += take;
            }
            counts[(long long)p * n_blocks + b] = cnt;
            if (cnt) atomicAdd(&n_touch, 1u);
        }
        key[b] = cnt ? ((unsigned long long)cnt << 32) | (0xffffffffu - (uint32_t)b) : 0ull;
    }
    __syncthreads();
    // bitonic sort, descending
    for (int size = 2; size <= n_pow2; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = tid; i < n_pow2 / 2; i += BR_THREADS) {
                const int lo = 2 * i - (i & (stride - 1));
                const int hi = lo + stride;
                const bool desc = (lo & size) == 0;
                const unsigned long long a = key[lo], c = key[hi];
                if ((a < c) == desc) { key[lo] = c; key[hi] = a; }
            }
            __syncthreads();
        }
    for (int r = tid; r < k_cache; r += BR_THREADS) {
        const unsigned long long kk = r < n_pow2 ? key[r] : 0ull;
        ranked[(long long)p * k_cache + r] = kk ? (int64_t)(0xffffffffu - (uint32_t)(kk & 0xffffffffu)) : -1;
    }
    if (tid == 0 && touched) touched[p] = n_touch;
}

// Global-memory variant for requests whose bitmap + sort keys exceed shared
// memory (block_size 1 over > 16K tokens, 128 over > 1M, ...): the distinct
// bitmap and per-block counts live in HBM, and the ranking is a top-k_cache
// select over the counts (select.cu, score mode: count desc, block id asc is
// exactly approx_topk's (score desc, id asc) order on integer-valued floats).
__global__ void block_bits_kernel(const int64_t* ids, long long ids_stride, int n_ids, int n_tokens, int words,
                                  uint32_t* bits) {
    const int p = blockIdx.y;
    const int64_t* ip = ids + p * ids_stride;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_ids; i += gridDim.x * blockDim.x) {
        const int64_t id = ip[i];
        if (id >= 0 && id < n_tokens) atomicOr(&bits[(long long)p * words + (id >> 5)], 1u << (id & 31));
    }
}

__global__ void block_counts_kernel(const uint32_t* bits, int words, int n_tokens, int block_size, int n_blocks,
                                    uint32_t* counts, float* fcounts, uint32_t* touched) {
    const int p = blockIdx.y;
    const uint32_t* bp = bits + (long long)p * words;
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < n_blocks; b += gridDim.x * blockDim.x) {
        const long long lo = (long long)b * block_size, hi = min((long long)n_tokens, lo + block_size);
        uint32_t cnt = 0;
        for (long long t = lo; t < hi;) {
            const int w = (int)(t >> 5), off = (int)(t & 31);
            const int take = (int)min((long long)(32 - off), hi - t);
            const uint32_t m = (take == 32 ? 0xffffffffu : ((1u << take) - 1u)) << off;
            cnt += __popc(bp[w] & m);
            t += take;
        }
        counts[(long long)p * n_blocks + b] = cnt;
        fcounts[(long long)p * n_blocks + b] = (float)cnt;
        if (cnt && touched) atomicAdd(&touched[p], 1u);
    }
}

// top ids of the count select -> ranked (-1 for untouched blocks / past n_blocks)
__global__ void block_ranked_kernel(const int64_t* top, int k_top, const uint32_t* counts, int n_blocks, int k_cache,
                                    int64_t* ranked) {
    const int p = blockIdx.y;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < k_cache; r += gridDim.x * blockDim.x) {
        int64_t v = -1;
        if (r < k_top) {
            const int64_t b = top[(long long)p * k_top + r];
            if (counts[(long long)p * n_blocks + b]) v = b;
        }
        ranked[(long long)p * k_cache + r] = v;
    }
}

}  // namespace

size_t block_rank_smem(size_t n_tokens, size_t n_blocks) {
    size_t n_pow2 = 1;
    while (n_pow2 < n_blocks) n_pow2 <<= 1;
    return n_pow2 * 8 + ceil_div(n_tokens, 32) * 4;
}

void launch_block_rank(pqkv_ctx* ctx, const int64_t* ids, size_t n_heads, size_t ids_stride, size_t n_ids,
                       size_t n_tokens, size_t block_size, size_t k_cache, uint32_t* bitmap, uint32_t* counts,
                       int64_t* ranked, uint32_t* touched, cudaStream_t st) {
    bind_device(ctx);
    if (block_size == 0) fail(PQKV_EINVAL, "block_rank: block_size must be >= 1");
    const size_t n_blocks = std::max<size_t>(1, ceil_div(n_tokens, block_size));
    size_t n_pow2 = 1;
    while (n_pow2 < n_blocks) n_pow2 <<= 1;
    const size_t smem = block_rank_smem(n_tokens, n_blocks);
    if (n_tokens > 0x7fffffff) fail(PQKV_EINVAL, "block_rank: too many tokens");
    if (n_heads == 0) return;
    if (smem > 200 * 1024) {
        const size_t words = ceil_div(n_tokens, 32);
        const size_t k_top = std::min(k_cache, n_blocks);
        char* buf = nullptr;
        const size_t o_bits = 0, o_cnt = round_up(n_heads * words * 4, 256),
                     o_f = o_cnt + round_up(n_heads * n_blocks * 4, 256),
                     o_top = o_f + round_up(n_heads * n_blocks * 4, 256), total = o_top + n_heads * k_top * 8 + 8;
        PQKV_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&buf), total, st));
        uint32_t* bits = bitmap ? bitmap : reinterpret_cast<uint32_t*>(buf + o_bits);
        float* fc = reinterpret_cast<float*>(buf + o_f);
        int64_t* top = reinterpret_cast<int64_t*>(buf + o_top);
        PQKV_CUDA(cudaMemsetAsync(bits, 0, n_heads * words * 4, st));
        if (touched) PQKV_CUDA(cudaMemsetAsync(touched, 0, n_heads * 4, st));
        const unsigned gx = (unsigned)std::max<size_t>(1, std::min<size_t>(4 * ctx->sm_count, ceil_div(n_ids, 256)));
        if (n_ids) {
            block_bits_kernel<<<dim3(gx, (unsigned)n_heads), 256, 0, st>>>(ids, (long long)ids_stride, (int)n_ids,
                                                                        (int)n_tokens, (int)words, bits);
            PQKV_LAUNCHED("block_bits_kernel");
        }
        const unsigned gb = (unsigned)std::max<size_t>(1, std::min<size_t>(4 * ctx->sm_count, ceil_div(n_blocks, 256)));
        block_counts_kernel<<<dim3(gb, (unsigned)n_heads), 256, 0, st>>>(bits, (int)words, (int)n_tokens,
                                                                      (int)block_size, (int)n_blocks, counts, fc,
                                                                      touched);
        PQKV_LAUNCHED("block_counts_kernel");
        if (k_top) {
            SelectSource ss;
            ss.scores = fc;
            ss.scores_stride = n_blocks;
            launch_select(ctx, ss, n_heads, n_blocks, k_top, nullptr, top, st, nullptr);
        }
        if (k_cache) {
            block_ranked_kernel<<<dim3((unsigned)ceil_div(k_cache, 256), (unsigned)n_heads), 256, 0, st>>>(
                top, (int)k_top, counts, (int)n_blocks, (int)k_cache, ranked);
            PQKV_LAUNCHED("block_ranked_kernel");
        }
        PQKV_CUDA(cudaFreeAsync(buf, st));
        return;
    }
    PQKV_CUDA(cudaFuncSetAttribute(block_rank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    block_rank_kernel<<<(unsigned)n_heads, BR_THREADS, smem, st>>>(
        ids, (long long)ids_stride, (int)n_ids, (int)n_tokens, (int)block_size, (int)n_blocks, (int)n_pow2,
        (int)k_cache, bitmap, counts, ranked, touched);
    PQKV_LAUNCHED("block_rank_kernel");
}

}  // namespace pqkv_dev
