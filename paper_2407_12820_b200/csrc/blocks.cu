// blocks.cu -- block-cache accounting of a fetch.
//
// KvStore::fetch_topk (kv_store.cpp:115-191) counts one lookup per distinct
// block of the requested tokens and then refreshes its fast-tier cache with
// the top-k_cache blocks of the request ranked by requested-token count, ties
// toward the lower block id (kv_store.cpp:158-166).  The per-request part --
// distinct tokens, per-block counts and that ranking -- runs here, one CTA
// per (layer, kv_head) unit, on the device-resident selection; the small
// sequential LRU/LFU state machine stays on the host (api.cpp).
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
    if (smem > 200 * 1024 || n_tokens > 0x7fffffff) fail(PQKV_EINVAL, "block_rank: too many tokens or blocks");
    if (n_heads == 0) return;
    PQKV_CUDA(cudaFuncSetAttribute(block_rank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    block_rank_kernel<<<(unsigned)n_heads, BR_THREADS, smem, st>>>(
        ids, (long long)ids_stride, (int)n_ids, (int)n_tokens, (int)block_size, (int)n_blocks, (int)n_pow2,
        (int)k_cache, bitmap, counts, ranked, touched);
    PQKV_LAUNCHED("block_rank_kernel");
}

}  // namespace pqkv_dev
