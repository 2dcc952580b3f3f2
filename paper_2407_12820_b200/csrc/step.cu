// step.cu -- on-device eviction for the e2e decode loop.
//
// KvStore::evict_local_append (kv_store.cpp:77-90) on the flat per-head
// layout: the fresh K/V row becomes token `total`, the oldest local token
// (total - n_local) moves from the local window into the middle segment,
// which on this layout only moves the segment boundary; its key is encoded
// with pq_encode_one (pq.cpp:74-99) and appended as middle code row s_mid
// (append_code, pq.cpp:101-108), and the code-pair tables of the m = 2 path
// count the new row.  One CTA per head; the decode that follows is the
// regular fused launch.
#include <cmath>

#include "internal.cuh"

namespace pqkv_dev {
namespace {

constexpr int ST_THREADS = 128;
constexpr int ST_WARPS = ST_THREADS / 32;

struct StepArgs {
    float* keys;
    float* values;
    long long kv_head_stride;
    const float* new_keys;  // [P][d_h]
    const float* new_values;
    int d_h, m, C, total, n_local, s_mid;
    const float* centroids;  // [P][m][C][d_m]
    uint16_t* codes;
    long long codes_head_stride;
    uint32_t* thist;  // [P][C*C] or null
    uint16_t* chist;  // [P][tchunks][C*C] or null
    long long tchunks;
};

__global__ void __launch_bounds__(ST_THREADS) evict_append_kernel(StepArgs a) {
    const int p = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int d_m = a.d_h / a.m;
    __shared__ uint32_t code_s[16];
    float* kp = a.keys + p * a.kv_head_stride;
    float* vp = a.values + p * a.kv_head_stride;
    // the evicted token's key: the oldest local row (written by an earlier
    // step or the prefill; the fresh row goes to a different row)
    const float* key = kp + (long long)(a.total - a.n_local) * a.d_h;
    const float* cen = a.centroids + (long long)p * a.m * a.C * d_m;
    for (int j = warp; j < a.m; j += ST_WARPS) {
        // pq_encode_one: nearest f32 centroid in fp64, separate sub/mul/add,
        // strict < in ascending c (lanes own c = lane mod 32, then a
        // lowest-index reduction)
        double best = INFINITY;
        int bi = 0x7fffffff;
        for (int c = lane; c < a.C; c += 32) {
            const float* cc = cen + ((long long)j * a.C + c) * d_m;
            double acc = 0.0;
            for (int t = 0; t < d_m; ++t) {
                const double diff = __dsub_rn((double)key[j * d_m + t], (double)cc[t]);
                acc = __dadd_rn(acc, __dmul_rn(diff, diff));
            }
            if (acc < best) { best = acc; bi = c; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(FULL, best, o);
            const int oi = __shfl_xor_sync(FULL, bi, o);
            if (ob < best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        if (lane == 0) {
            const uint32_t code = bi == 0x7fffffff ? 0u : (uint32_t)bi;
            if (j < 16) code_s[j] = code;
            a.codes[p * a.codes_head_stride + (long long)a.s_mid * a.m + j] = (uint16_t)code;
        }
    }
    // the fresh row: token `total`
    for (int t = tid; t < a.d_h; t += ST_THREADS) {
        kp[(long long)a.total * a.d_h + t] = a.new_keys[(long long)p * a.d_h + t];
        vp[(long long)a.total * a.d_h + t] = a.new_values[(long long)p * a.d_h + t];
    }
    __syncthreads();
    if (tid == 0 && a.thist) {  // m == 2: count the new middle row's code pair
        const uint32_t pair = code_s[0] * (uint32_t)a.C + code_s[1];
        const long long C2 = (long long)a.C * a.C;
        a.thist[p * C2 + pair] += 1u;
        a.chist[(p * a.tchunks + a.s_mid / PQKV_TUPLE_CHUNK) * C2 + pair] += 1u;
    }
}

}  // namespace

void launch_evict_append(pqkv_ctx* ctx, const pqkv_layer& L, const float* new_keys, const float* new_values,
                         cudaStream_t st) {
    bind_device(ctx);
    StepArgs a{};
    a.keys = const_cast<float*>(L.keys);
    a.values = const_cast<float*>(L.values);
    a.kv_head_stride = (long long)L.kv_head_stride;
    a.new_keys = new_keys;
    a.new_values = new_values;
    a.d_h = (int)L.d_h;
    a.m = (int)L.m;
    a.C = 1 << L.b;
    a.total = (int)L.total;
    a.n_local = (int)L.n_local;
    a.s_mid = (int)(L.total - L.n_init - L.n_local);
    a.centroids = L.centroids;
    a.codes = const_cast<uint16_t*>(L.codes);
    a.codes_head_stride = (long long)L.codes_head_stride;
    const bool tables = L.m == 2 && L.tuple_hist && L.tuple_chunk_hist;
    a.thist = tables ? const_cast<uint32_t*>(L.tuple_hist) : nullptr;
    a.chist = tables ? const_cast<uint16_t*>(L.tuple_chunk_hist) : nullptr;
    a.tchunks = (long long)(L.tuple_chunks ? L.tuple_chunks : ceil_div((size_t)a.s_mid + 1, PQKV_TUPLE_CHUNK));
    evict_append_kernel<<<(unsigned)L.n_heads, ST_THREADS, 0, st>>>(a);
    PQKV_LAUNCHED("evict_append_kernel");
}

}  // namespace pqkv_dev
