// metrics.cu -- the recall / output-error side of the experiments on the
// device: exact top-k of the summed group query,
// attention over every stored token, relative_error and overlap_fraction
// (experiments.cpp:26-70, attention.cpp:11-33), batched over (request,
// layer, kv_head) units so run_recall / run_e2e metrics need no host round
// trip per head.  Same arithmetic as the reference: f32 query sums in row
// order, fp64 sequential dots scaled once and rounded to f32, the topk.cpp
// tie rule, fp64 sequential error sums.
#include <cmath>

#include "internal.cuh"

namespace pqkv_dev {
namespace {

// sum_query_rows (experiments.cpp:26-31) then exact_scores (attention.cpp:11-26)
// against rows [0, n) of every unit; one thread per (unit, row).
__global__ void summed_scores_kernel(const float* queries, int g, int d_h, const float* keys, long long kv_head_stride,
                                     int n, double scale, float* scores) {
    extern __shared__ float qs[];  // the unit's summed query [d_h]
    const int p = blockIdx.y;
    for (int j = threadIdx.x; j < d_h; j += blockDim.x) {
        float acc = 0.0f;
        for (int r = 0; r < g; ++r) acc = __fadd_rn(acc, queries[((long long)p * g + r) * d_h + j]);
        qs[j] = acc;
    }
    __syncthreads();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float* k = keys + p * kv_head_stride + (long long)i * d_h;
    double acc = 0.0;
    for (int j = 0; j < d_h; ++j) acc = __fma_rn((double)qs[j], (double)__ldg(k + j), acc);
    scores[(long long)p * n + i] = (float)__dmul_rn(acc, scale);
}

// relative_error (experiments.cpp:41-50): sqrt(sum (got-want)^2 / sum want^2),
// sums in element order; one thread per row.
__global__ void relative_error_kernel(const float* got, const float* want, int rows, int n, double* out) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const float* a = got + (long long)r * n;
    const float* b = want + (long long)r * n;
    double num = 0.0, den = 0.0;
    for (int i = 0; i < n; ++i) {
        const double d = __dsub_rn((double)a[i], (double)b[i]);
        num = __dadd_rn(num, __dmul_rn(d, d));
        den = __dadd_rn(den, __dmul_rn((double)b[i], (double)b[i]));
    }
    out[r] = den > 0.0 ? sqrt(__ddiv_rn(num, den)) : sqrt(num);
}

// overlap_fraction (experiments.cpp:61-70): |got ∩ want| / |want| for id
// lists (ids in [0, n_ids); duplicates in `got` count once, as in the
// reference's set_intersection of sorted distinct lists); one CTA per row.
__global__ void overlap_kernel(const int64_t* got, int k_got, const int64_t* want, int k_want, int n_ids,
                               double* out) {
    extern __shared__ uint32_t bits[];
    const int r = blockIdx.x, words = (n_ids + 31) / 32;
    for (int w = threadIdx.x; w < words; w += blockDim.x) bits[w] = 0u;
    __syncthreads();
    for (int i = threadIdx.x; i < k_want; i += blockDim.x) {
        const int64_t id = want[(long long)r * k_want + i];
        if (id >= 0 && id < n_ids) atomicOr(&bits[id >> 5], 1u << (id & 31));
    }
    __syncthreads();
    __shared__ unsigned hits;
    if (threadIdx.x == 0) hits = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < k_got; i += blockDim.x) {
        const int64_t id = got[(long long)r * k_got + i];
        if (id >= 0 && id < n_ids) {
            const uint32_t m = 1u << (id & 31);
            if (atomicAnd(&bits[id >> 5], ~m) & m) atomicAdd(&hits, 1u);  // clear: a repeated id counts once
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) out[r] = k_want ? (double)hits / (double)k_want : 1.0;
}

__global__ void iota_rows_kernel(int64_t* rows, long long n, long long per) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        rows[i] = i % per;
}

}  // namespace

void launch_summed_scores(pqkv_ctx* ctx, const float* queries, size_t P, size_t g, size_t d_h, const float* keys,
                          size_t kv_head_stride, size_t n, float* scores, cudaStream_t st) {
    bind_device(ctx);
    if (!P || !n) return;
    const double scale = 1.0 / std::sqrt(static_cast<double>(d_h));
    dim3 grid((unsigned)ceil_div(n, 128), (unsigned)P);
    summed_scores_kernel<<<grid, 128, d_h * sizeof(float), st>>>(queries, (int)g, (int)d_h, keys,
                                                                (long long)kv_head_stride, (int)n, scale, scores);
    PQKV_LAUNCHED("summed_scores_kernel");
}

void launch_relative_error(pqkv_ctx* ctx, const float* got, const float* want, size_t rows, size_t n, double* out,
                           cudaStream_t st) {
    bind_device(ctx);
    if (!rows) return;
    relative_error_kernel<<<(unsigned)ceil_div(rows, 128), 128, 0, st>>>(got, want, (int)rows, (int)n, out);
    PQKV_LAUNCHED("relative_error_kernel");
}

void launch_overlap(pqkv_ctx* ctx, const int64_t* got, size_t k_got, const int64_t* want, size_t k_want, size_t rows,
                    size_t n_ids, double* out, cudaStream_t st) {
    bind_device(ctx);
    if (!rows) return;
    const size_t smem = ceil_div(n_ids, 32) * 4;
    if (smem > 200 * 1024) fail(PQKV_EINVAL, "overlap_fraction: id range too large");
    if (smem > 48 * 1024) PQKV_CUDA(cudaFuncSetAttribute(overlap_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    overlap_kernel<<<(unsigned)rows, 256, smem, st>>>(got, (int)k_got, want, (int)k_want, (int)n_ids, out);
    PQKV_LAUNCHED("overlap_kernel");
}

void launch_iota_rows(pqkv_ctx* ctx, int64_t* rows, size_t P, size_t t, cudaStream_t st) {
    bind_device(ctx);
    const size_t n = P * t;
    if (!n) return;
    const unsigned blocks = (unsigned)std::min<size_t>(ceil_div(n, 256), 8 * (size_t)ctx->sm_count);
    iota_rows_kernel<<<blocks, 256, 0, st>>>(rows, (long long)n, (long long)t);
    PQKV_LAUNCHED("iota_rows_kernel");
}

}  // namespace pqkv_dev
