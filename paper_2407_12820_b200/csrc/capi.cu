// capi.cu -- C-ABI entry points (include/pqkv_c.h): argument validation with
// the reference's rejection rules, then the launchers in kmeans.cu,
// select.cu and attend.cu.  Nothing here computes on the host.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <cstdlib>
#include <vector>

#include "internal.cuh"

using namespace pqkv_dev;

namespace {

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

void need_ctx(pqkv_ctx* ctx) {
    if (!ctx) fail(PQKV_EINVAL, "pqkv: context is NULL");
    bind_device(ctx);
}

// PqConfig::create / validate (pq.cpp:13-31)
void check_pq(size_t m, size_t b, size_t d_h) {
    if (m < 1) fail(PQKV_EINVAL, "pq: m must be >= 1");
    if (b < 1 || b > 16) fail(PQKV_EINVAL, "pq: b must be in [1, 16]");
    if (d_h < 1 || d_h % m != 0) fail(PQKV_EINVAL, "pq: head_dim must be a positive multiple of m");
}

}  // namespace

extern "C" {

int pqkv_kmeans_fit(pqkv_ctx* ctx, const float* d_points, size_t n_problems, size_t problem_stride,
                    size_t row_stride, size_t n, size_t dim, size_t k, size_t max_iter,
                    const uint64_t* h_seeds, float* d_centroids, uint32_t* d_assign,
                    uint32_t* d_iterations, double* d_inertia, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        // kmeans_fit argument checks (kmeans.cpp:160-164)
        if (n < 1 || dim < 1) fail(PQKV_EINVAL, "kmeans: points must be a non-empty 2-d grid");
        if (k < 1) fail(PQKV_EINVAL, "kmeans: n_clusters must be >= 1");
        if (max_iter < 1) fail(PQKV_EINVAL, "kmeans: max_iter must be >= 1");
        if (!d_points || !d_centroids || (!d_assign) || (!h_seeds && n > k))
            fail(PQKV_EINVAL, "kmeans: NULL buffer");
        std::vector<uint64_t> seeds(n_problems, 0);
        if (h_seeds) seeds.assign(h_seeds, h_seeds + n_problems);
        KmeansBatch b{};
        b.points = d_points;
        b.n_problems = n_problems;
        b.problem_stride = problem_stride;
        b.row_stride = row_stride;
        b.n = n;
        b.dim = dim;
        b.k = k;
        b.max_iter = max_iter;
        b.m_sub = 1;
        b.seeds = seeds.data();
        b.centroids = d_centroids;
        b.assign = d_assign;
        b.iterations = d_iterations;
        b.inertia = d_inertia;
        launch_kmeans(ctx, b, as_stream(stream));
    });
}

int pqkv_pq_build(pqkv_ctx* ctx, const float* d_keys, size_t n_heads, size_t key_head_stride,
                  size_t s, size_t d_h, size_t m, size_t b, size_t max_iter,
                  const uint64_t* h_seeds, float* d_centroids, uint16_t* d_codes,
                  size_t codes_head_stride, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        check_pq(m, b, d_h);
        if (s < 1) fail(PQKV_EINVAL, "pq: need at least one key");
        if (max_iter < 1) fail(PQKV_EINVAL, "kmeans: max_iter must be >= 1");
        if (!d_keys || !d_centroids || !d_codes || !h_seeds) fail(PQKV_EINVAL, "pq: NULL buffer");
        // subspace j of head p uses seed_p + 0x9e3779b97f4a7c15 * (j + 1)  (pq.cpp:64-65)
        std::vector<uint64_t> seeds(n_heads * m);
        for (size_t p = 0; p < n_heads; ++p)
            for (size_t j = 0; j < m; ++j)
                seeds[p * m + j] = h_seeds[p] + 0x9e3779b97f4a7c15ull * (uint64_t)(j + 1);
        KmeansBatch kb{};
        kb.points = d_keys;
        kb.n_problems = n_heads * m;
        kb.problem_stride = key_head_stride;
        kb.row_stride = d_h;
        kb.n = s;
        kb.dim = d_h / m;
        kb.k = size_t{1} << b;
        kb.max_iter = max_iter;
        kb.m_sub = m;
        kb.seeds = seeds.data();
        kb.centroids = d_centroids;
        kb.codes = d_codes;
        kb.codes_head_stride = codes_head_stride;
        launch_kmeans(ctx, kb, as_stream(stream));
    });
}

int pqkv_pq_encode(pqkv_ctx* ctx, const float* d_keys, size_t n_heads, size_t key_stride,
                   size_t d_h, size_t m, size_t b, const float* d_centroids, uint16_t* d_codes,
                   size_t codes_head_stride, size_t row, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        check_pq(m, b, d_h);
        if (n_heads == 0) return;
        launch_encode(ctx, d_keys, n_heads, key_stride, d_h, m, size_t{1} << b, d_centroids, d_codes,
                      codes_head_stride, row, as_stream(stream));
    });
}

int pqkv_assign_nearest(pqkv_ctx* ctx, const float* d_points, size_t n, size_t dim,
                        const float* d_centroids, size_t k, uint32_t* d_assign, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        if (dim < 1) fail(PQKV_EINVAL, "assign_nearest: dimension mismatch");
        if (k < 1) fail(PQKV_EINVAL, "assign_nearest: need at least one centroid");
        launch_assign_nearest(ctx, d_points, n, dim, d_centroids, k, d_assign, as_stream(stream));
    });
}

int pqkv_pq_score(pqkv_ctx* ctx, const float* d_queries, size_t n_heads, size_t g, size_t d_h,
                  size_t m, size_t b, const float* d_centroids, const uint16_t* d_codes,
                  size_t codes_head_stride, size_t s, float* d_scores, size_t scores_head_stride,
                  void* stream) {
    return guard([&] {
        need_ctx(ctx);
        check_pq(m, b, d_h);
        if (g < 1) fail(PQKV_EINVAL, "pq: queries must be a non-empty 2-d grid");
        if (n_heads == 0) return;
        launch_score(ctx, d_queries, n_heads, g, d_h, m, size_t{1} << b, d_centroids, d_codes,
                     codes_head_stride, s, d_scores, scores_head_stride, as_stream(stream));
    });
}

int pqkv_topk(pqkv_ctx* ctx, const float* d_scores, size_t n_rows, size_t n, size_t scores_stride,
              size_t k, const uint8_t* d_excluded, int64_t* d_ids, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        if (k > n) fail(PQKV_EINVAL, "top_k: k too large for the candidate set");
        if (k == 0 || n_rows == 0) return;
        if (!d_ids) fail(PQKV_EINVAL, "top_k: NULL output");
        SelectSource src;
        src.scores = d_scores;
        src.scores_stride = scores_stride;
        src.excluded = d_excluded;
        if (!launch_select(ctx, src, n_rows, n, k, nullptr, d_ids, as_stream(stream), nullptr))
            fail(PQKV_EINVAL, "top_k: k too large for the candidate set");
    });
}

// Code-pair path: m = 2, C^2 <= 16384 pairs, per-pair row counts below
// 2^(32 - 2b) (pair_select packs (pair << (32 - 2b) | count)).
static bool tuple_ok(size_t m, size_t b, const void* th, const void* ch, size_t n) {
    return m == 2 && b >= 1 && b <= 7 && th && ch && n < (size_t{1} << (32 - 2 * b));
}

int pqkv_pq_tuple_tables(pqkv_ctx* ctx, size_t n_heads, size_t b, const uint16_t* d_codes,
                         size_t codes_head_stride, size_t row_begin, size_t row_end, uint32_t* d_tuple_hist,
                         uint16_t* d_tuple_chunk_hist, size_t n_chunks, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        if (b < 1 || b > 7) fail(PQKV_EINVAL, "tuple tables: need b in [1, 7] (m == 2)");
        if (!d_codes || !d_tuple_hist || !d_tuple_chunk_hist) fail(PQKV_EINVAL, "tuple tables: NULL buffer");
        launch_tuple_tables(ctx, d_codes, n_heads, codes_head_stride, size_t{1} << b, row_begin, row_end,
                            d_tuple_hist, d_tuple_chunk_hist, n_chunks, as_stream(stream));
    });
}

int pqkv_pq_search(pqkv_ctx* ctx, const float* d_queries, size_t n_heads, size_t g, size_t d_h,
                   size_t m, size_t b, const float* d_centroids, const uint16_t* d_codes,
                   size_t codes_head_stride, size_t s, size_t k, uint32_t* d_bitmap,
                   int64_t* d_ids, const uint32_t* d_tuple_hist, const uint16_t* d_tuple_chunk_hist, size_t tuple_chunks,
                   void* stream) {
    return guard([&] {
        need_ctx(ctx);
        check_pq(m, b, d_h);
        if (g < 1) fail(PQKV_EINVAL, "pq: queries must be a non-empty 2-d grid");
        if (k > s) fail(PQKV_EINVAL, "top_k: k too large for the candidate set");
        SelectSource src;
        src.queries = d_queries;
        src.g = g;
        src.d_h = d_h;
        src.m = m;
        src.C = size_t{1} << b;
        src.centroids = d_centroids;
        src.codes = d_codes;
        src.codes_head_stride = codes_head_stride;
        src.tuple_chunk_stride = tuple_chunks;
        if (tuple_ok(m, b, d_tuple_hist, d_tuple_chunk_hist, s))
            launch_select_tuple(ctx, src, d_tuple_hist, d_tuple_chunk_hist, n_heads, s, k, d_bitmap,
                                k ? d_ids : nullptr, as_stream(stream), nullptr);
        else
            launch_select(ctx, src, n_heads, s, k, d_bitmap, k ? d_ids : nullptr, as_stream(stream), nullptr);
    });
}

int pqkv_attend_rows(pqkv_ctx* ctx, const float* d_queries, size_t n_heads, size_t g, size_t d_h,
                     const float* d_keys, const float* d_values, size_t kv_head_stride,
                     const int64_t* d_rows, size_t t, int precision, float* d_out, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        if (d_h < 1) fail(PQKV_EINVAL, "attention: query dim must match key dim");
        if (g < 1) fail(PQKV_EINVAL, "attention: queries must be a non-empty 2-d grid");
        if (precision != PQKV_PREC_F32 && precision != PQKV_PREC_F64)
            fail(PQKV_EINVAL, "attention: unknown precision");
        launch_attend_rows(ctx, d_queries, n_heads, g, d_h, d_keys, d_values, kv_head_stride, d_rows,
                           t, precision, d_out, as_stream(stream));
    });
}

int pqkv_exact_scores(pqkv_ctx* ctx, const float* d_queries, size_t n_heads, size_t g, size_t d_h,
                      const float* d_keys, size_t kv_head_stride, const int64_t* d_rows, size_t t,
                      float* d_scores, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        if (d_h < 1) fail(PQKV_EINVAL, "attention: query dim must match key dim");
        launch_exact_scores(ctx, d_queries, n_heads, g, d_h, d_keys, kv_head_stride, d_rows, t, d_scores,
                            as_stream(stream));
    });
}

int pqkv_exact_topk(pqkv_ctx* ctx, const float* d_queries, size_t n_heads, size_t g, size_t d_h, const float* d_keys,
                    size_t kv_head_stride, size_t n, size_t k, int64_t* d_ids, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        if (d_h < 1) fail(PQKV_EINVAL, "attention: query dim must match key dim");
        if (g < 1) fail(PQKV_EINVAL, "attention: queries must be a non-empty 2-d grid");
        if (k > n) fail(PQKV_EINVAL, "top_k: k too large for the candidate set");
        if (!n_heads || !k) return;
        if (!d_queries || !d_keys || !d_ids) fail(PQKV_EINVAL, "exact_topk: NULL buffer");
        cudaStream_t st = as_stream(stream);
        float* scores = nullptr;
        PQKV_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&scores), n_heads * n * sizeof(float), st));
        launch_summed_scores(ctx, d_queries, n_heads, g, d_h, d_keys, kv_head_stride, n, scores, st);
        SelectSource src;
        src.scores = scores;
        src.scores_stride = n;
        launch_select(ctx, src, n_heads, n, k, nullptr, d_ids, st, nullptr);
        PQKV_CUDA(cudaFreeAsync(scores, st));
    });
}

int pqkv_attend_dense(pqkv_ctx* ctx, const float* d_queries, size_t n_heads, size_t g, size_t d_h, const float* d_keys,
                      const float* d_values, size_t kv_head_stride, size_t t, int precision, float* d_out,
                      void* stream) {
    return guard([&] {
        need_ctx(ctx);
        if (t < 1) fail(PQKV_EINVAL, "attention: need at least one token");
        if (!n_heads) return;
        cudaStream_t st = as_stream(stream);
        int64_t* rows = nullptr;
        PQKV_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&rows), n_heads * t * sizeof(int64_t), st));
        launch_iota_rows(ctx, rows, n_heads, t, st);
        const int rc = pqkv_attend_rows(ctx, d_queries, n_heads, g, d_h, d_keys, d_values, kv_head_stride, rows, t,
                                        precision, d_out, stream);
        PQKV_CUDA(cudaFreeAsync(rows, st));
        if (rc != PQKV_OK) fail(rc, pqkv_last_error());
    });
}

int pqkv_relative_error(pqkv_ctx* ctx, const float* d_got, const float* d_want, size_t n_rows, size_t n,
                        double* d_out, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        if (n_rows && (!d_got || !d_want || !d_out)) fail(PQKV_EINVAL, "relative_error: NULL buffer");
        launch_relative_error(ctx, d_got, d_want, n_rows, n, d_out, as_stream(stream));
    });
}

int pqkv_overlap_fraction(pqkv_ctx* ctx, const int64_t* d_got, size_t k_got, const int64_t* d_want, size_t k_want,
                          size_t n_rows, size_t n_ids, double* d_out, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        if (n_rows && !d_out) fail(PQKV_EINVAL, "overlap_fraction: NULL buffer");
        launch_overlap(ctx, d_got, k_got, d_want, k_want, n_rows, n_ids, d_out, as_stream(stream));
    });
}

static void check_layer(const pqkv_layer* L, size_t g, size_t k) {
    if (!L) fail(PQKV_EINVAL, "decode: layer is NULL");
    check_pq(L->m, L->b, L->d_h);
    if (g < 1) fail(PQKV_EINVAL, "decode: g must be >= 1");
    if (L->n_local < 1) fail(PQKV_EINVAL, "segments: n_local must be >= 1");
    if (L->n_init + L->n_local > L->total)
        fail(PQKV_EINVAL, "segments: n_init + n_local must be <= sequence length");
    size_t s_mid = L->total - L->n_init - L->n_local;
    if (s_mid < 1) fail(PQKV_EINVAL, "e2e: middle segment must be non-empty");
    if (k > s_mid) fail(PQKV_EINVAL, "e2e: k exceeds the middle segment");
    if (L->kv_head_stride < L->total * L->d_h) fail(PQKV_EINVAL, "decode: kv_head_stride too small");
    if (L->total > 0x7fffffff) fail(PQKV_EINVAL, "decode: context too long");
}

// The path pqkv_decode takes for a layer (pqkv_decode_plan reports it).
static int decode_mode(const pqkv_layer& L, size_t g, size_t k, bool with_ids) {
    const size_t s_mid = L.total - L.n_init - L.n_local;
    const bool tup = tuple_ok(L.m, L.b, L.tuple_hist, L.tuple_chunk_hist, s_mid);
    const bool fast = decode_fast_path(L, g);
    if (!fast) return PQKV_MODE_GENERIC;
    if (with_ids || k == 0) return PQKV_MODE_BITMAP;
    // g > 1: one launch, every (wide) attention CTA selects its head's pairs,
    // classifies its own codes and gathers.  g = 1: a pair-select launch
    // (one 256-thread CTA per head with the whole register file) chained
    // by programmatic launch to the attention grid, which stages its codes
    // while the select runs (north star 155.4 / 164.5 -> 152.9 / 160.4 us
    // against the 8-CTA-cluster fused launch, whose selecting CTA runs at 64
    // registers beside three others).  PQKV_PAIRS_FUSED=1 / PQKV_PAIRS_SPLIT=1
    // force either (experiments).
    static const bool force_split = std::getenv("PQKV_PAIRS_SPLIT") != nullptr;
    static const bool force_fused = std::getenv("PQKV_PAIRS_FUSED") != nullptr;
    if (tup && decode_pairs_fused(L, g) && !force_split && (g > 1 || force_fused)) return PQKV_MODE_PAIRS_FUSED;
    // per-head cluster computes ADC keys and radix-selects through DSMEM,
    // then gathers (same launch, or a second finer bitmap-mode launch)
    if (!(tup && L.b <= 6) && decode_keys_fused(L, g))
        return decode_keys_split(L, g) ? PQKV_MODE_KEYS_SPLIT : PQKV_MODE_KEYS_FUSED;
    // pair-level select launch -> attention classifies its own codes
    if (tup) return PQKV_MODE_PAIRS_SPLIT;
    return PQKV_MODE_BITMAP;
}

// pqkv_decode with the queries possibly in host-mapped memory (q_host):
// the split pair path's select reads them there and copies them to
// d_queries for the attention; every other path reads d_queries (filled by
// the caller).
static void decode_core(pqkv_ctx* ctx, const pqkv_layer* L, const float* d_queries, const float* q_host, size_t g,
                        size_t k, float* d_out, int64_t* d_ids, cudaStream_t st) {
        if (L->n_heads == 0) return;
        const size_t P = L->n_heads, s_mid = L->total - L->n_init - L->n_local;
        const size_t words = ceil_div(s_mid, 32), C = size_t{1} << L->b;
        const bool tup = tuple_ok(L->m, L->b, L->tuple_hist, L->tuple_chunk_hist, s_mid);
        SelectSource src;
        src.queries = d_queries;
        src.g = g;
        src.d_h = L->d_h;
        src.m = L->m;
        src.C = C;
        src.centroids = L->centroids;
        src.codes = L->codes;
        src.codes_head_stride = L->codes_head_stride;
        src.tuple_chunk_stride = L->tuple_chunks;
        const int mode = decode_mode(*L, g, k, d_ids != nullptr);
        if (q_host && mode != PQKV_MODE_PAIRS_SPLIT) fail(PQKV_EINVAL, "decode: host queries only on the split pair path");
        switch (mode) {
            case PQKV_MODE_PAIRS_FUSED:
                launch_decode_attend(ctx, *L, d_queries, g, nullptr, nullptr, nullptr, d_out, st, k);
                return;
            case PQKV_MODE_KEYS_FUSED:
            case PQKV_MODE_KEYS_SPLIT: {
                uint32_t* bm = mode == PQKV_MODE_KEYS_SPLIT
                                   ? static_cast<uint32_t*>(decode_workspace(ctx, P * words * 4))
                                   : nullptr;
                launch_decode_attend(ctx, *L, d_queries, g, bm, nullptr, nullptr, d_out, st, 0, k);
                return;
            }
            case PQKV_MODE_PAIRS_SPLIT: {
                char* ws = static_cast<char*>(decode_workspace(ctx, round_up(P * C * C, 256) + P * 2 * sizeof(int)));
                uint8_t* cls = reinterpret_cast<uint8_t*>(ws);
                int* cut = reinterpret_cast<int*>(ws + round_up(P * C * C, 256));
                unsigned* ready = ready_counters(ctx, P, st);
                if (q_host) {
                    src.queries = q_host;
                    src.queries_copy = const_cast<float*>(d_queries);
                }
                launch_tuple_select(ctx, src, L->tuple_hist, L->tuple_chunk_hist, P, s_mid, k, cls, cut, nullptr,
                                    nullptr, st, ready);
                launch_decode_attend(ctx, *L, d_queries, g, nullptr, cls, cut, d_out, st, 0, 0, ready);
                return;
            }
            default:
                break;
        }
        uint32_t* bm = static_cast<uint32_t*>(decode_workspace(ctx, P * words * 4));
        if (tup)
            launch_select_tuple(ctx, src, L->tuple_hist, L->tuple_chunk_hist, P, s_mid, k, bm, d_ids, st, nullptr);
        else
            launch_select(ctx, src, P, s_mid, k, bm, d_ids, st, nullptr);
        if (mode == PQKV_MODE_BITMAP) {
            launch_decode_attend(ctx, *L, d_queries, g, bm, nullptr, nullptr, d_out, st);
            return;
        }
        // generic geometry: ascending row lists, then the fp64 kernels
        const size_t T = L->n_init + k + L->n_local;
        int64_t* rows = nullptr;
        PQKV_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&rows), P * T * 8, st));
        launch_bitmap_rows(ctx, bm, P, words, L->n_init, L->n_local, L->total, T, rows, st);
        launch_exact(ctx, d_queries, P, g, L->d_h, L->keys, L->values, L->kv_head_stride, rows, T, d_out, st);
        PQKV_CUDA(cudaFreeAsync(rows, st));
}

int pqkv_decode(pqkv_ctx* ctx, const pqkv_layer* L, const float* d_queries, size_t g, size_t k,
                float* d_out, int64_t* d_ids, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        check_layer(L, g, k);
        decode_core(ctx, L, d_queries, nullptr, g, k, d_out, d_ids, as_stream(stream));
    });
}

int pqkv_decode_plan(pqkv_ctx* ctx, const pqkv_layer* L, size_t g, size_t k, int with_ids,
                     pqkv_decode_plan_t* out) {
    return guard([&] {
        need_ctx(ctx);
        if (!out) fail(PQKV_EINVAL, "decode_plan: out is NULL");
        check_layer(L, g, k);
        *out = pqkv_decode_plan_t{};
        out->mode = decode_mode(*L, g, k, with_ids != 0);
        out->launches = pqkv_decode_launches(L, g, with_ids);
        switch (out->mode) {
            case PQKV_MODE_PAIRS_FUSED: plan_decode_attend(ctx, *L, g, k, 0, false, out); break;
            case PQKV_MODE_KEYS_FUSED: plan_decode_attend(ctx, *L, g, 0, k, false, out); break;
            case PQKV_MODE_PAIRS_SPLIT: plan_decode_attend(ctx, *L, g, 0, 0, true, out); break;
            case PQKV_MODE_KEYS_SPLIT:
            case PQKV_MODE_BITMAP: plan_decode_attend(ctx, *L, g, 0, 0, false, out); break;
            default: break;
        }
    });
}

int pqkv_decode_step(pqkv_ctx* ctx, pqkv_layer* L, size_t codes_cap, const float* d_new_keys,
                     const float* d_new_values, const float* d_queries, size_t g, size_t k, float* d_out,
                     int64_t* d_ids, void* stream) {
    int rc = guard([&] {
        need_ctx(ctx);
        check_layer(L, g, 0);
        if (!d_new_keys || !d_new_values) fail(PQKV_EINVAL, "decode_step: NULL fresh K/V rows");
        // kv_store.cpp:81-83
        if (L->n_local == 0) fail(PQKV_ESTATE, "kv_store: local segment is empty");
        const size_t s_mid = L->total - L->n_init - L->n_local;
        if (L->kv_head_stride < (L->total + 1) * L->d_h) fail(PQKV_EINVAL, "decode_step: no room for the new token");
        if (codes_cap < s_mid + 1 || L->codes_head_stride < codes_cap * L->m)
            fail(PQKV_EINVAL, "decode_step: no room for the new code row");
        if (L->m == 2 && L->tuple_hist && L->tuple_chunk_hist &&
            L->tuple_chunks < ceil_div(s_mid + 1, PQKV_TUPLE_CHUNK))
            fail(PQKV_EINVAL, "decode_step: tuple_chunks must cover the grown middle segment");
        // everything pqkv_decode will check on the grown layer is checked
        // here, before evict_append mutates the cache, the codes and the pair
        // tables: a rejected step leaves the device state untouched
        pqkv_layer grown = *L;
        grown.total += 1;
        check_layer(&grown, g, k);
        if (L->n_heads == 0) return;
        launch_evict_append(ctx, *L, d_new_keys, d_new_values, as_stream(stream));
    });
    if (rc != PQKV_OK) return rc;
    L->total += 1;  // the step's mutation is on the stream; the layer now has one more token
    return pqkv_decode(ctx, L, d_queries, g, k, d_out, d_ids, stream);
}

int pqkv_gen_workload(pqkv_ctx* ctx, int kind, size_t s, size_t d_h, size_t h_kv, size_t g, size_t n_components,
                      double spread, double zipf_exponent, uint64_t seed, float* d_keys, float* d_values,
                      float* d_queries, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        if (!d_keys || !d_values || !d_queries) fail(PQKV_EINVAL, "workload: NULL buffer");
        launch_workload(ctx, kind, s, d_h, h_kv, g, n_components, spread, zipf_exponent, seed, d_keys, d_values,
                        d_queries, as_stream(stream));
    });
}

int pqkv_block_rank(pqkv_ctx* ctx, const int64_t* d_ids, size_t n_heads, size_t ids_stride, size_t n_ids,
                    size_t n_tokens, size_t block_size, size_t k_cache, uint32_t* d_bitmap, uint32_t* d_counts,
                    int64_t* d_ranked, uint32_t* d_touched, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        if ((!d_ids && n_ids) || !d_counts || (!d_ranked && k_cache)) fail(PQKV_EINVAL, "block_rank: NULL buffer");
        launch_block_rank(ctx, d_ids, n_heads, ids_stride, n_ids, n_tokens, block_size, k_cache, d_bitmap,
                          d_counts, d_ranked, d_touched, as_stream(stream));
    });
}

int pqkv_decode_attend(pqkv_ctx* ctx, const pqkv_layer* L, const float* d_queries, size_t g,
                       const uint32_t* d_bitmap, float* d_out, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        check_layer(L, g, 0);
        if (L->n_heads == 0) return;
        if (!decode_fast_path(*L, g)) fail(PQKV_EINVAL, "decode_attend: needs d_h == 128 and g in {1, 2, 4}");
        launch_decode_attend(ctx, *L, d_queries, g, d_bitmap, nullptr, nullptr, d_out, as_stream(stream));
    });
}

// The stream work of pqkv_decode_host: queries in, the decode launches, the
// outputs out (no synchronize).
static int decode_host_ops(pqkv_ctx* ctx, const pqkv_layer* L, const float* h_queries, size_t g, size_t k,
                           float* h_out, cudaStream_t st) {
    return guard([&] {
        const size_t qbytes = L->n_heads * g * L->d_h * sizeof(float);
        float* dq = static_cast<float*>(host_io_staging(ctx, 2 * qbytes));
        float* d_q = dq;
        float* d_o = dq + L->n_heads * g * L->d_h;
        // page-locked, device-mapped output buffer (cudaHostAlloc / pinned
        // tensors under UVA): the combining CTAs write the outputs straight
        // into host memory, so no D2H copy sits between the kernel and the
        // synchronize
        auto device_view = [](const void* h) -> void* {
            cudaPointerAttributes pa{};
            void* d = nullptr;
            if (cudaPointerGetAttributes(&pa, h) == cudaSuccess && pa.type == cudaMemoryTypeHost)
                d = pa.devicePointer;
            cudaGetLastError();
            return d;
        };
        float* mapped = static_cast<float*>(device_view(h_out));
        // with g > 1 the attention-kernel modes read each head's queries
        // once into shared memory, so page-locked, device-mapped queries go
        // straight in (no copy launch ahead of the kernel); g = 1 and the
        // other modes' select kernels read them repeatedly: device copy
        const int mode = decode_mode(*L, g, k, false);
        const bool direct = g > 1 && (mode == PQKV_MODE_PAIRS_FUSED || mode == PQKV_MODE_KEYS_FUSED ||
                                      mode == PQKV_MODE_KEYS_SPLIT);
        const float* mapped_q = direct ? static_cast<const float*>(device_view(h_queries)) : nullptr;
        // split pair path (g = 1 north star): its select kernel reads the
        // page-locked queries once and copies them for the attention grid
        const float* sel_q = mode == PQKV_MODE_PAIRS_SPLIT ? static_cast<const float*>(device_view(h_queries)) : nullptr;
        if (!mapped_q && !sel_q) PQKV_CUDA(cudaMemcpyAsync(d_q, h_queries, qbytes, cudaMemcpyHostToDevice, st));
        check_layer(L, g, k);
        decode_core(ctx, L, mapped_q ? mapped_q : d_q, sel_q, g, k, mapped ? mapped : d_o, nullptr, st);
        if (!mapped) PQKV_CUDA(cudaMemcpyAsync(h_out, d_o, qbytes, cudaMemcpyDeviceToHost, st));
    });
}

// Everything a captured pqkv_decode_host baked into its graph: the layer
// struct, the host buffers, g, k, the stream and the context's scratch and
// workspace allocations (a regrow between calls changes the key).
static std::vector<unsigned char> host_graph_key(const pqkv_ctx* ctx, const pqkv_layer* L, const float* hq, size_t g,
                                                 size_t k, const float* ho, cudaStream_t st) {
    std::vector<unsigned char> key(sizeof(pqkv_layer));
    std::memcpy(key.data(), L, sizeof(pqkv_layer));
    auto put = [&](const void* v, size_t n) {
        const auto* b = static_cast<const unsigned char*>(v);
        key.insert(key.end(), b, b + n);
    };
    put(&hq, sizeof hq);
    put(&ho, sizeof ho);
    put(&g, sizeof g);
    put(&k, sizeof k);
    put(&st, sizeof st);
    put(&ctx->arena, sizeof ctx->arena);
    put(&ctx->arena_bytes, sizeof ctx->arena_bytes);
    put(&ctx->ws, sizeof ctx->ws);
    put(&ctx->ws_bytes, sizeof ctx->ws_bytes);
    put(&ctx->io, sizeof ctx->io);
    put(&ctx->d_arrivals, sizeof ctx->d_arrivals);
    put(&ctx->d_ready, sizeof ctx->d_ready);
    return key;
}

int pqkv_decode_host(pqkv_ctx* ctx, const pqkv_layer* L, const float* h_queries, size_t g, size_t k,
                     float* h_out, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        check_layer(L, g, k);
        cudaStream_t st = as_stream(stream);
        // repeated calls replay a CUDA graph of the copy-in + decode launches
        // (one launch call instead of the copy and two kernel launches, and
        // no per-launch host work): captured on a context stream the second
        // time a key is seen, launched on the caller's stream
        static const bool graphs_on = std::getenv("PQKV_NO_GRAPHS") == nullptr;
        const bool graphable = graphs_on && !ctx->profiling && !ctx->sel_dump;
        std::vector<unsigned char> key;
        if (graphable) {
            key = host_graph_key(ctx, L, h_queries, g, k, h_out, st);
            for (auto& hg : ctx->host_graphs)
                if (hg.key == key) {
                    hg.last_use = ++ctx->host_graph_clock;
                    if (!hg.exec) break;  // this key did not capture: plain launches
                    PQKV_CUDA(cudaGraphLaunch(hg.exec, st));
                    PQKV_CUDA(cudaStreamSynchronize(st));
                    return;
                }
        }
        bool capture = false;
        const bool failed_before = graphable && std::any_of(ctx->host_graphs.begin(), ctx->host_graphs.end(),
                                                            [&](const auto& hg) { return hg.key == key; });
        if (graphable && !failed_before) {
            auto& seen = ctx->host_graph_seen;
            auto it = std::find(seen.begin(), seen.end(), key);
            if (it != seen.end()) {
                capture = true;
                seen.erase(it);
            } else {
                seen.push_back(key);
                if (seen.size() > 64) seen.erase(seen.begin());
            }
        }
        if (capture) {
            if (!ctx->capture_stream) PQKV_CUDA(cudaStreamCreateWithFlags(&ctx->capture_stream, cudaStreamNonBlocking));
            cudaGraph_t graph = nullptr;
            cudaGraphExec_t exec = nullptr;
            bool ok = cudaStreamBeginCapture(ctx->capture_stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
            if (ok) {
                const int rc = decode_host_ops(ctx, L, h_queries, g, k, h_out, ctx->capture_stream);
                ok = cudaStreamEndCapture(ctx->capture_stream, &graph) == cudaSuccess && rc == PQKV_OK && graph;
            }
            if (ok) ok = cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
            if (graph) cudaGraphDestroy(graph);
            cudaGetLastError();
            if (ok && host_graph_key(ctx, L, h_queries, g, k, h_out, st) == key) {
                if (ctx->host_graphs.size() >= 32) {  // drop the least recently used
                    auto lru = std::min_element(ctx->host_graphs.begin(), ctx->host_graphs.end(),
                                                [](const auto& a, const auto& b) { return a.last_use < b.last_use; });
                    if (lru->exec) cudaGraphExecDestroy(lru->exec);
                    ctx->host_graphs.erase(lru);
                }
                ctx->host_graphs.push_back({key, exec, ++ctx->host_graph_clock});
                PQKV_CUDA(cudaGraphLaunch(exec, st));
                PQKV_CUDA(cudaStreamSynchronize(st));
                return;
            }
            if (exec) cudaGraphExecDestroy(exec);
            if (ctx->host_graphs.size() >= 32) {
                auto lru = std::min_element(ctx->host_graphs.begin(), ctx->host_graphs.end(),
                                            [](const auto& a, const auto& b) { return a.last_use < b.last_use; });
                if (lru->exec) cudaGraphExecDestroy(lru->exec);
                ctx->host_graphs.erase(lru);
            }
            ctx->host_graphs.push_back({key, nullptr, ++ctx->host_graph_clock});  // remembered as not capturable
        }
        const int rc = decode_host_ops(ctx, L, h_queries, g, k, h_out, st);
        if (rc != PQKV_OK) fail(rc, pqkv_last_error());
        PQKV_CUDA(cudaStreamSynchronize(st));
    });
}

int pqkv_decode_launches(const pqkv_layer* L, size_t g, int with_ids) {
    if (!L || L->total < L->n_init + L->n_local) return 0;
    const bool tup = tuple_ok(L->m, L->b, L->tuple_hist, L->tuple_chunk_hist, L->total - L->n_init - L->n_local);
    switch (decode_mode(*L, g, 1, with_ids != 0)) {
        case PQKV_MODE_PAIRS_FUSED:
        case PQKV_MODE_KEYS_FUSED: return 1;
        case PQKV_MODE_KEYS_SPLIT:
        case PQKV_MODE_PAIRS_SPLIT: return 2;
        case PQKV_MODE_BITMAP: return (tup ? 2 : 1) + (with_ids ? 1 : 0) + 1;
        default: return (tup ? 2 : 1) + (with_ids ? 1 : 0) + 3;
    }
}

}  // extern "C"
