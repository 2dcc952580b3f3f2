/*
 * pqkv_c.h -- C ABI of the B200-native PQCache hot paths (libpqkv.so).
 *
 * This is the drop-in boundary for the two data-parallel hot paths of the
 * reference `pqkv` library (/root/reference/proj):
 *
 *   (A) prefill PQ codebook build   pq_construct -> kmeans_fit   (pq.cpp:42-72,
 *                                                                kmeans.cpp:159-190)
 *   (B) decode retrieval             pq_score_gqa -> approx_topk -> fetch_topk /
 *                                    selective_attention          (pq.cpp:152-177,
 *                                    topk.cpp:8-25, kv_store.cpp:115-153,
 *                                    attention.cpp:35-104)
 *
 * Every entry point is `extern "C"`, takes plain pointers and sizes (no torch
 * or C++ types), returns a pqkv_status and records a thread-local message for
 * pqkv_last_error().  Pointers named d_* are device (HBM) pointers, h_* are
 * host pointers.  `stream` is a cudaStream_t passed as void* (NULL = legacy
 * default stream).  Calls are asynchronous on `stream` unless documented.
 *
 * Status mapping back to the reference's exception types (the C++ layer in
 * include/pqkv/pqkv.hpp re-throws them):
 *   PQKV_EINVAL  -> std::invalid_argument   PQKV_ERANGE -> std::out_of_range
 *   PQKV_ESTATE  -> std::logic_error        PQKV_ERUNTIME / PQKV_ECUDA -> std::runtime_error
 *
 * Exactness contract (checked by tests/ against oracle/):
 *   codes, k-means assignments, ADC scores and top-k index sets are
 *   bit-identical to the reference; centroids are the reference's fp64 means
 *   rounded once to f32 (bit-identical); attention outputs are within 1e-3
 *   relative on the fp32 fast path (PQKV_PREC_F32) and follow the reference's
 *   fp64 arithmetic order on PQKV_PREC_F64.
 *
 * Threading: one pqkv_ctx owns a scratch arena and must not be used by two
 * host threads at once; create one context per host thread / stream.
 */
#ifndef PQKV_C_H
#define PQKV_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PQKV_ABI_VERSION 2

#if defined(__GNUC__)
#define PQKV_API __attribute__((visibility("default")))
#else
#define PQKV_API
#endif

typedef enum {
    PQKV_OK = 0,
    PQKV_EINVAL = 1,   /* std::invalid_argument */
    PQKV_ERANGE = 2,   /* std::out_of_range */
    PQKV_ESTATE = 3,   /* std::logic_error */
    PQKV_ERUNTIME = 4, /* std::runtime_error */
    PQKV_ECUDA = 5     /* CUDA error (runtime_error) */
} pqkv_status;

typedef enum { PQKV_PREC_F32 = 0, PQKV_PREC_F64 = 1 } pqkv_precision;

/* Middle rows per chunk of the code-pair chunk histogram (see
 * pqkv_pq_tuple_tables). */
#define PQKV_TUPLE_CHUNK 4096
/* u64 timestamps per attention CTA recorded in profiling mode */
#define PQKV_PROF_SLOTS 24

/* k-means assign-step arithmetic.  Both produce bit-identical assignments:
 * EXACT evaluates every distance in the reference's fp64 order;
 * FILTERED evaluates fp32 distances with a rigorous error bound and
 * re-evaluates only the points whose nearest centroid is not certified. */
typedef enum { PQKV_ASSIGN_FILTERED = 0, PQKV_ASSIGN_EXACT = 1 } pqkv_assign_mode;

typedef struct pqkv_ctx pqkv_ctx;

/* ---- context ---------------------------------------------------------- */
PQKV_API int pqkv_abi_version(void);
PQKV_API const char* pqkv_last_error(void);
/* Binds `device` and allocates the scratch arena lazily. */
PQKV_API int pqkv_ctx_create(int device, pqkv_ctx** out);
PQKV_API int pqkv_ctx_destroy(pqkv_ctx* ctx);
/* Assign-step mode for subsequent builds on this context (default FILTERED). */
PQKV_API int pqkv_ctx_set_assign_mode(pqkv_ctx* ctx, int mode);
/* Counters of the last build on this context: fp64 re-checked points. */
PQKV_API int pqkv_ctx_last_build_stats(pqkv_ctx* ctx, uint64_t* rechecked_points, uint64_t* total_points);

/* SM cycles per build phase of problem 0 of the last build (profiling):
 * [0] k-means++ running sums + search, [1] k-means++ distances,
 * [2] assign + repair, [4] ordered update, [5] other. */
PQKV_API int pqkv_ctx_last_build_profile(pqkv_ctx* ctx, uint64_t cycles[8]);

/* Profiling mode (off by default): the attention kernel records per-CTA
 * phase timestamps; pqkv_ctx_last_decode_profile returns mean SM cycles per
 * CTA: [0] row-list prologue (incl. pair select), [1] pair select + DSMEM
 * share of [0], [2] gather + softmax, [3] number of CTAs. */
PQKV_API int pqkv_ctx_set_profiling(pqkv_ctx* ctx, int on);
/* Test hook: when d_bitmap != NULL, the fused single-launch decodes also
 * write their selection words (bit r = middle row r selected) to
 * d_bitmap [n_heads][ceil(s_mid/32)]. */
PQKV_API int pqkv_ctx_set_selection_dump(pqkv_ctx* ctx, uint32_t* d_bitmap);
PQKV_API int pqkv_ctx_last_decode_profile(pqkv_ctx* ctx, double out[4]);
/* Raw per-CTA timestamps of the last attention launch: PQKV_PROF_SLOTS u64 per CTA --
 * clock64 at start / after pair select / after the row list / after the
 * gather; globaltimer ns at start / after the row list / after the gather /
 * at exit; clock64 at the pair-select phase marks 0..6 (cluster rank 0) and
 * after the first cluster barrier; [16] SM id, [17] cluster rank.  Key-path
 * select (PQKV_PROF_SELECT=1 profiles that launch): [8..15] clock64 phase
 * marks, [21] value passes | candidate path << 8, [22] candidates in the
 * final bin, [23] that bin's cluster-wide count.
 * *n_ctas = CTAs; copies min(cap, PQKV_PROF_SLOTS*n). */
PQKV_API int pqkv_ctx_decode_profile_raw(pqkv_ctx* ctx, uint64_t* out, size_t cap, size_t* n_ctas);

/* ---- device memory helpers (for FFI hosts without a CUDA runtime) ----- */
PQKV_API int pqkv_device_alloc(pqkv_ctx* ctx, size_t bytes, void** out);
PQKV_API int pqkv_device_free(pqkv_ctx* ctx, void* ptr);
/* kind: 0 host->device, 1 device->host, 2 device->device; synchronous. */
PQKV_API int pqkv_copy(pqkv_ctx* ctx, void* dst, const void* src, size_t bytes, int kind);
PQKV_API int pqkv_stream_sync(pqkv_ctx* ctx, void* stream);
/* Row scatter into a token-indexed K/V buffer (host runtimes keep a device
 * copy of a KV cache this way): row i of d_src_k / d_src_v (n x d_h) goes
 * to token d_rows[i] of d_dst_k / d_dst_v (row t at + t*d_h). */
PQKV_API int pqkv_scatter_rows(pqkv_ctx* ctx, const float* d_src_k, const float* d_src_v, const int64_t* d_rows,
                               size_t n, size_t d_h, float* d_dst_k, float* d_dst_v, void* stream);

/* ---- geometry: PqConfig::create (pq.cpp:13-25) ------------------------- */
PQKV_API int pqkv_pq_config(size_t m, size_t b, size_t d_h, size_t* d_m, size_t* n_clusters);
/* codes_memory_ratio (pq.cpp:179-182) */
PQKV_API int pqkv_codes_memory_ratio(size_t m, size_t b, size_t d_h, double* ratio);

/* ---- (A) build --------------------------------------------------------- */

/* kmeans_fit (kmeans.cpp:159-190) for n_problems independent problems.
 * Problem q's point i is the `dim` contiguous floats at
 *   d_points + q*problem_stride + i*row_stride.
 * h_seeds[q] is the kmeans_fit seed.  Outputs: d_centroids [q][k][dim] f32,
 * d_assign [q][n] u32, d_iterations [q] u32 (nullable), d_inertia
 * [q][max_iter] f64 (nullable; computed only when non-NULL). */
PQKV_API int pqkv_kmeans_fit(pqkv_ctx* ctx, const float* d_points, size_t n_problems,
                    size_t problem_stride, size_t row_stride, size_t n, size_t dim, size_t k,
                    size_t max_iter, const uint64_t* h_seeds, float* d_centroids,
                    uint32_t* d_assign, uint32_t* d_iterations, double* d_inertia,
                    void* stream);

/* pq_construct (pq.cpp:42-72) for n_heads heads at once: the m subspace
 * problems of every head run concurrently.  d_keys: head p's token i at
 * d_keys + p*key_head_stride + i*d_h.  h_seeds[p] is head p's pq_construct
 * seed (subspace j uses seed + 0x9e3779b97f4a7c15*(j+1)).  Outputs:
 * d_centroids [p][m][2^b][d_m] f32; d_codes: head p's token i row of m u16 at
 * d_codes + p*codes_head_stride + i*m. */
PQKV_API int pqkv_pq_build(pqkv_ctx* ctx, const float* d_keys, size_t n_heads, size_t key_head_stride,
                  size_t s, size_t d_h, size_t m, size_t b, size_t max_iter,
                  const uint64_t* h_seeds, float* d_centroids, uint16_t* d_codes,
                  size_t codes_head_stride, void* stream);

/* pq_encode_one (pq.cpp:74-99) + append_code (pq.cpp:101-108) for n_heads
 * heads: key p (d_keys + p*key_stride) is encoded against head p's f32
 * centroids and its m-entry code row is written to
 * d_codes + p*codes_head_stride + row*m. */
PQKV_API int pqkv_pq_encode(pqkv_ctx* ctx, const float* d_keys, size_t n_heads, size_t key_stride,
                   size_t d_h, size_t m, size_t b, const float* d_centroids,
                   uint16_t* d_codes, size_t codes_head_stride, size_t row, void* stream);

/* assign_nearest (kmeans.cpp:192-220). */
PQKV_API int pqkv_assign_nearest(pqkv_ctx* ctx, const float* d_points, size_t n, size_t dim,
                        const float* d_centroids, size_t k, uint32_t* d_assign, void* stream);

/* ---- (B) decode retrieval ---------------------------------------------- */

/* Code-pair tables for the m == 2 fast selection path (b <= 7): for every
 * head, d_tuple_hist [p][C*C] u32 counts middle rows per code pair
 * (c0*C + c1) and d_tuple_chunk_hist [p][ceil(cap/PQKV_TUPLE_CHUNK)][C*C] u16
 * counts them per PQKV_TUPLE_CHUNK-row chunk.  ADDS the rows
 * [row_begin, row_end) of every head (zero the tables before the first call;
 * after an append call it again with the appended rows).  n_chunks is the
 * chunk dimension of d_tuple_chunk_hist. */
PQKV_API int pqkv_pq_tuple_tables(pqkv_ctx* ctx, size_t n_heads, size_t b, const uint16_t* d_codes,
                                  size_t codes_head_stride, size_t row_begin, size_t row_end,
                                  uint32_t* d_tuple_hist, uint16_t* d_tuple_chunk_hist,
                                  size_t n_chunks, void* stream);

/* pq_score_gqa (pq.cpp:113-161) for n_heads heads: d_queries [p][g][d_h],
 * codes as in pqkv_pq_build, d_scores + p*scores_head_stride + i. */
PQKV_API int pqkv_pq_score(pqkv_ctx* ctx, const float* d_queries, size_t n_heads, size_t g, size_t d_h,
                  size_t m, size_t b, const float* d_centroids, const uint16_t* d_codes,
                  size_t codes_head_stride, size_t s, float* d_scores,
                  size_t scores_head_stride, void* stream);

/* top_k_desc / approx_topk (topk.cpp:8-25, pq.cpp:174-177) for n_rows rows:
 * the k largest of d_scores + r*scores_stride [0..n) that are not excluded
 * (d_excluded + r*n, u8, nullable), written to d_ids + r*k in (score desc,
 * id asc) order.  EINVAL when k exceeds the candidate count (checked on
 * device; the call synchronizes `stream` to report it). */
PQKV_API int pqkv_topk(pqkv_ctx* ctx, const float* d_scores, size_t n_rows, size_t n,
              size_t scores_stride, size_t k, const uint8_t* d_excluded, int64_t* d_ids,
              void* stream);

/* Fused pq_score_gqa + approx_topk without materialising scores: builds the
 * fp64 ADC table in shared memory, scans the codes and radix-selects the k
 * best middle rows of each head with the reference's tie rule.  Writes the
 * selection bitmap d_bitmap [p][ceil(s/32)] u32 (bit r of the middle row r;
 * nullable) and/or the ordered ids d_ids [p][k] (nullable).  With m == 2,
 * b <= 7 and the code-pair tables of pqkv_pq_tuple_tables (nullable) the
 * selection runs over code pairs instead of tokens. */
PQKV_API int pqkv_pq_search(pqkv_ctx* ctx, const float* d_queries, size_t n_heads, size_t g, size_t d_h,
                   size_t m, size_t b, const float* d_centroids, const uint16_t* d_codes,
                   size_t codes_head_stride, size_t s, size_t k, uint32_t* d_bitmap,
                   int64_t* d_ids, const uint32_t* d_tuple_hist,
                   const uint16_t* d_tuple_chunk_hist, size_t tuple_chunks, void* stream);

/* Softmax attention over explicit row lists (softmax_attention,
 * gqa_group_attention, selective_attention: attention.cpp:35-104).  For head
 * p, query row r: softmax over d_rows[p][0..t) of K/V rows
 * (d_keys + p*kv_head_stride + row*d_h) -> d_out [p][g][d_h]. */
PQKV_API int pqkv_attend_rows(pqkv_ctx* ctx, const float* d_queries, size_t n_heads, size_t g,
                     size_t d_h, const float* d_keys, const float* d_values,
                     size_t kv_head_stride, const int64_t* d_rows, size_t t, int precision,
                     float* d_out, void* stream);

/* exact_scores (attention.cpp:11-26): f32(fp64 dot * 1/sqrt(d_h)) for every
 * head p, query row r and list row i -> d_scores [p][g][t].  Bit-identical. */
PQKV_API int pqkv_exact_scores(pqkv_ctx* ctx, const float* d_queries, size_t n_heads, size_t g,
                               size_t d_h, const float* d_keys, size_t kv_head_stride,
                               const int64_t* d_rows, size_t t, float* d_scores, void* stream);

/* ---- experiment metrics on the device (experiments.cpp:26-139) ---- */

/* exact_topk of the summed group query (sum_query_rows + exact_scores +
 * top_k_desc, experiments.cpp:26-31, attention.cpp:11-33) for every unit p:
 * the k best of key rows [0, n) of d_keys + p*kv_head_stride for the f32 sum
 * of d_queries [p][0..g) -> d_ids [p][k], (score desc, id asc). */
PQKV_API int pqkv_exact_topk(pqkv_ctx* ctx, const float* d_queries, size_t n_heads, size_t g, size_t d_h,
                             const float* d_keys, size_t kv_head_stride, size_t n, size_t k, int64_t* d_ids,
                             void* stream);
/* Softmax attention of d_queries [p][g][d_h] over key/value rows [0, t) of
 * every unit (gqa_group_attention over all stored tokens). */
PQKV_API int pqkv_attend_dense(pqkv_ctx* ctx, const float* d_queries, size_t n_heads, size_t g, size_t d_h,
                               const float* d_keys, const float* d_values, size_t kv_head_stride, size_t t,
                               int precision, float* d_out, void* stream);
/* relative_error (experiments.cpp:41-50) per row of n floats -> d_out [rows] f64. */
PQKV_API int pqkv_relative_error(pqkv_ctx* ctx, const float* d_got, const float* d_want, size_t n_rows, size_t n,
                                 double* d_out, void* stream);
/* overlap_fraction (experiments.cpp:61-70) per row: |got ∩ want| / |want|,
 * ids in [0, n_ids) -> d_out [rows] f64. */
PQKV_API int pqkv_overlap_fraction(pqkv_ctx* ctx, const int64_t* d_got, size_t k_got, const int64_t* d_want,
                                   size_t k_want, size_t n_rows, size_t n_ids, double* d_out, void* stream);
/* The seeder draws of run_recall (experiments.cpp:90-113; Rng, rng.hpp): for
 * each of h_kv heads one fork_seed (-> fork_seeds[h]) then, for every k of
 * ks[0..n_k), k distinct ids of [0, s) by partial Fisher-Yates
 * (-> random_ids[h][sum of earlier ks .. + k)). */
PQKV_API int pqkv_recall_seeds(uint64_t seed, size_t h_kv, const size_t* ks, size_t n_k, size_t s,
                               uint64_t* fork_seeds, int64_t* random_ids);

/* One decode layer's KV cache + PQ index, device resident.  Token ids of a
 * head are its row indices: init [0,n_init), middle [n_init, total-n_local)
 * (middle row r = token n_init+r = code row r), local [total-n_local, total),
 * i.e. the reference's three segments (kv_store.hpp:61-79) collapsed into one
 * HBM buffer per head. */
typedef struct {
    const float* keys;        /* [n_heads][kv_head_stride] f32, row = token id */
    const float* values;      /* same layout as keys */
    size_t kv_head_stride;    /* floats between heads (>= total*d_h) */
    size_t n_heads;           /* (request, layer, kv_head) units */
    size_t total;             /* tokens per head */
    size_t n_init, n_local;   /* SegmentConfig (model.hpp:30-36) */
    size_t d_h, m, b;         /* PqConfig */
    const float* centroids;   /* [n_heads][m][2^b][d_m] f32 */
    const uint16_t* codes;    /* head p, middle row r at codes + p*codes_head_stride + r*m */
    size_t codes_head_stride;
    /* optional code-pair tables (pqkv_pq_tuple_tables) for m == 2, b <= 7 */
    const uint32_t* tuple_hist;
    const uint16_t* tuple_chunk_hist;
    size_t tuple_chunks;      /* chunks per head of tuple_chunk_hist (0 = ceil(s_mid/PQKV_TUPLE_CHUNK)) */
} pqkv_layer;

/* Fused decode retrieval + sparse attention for one layer (the hot path):
 * ADC table -> code scan -> top-k select (bitmap) -> K/V gather of
 * init + selected + local rows -> split-K fp32 online softmax -> combine.
 * d_queries/d_out [n_heads][g][d_h].  d_ids (nullable) additionally receives
 * the selected middle rows in (score desc, id asc) order. */
PQKV_API int pqkv_decode(pqkv_ctx* ctx, const pqkv_layer* layer, const float* d_queries, size_t g,
                size_t k, float* d_out, int64_t* d_ids, void* stream);

/* The attention half of pqkv_decode for a given selection bitmap
 * d_bitmap [n_heads][ceil(s_mid/32)] (bit r = middle row r, as written by
 * pqkv_pq_search): gather of init + selected + local rows, split-K fp32
 * online softmax and the partial combine. */
PQKV_API int pqkv_decode_attend(pqkv_ctx* ctx, const pqkv_layer* layer, const float* d_queries,
                                size_t g, const uint32_t* d_bitmap, float* d_out, void* stream);

/* pqkv_decode with HOST query/output buffers: copies h_queries in, runs the
 * fused layer, copies d_out back and synchronizes `stream`. */
PQKV_API int pqkv_decode_host(pqkv_ctx* ctx, const pqkv_layer* layer, const float* h_queries,
                     size_t g, size_t k, float* h_out, void* stream);

/* One decode step of the e2e loop (run_e2e, experiments.cpp:197-260) for every
 * head: evict_local_append (kv_store.cpp:77-90) -- the fresh K/V rows
 * d_new_keys / d_new_values [n_heads][d_h] become token `total` (the newest
 * local token) and the oldest local token (total - n_local) joins the middle
 * segment: its key is encoded against the head's centroids (pq_encode_one,
 * pq.cpp:74-99), appended as code row s_mid (append_code, pq.cpp:101-108) and
 * counted in the code-pair tables when present -- then pqkv_decode with the
 * step's queries.  layer->total is incremented on success.  The K/V, code
 * and chunk-table buffers must be writable with room for the new row
 * (kv_head_stride >= (total+1)*d_h, codes_cap rows of codes per head,
 * tuple_chunks covering s_mid+1 rows). */
PQKV_API int pqkv_decode_step(pqkv_ctx* ctx, pqkv_layer* layer, size_t codes_cap, const float* d_new_keys,
                              const float* d_new_values, const float* d_queries, size_t g, size_t k,
                              float* d_out, int64_t* d_ids, void* stream);

/* Block-cache accounting of a fetch (kv_store.cpp:115-191), per head p:
 * the distinct requested tokens among d_ids + p*ids_stride [0..n_ids) (ids
 * outside [0, n_tokens) are ignored) -> d_bitmap [p][ceil(n_tokens/32)] u32
 * (nullable), distinct tokens per block of block_size token ids ->
 * d_counts [p][ceil(n_tokens/block_size)] u32, the k_cache most requested
 * blocks, count desc then block id asc (kv_store.cpp:158-166) -> d_ranked
 * [p][k_cache] i64 (-1 padded), and the number of distinct blocks touched
 * -> d_touched [p] (nullable). */
PQKV_API int pqkv_block_rank(pqkv_ctx* ctx, const int64_t* d_ids, size_t n_heads, size_t ids_stride,
                             size_t n_ids, size_t n_tokens, size_t block_size, size_t k_cache,
                             uint32_t* d_bitmap, uint32_t* d_counts, int64_t* d_ranked, uint32_t* d_touched,
                             void* stream);

/* Synthetic KV workloads on the device (workload.cpp:16-117 distributions,
 * counter-based generator: every value is a function of (seed, head, token,
 * dim), so it is not the reference's sequential mt19937_64 stream).  kind:
 * PQKV_WORKLOAD_GAUSSIAN (n_components means, spread) or
 * PQKV_WORKLOAD_POWERLAW (zipf exponent; scaled exact score of rank r =
 * 8/(r+1)^zipf).  Outputs d_keys/d_values [h_kv][s][d_h], d_queries
 * [h_kv][g][d_h] f32. */
enum { PQKV_WORKLOAD_GAUSSIAN = 0, PQKV_WORKLOAD_POWERLAW = 1 };
PQKV_API int pqkv_gen_workload(pqkv_ctx* ctx, int kind, size_t s, size_t d_h, size_t h_kv, size_t g,
                               size_t n_components, double spread, double zipf_exponent, uint64_t seed,
                               float* d_keys, float* d_values, float* d_queries, void* stream);

/* Number of kernels pqkv_decode launches for this geometry (for the bench's
 * gpu_launches accounting). */
PQKV_API int pqkv_decode_launches(const pqkv_layer* layer, size_t g, int with_ids);

/* ---- multi-GPU: head / request sharded decode over NCCL ----
 * Units shard across GPUs with no exchange inside the path; the one
 * collective is the all-gather of the per-unit attention outputs, batched
 * over the layers of a call.  NCCL is loaded at run time (libnccl.so.2, the
 * process's own when already loaded).  Protocol = ncclCommInitRank: rank 0
 * calls pqkv_comm_unique_id, the host broadcasts the 128 bytes, every rank
 * calls pqkv_comm_init. */
typedef struct pqkv_comm pqkv_comm;
PQKV_API int pqkv_comm_unique_id(uint8_t out[128]);
PQKV_API int pqkv_comm_init(pqkv_ctx* ctx, const uint8_t id[128], int n_ranks, int rank, pqkv_comm** out);
PQKV_API int pqkv_comm_destroy(pqkv_comm* comm);
/* This rank decodes its units of every layer (layers[l]: this rank's shard,
 * at most units_per_rank units; fewer pad with zero rows) with queries
 * d_queries[l] [units][g][d_h], then one all-gather over the communicator
 * (its own stream, ordered after the decodes; `stream` waits for it) fills
 * d_out_all [n_ranks][n_layers][units_per_rank][g][d_h]. */
PQKV_API int pqkv_decode_sharded(pqkv_ctx* ctx, pqkv_comm* comm, const pqkv_layer* layers, size_t n_layers,
                                 size_t units_per_rank, const float* const* d_queries, size_t g, size_t k,
                                 float* d_out_all, void* stream);

/* The launch plan pqkv_decode picks for this layer, g, k (on ctx's device):
 * which fused mode runs, how the middle tokens are split over attention CTAs
 * and how those CTAs are grouped.  Used by tests to pin a parity case to the
 * exact geometry a benchmark runs, and by tools for reporting. */
enum {
    PQKV_MODE_PAIRS_FUSED = 1, /* m == 2, b <= 6 + pair tables: select fused into the attention (1 launch) */
    PQKV_MODE_KEYS_FUSED = 2,  /* per-token ADC keys, cluster radix select fused into the attention */
    PQKV_MODE_KEYS_SPLIT = 3,  /* cluster key select -> bitmap, then a bitmap-mode attention launch */
    PQKV_MODE_PAIRS_SPLIT = 4, /* pair select launch -> attention classifies its codes */
    PQKV_MODE_BITMAP = 5,      /* separate select (+ ordered ids) -> bitmap-mode attention */
    PQKV_MODE_GENERIC = 6      /* d_h != 128 or g not in {1,2,4}: row lists + the fp64 kernels */
};
typedef struct {
    int mode;               /* PQKV_MODE_* */
    int launches;           /* kernels per call (pqkv_decode_launches) */
    int chunk_tokens;       /* middle tokens per attention CTA (fused / bitmap modes) */
    int ctas_per_head;      /* attention CTAs per head (after cluster padding) */
    int cluster;            /* CTAs per thread-block cluster of the attention launch */
    int staged;             /* pair modes: the CTA's codes are staged in shared memory */
    int window;             /* selected rows expanded per gather window (== chunk_tokens: one window) */
    int ring_depth;         /* g > 1: rows in flight per gather slot */
    size_t smem_bytes;      /* dynamic shared memory per attention CTA */
} pqkv_decode_plan_t;
PQKV_API int pqkv_decode_plan(pqkv_ctx* ctx, const pqkv_layer* layer, size_t g, size_t k, int with_ids,
                              pqkv_decode_plan_t* out);

#ifdef __cplusplus
}
#endif

#endif /* PQKV_C_H */
