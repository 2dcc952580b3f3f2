// internal.cuh -- context object and the host-side launch API shared by the
// C-ABI translation units.
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "common.cuh"

struct pqkv_ctx {
    int device = 0;
    int sm_count = 148;
    int assign_mode = PQKV_ASSIGN_FILTERED;
    // Scratch arena: one device allocation grown on demand; carved per call.
    void* arena = nullptr;
    size_t arena_bytes = 0;
    // Pinned + device staging for the host-buffer entry points.
    void* pinned = nullptr;
    size_t pinned_bytes = 0;
    // Per-head arrival counters of the fused attention combine (kept zero
    // between launches by the kernel itself).
    unsigned* d_arrivals = nullptr;
    size_t n_arrivals = 0;
    // Per-unit counts of finished select CTAs of the split key path (the
    // gather polls them; reset by its combining CTAs).
    unsigned* d_ready = nullptr;
    size_t n_ready = 0;

    // Profiling mode: attention-kernel phase timestamps of the last launch.
    int profiling = 0;
    uint32_t* sel_dump = nullptr;  // test hook: fused decodes write their selection words here
    unsigned long long* d_prof = nullptr;
    size_t n_prof = 0;
    // Decode workspace (selection bitmap / pair classes between kernels).
    void* ws = nullptr;
    size_t ws_bytes = 0;
    // Device staging of pqkv_decode_host (queries in, outputs out).
    void* io = nullptr;
    size_t io_bytes = 0;
    // Device counters written by the build kernels (rechecked, total).
    unsigned long long* d_stats = nullptr;
    uint64_t last_rechecked = 0, last_total = 0;
    unsigned long long last_phase_cycles[8] = {};  // problem 0 of the last build
    // pqkv_decode_host: CUDA graphs of repeated calls (copy in + decode
    // launches), keyed by everything the captured launches bake in
    struct HostGraph {
        std::vector<unsigned char> key;
        cudaGraphExec_t exec = nullptr;
        unsigned long long last_use = 0;
    };
    std::vector<HostGraph> host_graphs;
    std::vector<std::vector<unsigned char>> host_graph_seen;  // keys seen once (captured on the second call)
    cudaStream_t capture_stream = nullptr;
    unsigned long long host_graph_clock = 0;
};

namespace pqkv_dev {

// Bump allocator over the context arena.  reserve() grows the arena (after a
// device synchronize) when a call needs more than is currently allocated, so
// one call's scratch never aliases another live buffer of the same call.
class Scratch {
public:
    Scratch(pqkv_ctx* ctx) : ctx_(ctx) {}
    // Two-phase use: plan() sizes, then commit() returns pointers in order.
    template <typename T>
    size_t plan(size_t count) {
        size_t off = round_up(total_, 256);
        total_ = off + count * sizeof(T);
        offsets_.push_back(off);
        return offsets_.size() - 1;
    }
    void commit();
    template <typename T>
    T* get(size_t handle) const {
        return reinterpret_cast<T*>(static_cast<char*>(ctx_->arena) + offsets_[handle]);
    }

private:
    pqkv_ctx* ctx_;
    size_t total_ = 0;
    std::vector<size_t> offsets_;
};

void bind_device(pqkv_ctx* ctx);
void set_last_error(const std::string& msg);

// Runs `f`, converting exceptions into a pqkv_status + pqkv_last_error().
template <class F>
int guard(F&& f) {
    try {
        f();
        set_last_error(std::string());
        return PQKV_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return PQKV_ERUNTIME;
    }
}
void* pinned_staging(pqkv_ctx* ctx, size_t bytes);
// Device staging owned by the context (never aliases the arena or the decode
// workspace); grown on demand after synchronizing the context's device.
void* host_io_staging(pqkv_ctx* ctx, size_t bytes);
// Multiprocessor count of the current device (cached per device id).
int current_sm_count();
unsigned* arrival_counters(pqkv_ctx* ctx, size_t n, cudaStream_t st);
unsigned* ready_counters(pqkv_ctx* ctx, size_t n, cudaStream_t st);


// ---- launchers implemented in the kernel translation units -----------------

struct KmeansBatch {
    const float* points;
    size_t n_problems, problem_stride, row_stride, n, dim, k, max_iter;
    // problem q = (head q / m_sub, subspace q % m_sub): element (q, i) lives at
    // points + (q / m_sub) * problem_stride + (q % m_sub) * dim + i*row_stride
    size_t m_sub;
    const uint64_t* seeds;  // host, one per problem (final kmeans_fit seed)
    float* centroids;       // [q][k][dim]
    uint32_t* assign;       // [q][n] (nullable when codes given)
    uint16_t* codes;        // pq_build output: head h row i entry j (nullable)
    size_t codes_head_stride;
    uint32_t* iterations;   // nullable
    double* inertia;        // nullable
};
void launch_kmeans(pqkv_ctx* ctx, const KmeansBatch& b, cudaStream_t stream);

void launch_workload(pqkv_ctx* ctx, int kind, size_t s, size_t d, size_t h, size_t g, size_t n_comp,
                     double spread, double zipf, uint64_t seed, float* keys, float* values, float* queries,
                     cudaStream_t st);
void launch_block_rank(pqkv_ctx* ctx, const int64_t* ids, size_t n_heads, size_t ids_stride, size_t n_ids,
                       size_t n_tokens, size_t block_size, size_t k_cache, uint32_t* bitmap, uint32_t* counts,
                       int64_t* ranked, uint32_t* touched, cudaStream_t st);
void launch_evict_append(pqkv_ctx* ctx, const pqkv_layer& L, const float* new_keys, const float* new_values,
                         cudaStream_t st);
void launch_encode(pqkv_ctx* ctx, const float* keys, size_t n_heads, size_t key_stride,
                   size_t d_h, size_t m, size_t C, const float* centroids, uint16_t* codes,
                   size_t codes_head_stride, size_t row, cudaStream_t stream);
void launch_assign_nearest(pqkv_ctx* ctx, const float* points, size_t n, size_t dim,
                           const float* centroids, size_t k, uint32_t* assign,
                           cudaStream_t stream);

void launch_score(pqkv_ctx* ctx, const float* queries, size_t n_heads, size_t g, size_t d_h,
                  size_t m, size_t C, const float* centroids, const uint16_t* codes,
                  size_t codes_head_stride, size_t s, float* scores, size_t scores_stride,
                  cudaStream_t stream);

// Selection source: either ADC (queries + index) or explicit scores.
struct SelectSource {
    // ADC mode
    const float* queries = nullptr;
    size_t g = 0, d_h = 0, m = 0, C = 0;
    const float* centroids = nullptr;
    const uint16_t* codes = nullptr;
    size_t codes_head_stride = 0;
    size_t tuple_chunk_stride = 0;  // chunks per head of the code-pair chunk table (0 = ceil(n/4096))
    float* queries_copy = nullptr;  // tuple select: copy each head's queries here (the attention reads them)
    // score mode
    const float* scores = nullptr;
    size_t scores_stride = 0;
    const uint8_t* excluded = nullptr;
};
// Returns false (after synchronizing) when k exceeds some row's candidates
// (only possible with an exclusion mask).
bool launch_select(pqkv_ctx* ctx, const SelectSource& src, size_t n_rows, size_t n, size_t k,
                   uint32_t* bitmap, int64_t* ids, cudaStream_t stream, int* launches);

// Tuple path (m == 2): per-head pair histograms + pair-level radix select.
void launch_tuple_tables(pqkv_ctx* ctx, const uint16_t* codes, size_t P, size_t codes_head_stride,
                         size_t C, size_t row_begin, size_t row_end, uint32_t* thist, uint16_t* chist,
                         size_t n_chunks, cudaStream_t st);
void launch_select_tuple(pqkv_ctx* ctx, const SelectSource& src, const uint32_t* thist,
                         const uint16_t* chist, size_t rows, size_t n, size_t k, uint32_t* bitmap,
                         int64_t* ids, cudaStream_t st, int* launches);

void launch_attend_rows(pqkv_ctx* ctx, const float* queries, size_t n_heads, size_t g,
                        size_t d_h, const float* keys, const float* values,
                        size_t kv_head_stride, const int64_t* rows, size_t t, int precision,
                        float* out, cudaStream_t stream);

// Fused fast path (d_h == 128, g in {1,2,4}): selection from a bitmap or from
// the code-pair classes (cls, cut) of launch_tuple_select.
bool decode_fast_path(const pqkv_layer& L, size_t g);
// k_pairs > 0: the per-head pair select runs in the attention prologue
// (decode_pairs_fused geometry); cls/cut/bitmap are then unused.
bool decode_pairs_fused(const pqkv_layer& L, size_t g);
// Generic m, b (m * 2^b * 8 <= 16 KB, s_mid <= 16 chunks): the exact top-k
// over per-token ADC keys runs in the attention prologue, one thread-block
// cluster per head (k_keys > 0).
bool decode_keys_fused(const pqkv_layer& L, size_t g);
bool decode_keys_split(const pqkv_layer& L, size_t g);
void launch_decode_attend(pqkv_ctx* ctx, const pqkv_layer& L, const float* queries, size_t g,
                          const uint32_t* bitmap, const uint8_t* cls, const int* cut, float* out,
                          cudaStream_t stream, size_t k_pairs = 0, size_t k_keys = 0, unsigned* ready = nullptr);
// Geometry of the attention launch launch_decode_attend would make (chunk,
// CTAs per head, cluster, staging, window, ring depth, shared memory).
void plan_decode_attend(pqkv_ctx* ctx, const pqkv_layer& L, size_t g, size_t k_pairs, size_t k_keys,
                        bool tuple_cls, pqkv_decode_plan_t* out);
// Pair-level select only (writes cls [rows][C*C], cut [rows][2]).
void launch_tuple_select(pqkv_ctx* ctx, const SelectSource& src, const uint32_t* thist,
                         const uint16_t* chist, size_t rows, size_t n, size_t k, uint8_t* cls, int* cut,
                         uint32_t* tkey, uint32_t* sel_before, cudaStream_t st, unsigned* ready = nullptr);
// Device buffer for decode-level intermediates (never aliases the arena).
void* decode_workspace(pqkv_ctx* ctx, size_t bytes);
void launch_exact(pqkv_ctx* ctx, const float* queries, size_t P, size_t G, size_t d_h,
                  const float* keys, const float* values, size_t kv_head_stride,
                  const int64_t* rows, size_t t, float* out, cudaStream_t st);
void launch_exact_scores(pqkv_ctx* ctx, const float* queries, size_t P, size_t G, size_t d_h,
                         const float* keys, size_t kv_head_stride, const int64_t* rows, size_t t,
                         float* scores, cudaStream_t st);
void launch_bitmap_rows(pqkv_ctx* ctx, const uint32_t* bitmap, size_t P, size_t words,
                        size_t n_init, size_t n_local, size_t total, size_t T, int64_t* rows,
                        cudaStream_t st);

// metrics.cu (experiment metrics on the device)
void launch_summed_scores(pqkv_ctx* ctx, const float* queries, size_t P, size_t g, size_t d_h, const float* keys,
                          size_t kv_head_stride, size_t n, float* scores, cudaStream_t st);
void launch_relative_error(pqkv_ctx* ctx, const float* got, const float* want, size_t rows, size_t n, double* out,
                           cudaStream_t st);
void launch_overlap(pqkv_ctx* ctx, const int64_t* got, size_t k_got, const int64_t* want, size_t k_want, size_t rows,
                    size_t n_ids, double* out, cudaStream_t st);
void launch_iota_rows(pqkv_ctx* ctx, int64_t* rows, size_t P, size_t t, cudaStream_t st);

}  // namespace pqkv_dev
