// pqkv.hpp -- C++ drop-in API of the B200-native PQCache hot paths.
//
// Same namespace, types, signatures, value semantics and exception types as
// the reference library's hot-path API (/root/reference/proj/include/pqkv:
// tensor.hpp:13-46, rng.hpp:11-37, model.hpp:30-36, kmeans.hpp:10-30,
// pq.hpp:16-67, topk.hpp:13-14, attention.hpp:13-32, kv_store.hpp:17-130), so
// a caller recompiles against this header and links libpqkv.so instead.
// Every computing function runs on the GPU through the C ABI (pqkv_c.h); the
// host side only validates arguments and moves the caller's host buffers.
//
// Not provided here (out of the hot-path scope): the cost
// model, simulator/timeline, workload generator, experiments drivers and CLI.
// KvStore's block-cache accounting (fetch_topk hits/misses/bytes, LRU/LFU
// cache, cache_stats, trace) follows kv_store.cpp:93-203, with the
// per-request block counts and ranking computed on the GPU (pqkv_block_rank).
#pragma once

#include <cstddef>
#include <cstdint>
#include <deque>
#include <iosfwd>
#include <map>
#include <random>
#include <span>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <utility>
#include <vector>

#include "pqkv_c.h"

#if defined(__GNUC__)
#define PQKV_CXX_API __attribute__((visibility("default")))
#else
#define PQKV_CXX_API
#endif

namespace pqkv {

// ---- boundary types ---------------------------------------------------------

/// Dense row-major float32 tensor; data holds exactly prod(dims) finite values.
struct PQKV_CXX_API TensorF32 {
    std::vector<std::size_t> dims;
    std::vector<float> data;

    TensorF32() = default;
    TensorF32(std::vector<std::size_t> dims_, std::vector<float> data_);

    std::size_t numel() const;
    std::size_t ndim() const { return dims.size(); }
    const float* row(std::size_t i) const;
    float* row(std::size_t i);
    /// std::invalid_argument on a size mismatch or a non-finite value.
    void validate() const;
};

// ---- .pqt files (tensor.cpp:46-150; the code's header: magic "PQKV", u32
// version, u8 dtype (0 f32, 1 u16), u8 ndim, u64 dims, little-endian payload)

inline constexpr std::uint32_t kTensorFormatVersion = 1;
PQKV_CXX_API void write_tensor(std::ostream& out, const TensorF32& t);
PQKV_CXX_API TensorF32 read_tensor(std::istream& in);
PQKV_CXX_API void write_grid_u16(std::ostream& out, const std::vector<std::size_t>& dims,
                                 const std::vector<std::uint16_t>& data);
PQKV_CXX_API void read_grid_u16(std::istream& in, std::vector<std::size_t>& dims,
                                std::vector<std::uint16_t>& data);
PQKV_CXX_API void save_tensor(const std::string& path, const TensorF32& t);
PQKV_CXX_API TensorF32 load_tensor(const std::string& path);

/// mt19937_64 with explicit draw math (bit-identical streams to the reference).
class PQKV_CXX_API Rng {
public:
    explicit Rng(std::uint64_t seed) : engine_(seed) {}
    std::uint64_t next_u64() { return engine_(); }
    double uniform() { return static_cast<double>(engine_() >> 11) * 0x1.0p-53; }
    double normal();
    std::size_t index(std::size_t n) { return static_cast<std::size_t>(engine_() % n); }
    std::uint64_t fork_seed() { return engine_() ^ 0x9e3779b97f4a7c15ull; }

private:
    std::mt19937_64 engine_;
};

/// Token segments: n_init resident, n_local sliding window, k selected middle.
struct PQKV_CXX_API SegmentConfig {
    std::size_t n_init = 16;
    std::size_t n_local = 64;
    std::size_t k = 0;
    void validate() const;
};

// ---- k-means ------------------------------------------------------------------

struct KmeansResult {
    TensorF32 centroids;                   // [n_clusters, dim]
    std::vector<std::size_t> assignments;  // cluster id per point
    std::vector<double> inertia_trace;     // one entry per iteration
    std::size_t iterations_run = 0;
};

PQKV_CXX_API KmeansResult kmeans_fit(const TensorF32& points, std::size_t n_clusters,
                                     std::size_t max_iter, std::uint64_t seed);
PQKV_CXX_API std::vector<std::size_t> assign_nearest(const TensorF32& points,
                                                     const TensorF32& centroids);

// ---- product quantization ---------------------------------------------------

struct PQKV_CXX_API PqConfig {
    std::size_t m = 2;
    std::size_t b = 6;
    std::size_t d_m = 0;
    std::size_t n_clusters = 64;

    static PqConfig create(std::size_t m, std::size_t b, std::size_t d_h);
    void validate() const;
    std::size_t head_dim() const { return m * d_m; }
};

struct PQKV_CXX_API PqIndex {
    PqConfig cfg;
    TensorF32 centroids;               // [m, 2^b, d_m]
    std::vector<std::uint16_t> codes;  // [s, m] row-major

    std::size_t size() const { return cfg.m ? codes.size() / cfg.m : 0; }
    const float* centroid(std::size_t partition, std::size_t cluster) const;
    const std::uint16_t* code_row(std::size_t token) const;
};

PQKV_CXX_API PqIndex pq_construct(const TensorF32& keys, const PqConfig& cfg,
                                  std::size_t max_iter, std::uint64_t seed);
PQKV_CXX_API std::vector<std::uint16_t> pq_encode_one(std::span<const float> key,
                                                      const PqIndex& index);
PQKV_CXX_API void append_code(PqIndex& index, std::span<const std::uint16_t> code);
PQKV_CXX_API std::vector<float> pq_score(std::span<const float> query, const PqIndex& index);
PQKV_CXX_API std::vector<float> pq_score_gqa(const TensorF32& queries, const PqIndex& index);
PQKV_CXX_API std::vector<float> reconstruct(const PqIndex& index, std::size_t token);
PQKV_CXX_API std::vector<std::size_t> approx_topk(
    std::span<const float> scores, std::size_t k,
    const std::unordered_set<std::size_t>& excluded = {});
PQKV_CXX_API double codes_memory_ratio(const PqConfig& cfg, std::size_t d_h);

/// Index files (pq.cpp:184-222): the centroid tensor, then the [s, m] u16 code grid.
PQKV_CXX_API void write_index(std::ostream& out, const PqIndex& index);
PQKV_CXX_API PqIndex read_index(std::istream& in);
PQKV_CXX_API void save_index(const std::string& path, const PqIndex& index);
PQKV_CXX_API PqIndex load_index(const std::string& path);

PQKV_CXX_API std::vector<std::size_t> top_k_desc(
    std::span<const float> scores, std::size_t k,
    const std::unordered_set<std::size_t>& excluded = {});

// ---- KV store (data path only) -------------------------------------------------

struct KvEntry {
    std::vector<float> key;
    std::vector<float> value;
};

enum class CachePolicy { kLru, kLfu };

struct FetchReport {
    std::vector<KvEntry> entries;  // request order, bit-identical to the offload
    std::size_t hits = 0;
    std::size_t misses = 0;
    std::size_t bytes_from_slow_tier = 0;
};

struct OffloadReport {
    std::size_t init_tokens = 0;
    std::size_t local_tokens = 0;
    std::size_t middle_tokens = 0;
    std::size_t middle_blocks = 0;
    std::size_t bytes_offloaded = 0;
};

struct CacheStats {
    std::size_t hits = 0;
    std::size_t misses = 0;
    std::size_t requests = 0;  // distinct block lookups
    std::size_t occupancy_tokens = 0;
    double hit_rate = 0.0;
};

struct TraceRow {
    std::size_t step = 0;  // per-state fetch ordinal, 1-based
    std::size_t layer = 0;
    std::size_t kv_head = 0;
    std::size_t block_id = 0;
    bool hit = false;
};

/// One (layer, kv_head) slice: init segment, local ring (oldest first) and the
/// middle tokens, with the reference's public members.
struct HeadState {
    struct CachedBlock {
        std::map<std::size_t, KvEntry> snapshot;
        std::size_t freq = 0;
        std::uint64_t last_used = 0;
    };

    std::vector<KvEntry> init_entries;
    std::deque<std::pair<std::size_t, KvEntry>> local;
    std::unordered_map<std::size_t, KvEntry> middle;
    std::map<std::size_t, CachedBlock> cache;

    std::size_t total_tokens = 0;  // next fresh token id
    std::size_t occupancy_tokens = 0;
    std::size_t hits = 0, misses = 0, requests = 0;
    std::size_t fetch_calls = 0;
    std::uint64_t tick = 0;
    bool prefilled = false;
};

class PQKV_CXX_API KvStore {
public:
    KvStore(std::size_t num_layers, std::size_t num_kv_heads, std::size_t block_size,
            std::size_t cache_capacity_tokens, CachePolicy policy);
    OffloadReport offload_prefill(std::size_t layer, std::size_t kv_head, const TensorF32& keys,
                                  const TensorF32& values, const SegmentConfig& seg);
    std::size_t evict_local_append(std::size_t layer, std::size_t kv_head, KvEntry new_entry,
                                   PqIndex& index);
    FetchReport fetch_topk(std::size_t layer, std::size_t kv_head,
                           std::span<const std::size_t> token_ids, std::size_t k_cache);
    CacheStats cache_stats(std::size_t layer, std::size_t kv_head) const;
    const HeadState& state(std::size_t layer, std::size_t kv_head) const;
    std::size_t block_size() const { return block_size_; }
    std::size_t cache_capacity() const { return cache_capacity_; }
    void enable_trace() { trace_enabled_ = true; }
    const std::vector<TraceRow>& trace() const { return trace_; }

private:
    HeadState& state_mut(std::size_t layer, std::size_t kv_head);
    void evict_until_fits(HeadState& st, std::size_t incoming_tokens);
    std::size_t token_bytes() const { return 2 * 2 * head_dim_; }  // fp16 K + V
    std::size_t num_layers_, num_kv_heads_, block_size_, cache_capacity_;
    CachePolicy policy_;
    std::size_t head_dim_ = 0;
    std::vector<HeadState> states_;
    bool trace_enabled_ = false;
    std::vector<TraceRow> trace_;
};

// ---- attention -----------------------------------------------------------------

PQKV_CXX_API std::vector<float> exact_scores(std::span<const float> query, const TensorF32& keys);
PQKV_CXX_API std::vector<std::size_t> exact_topk(
    std::span<const float> query, const TensorF32& keys, std::size_t k,
    const std::unordered_set<std::size_t>& excluded = {});
PQKV_CXX_API std::vector<float> softmax_attention(std::span<const float> query,
                                                  const TensorF32& keys, const TensorF32& values);
PQKV_CXX_API std::vector<float> selective_attention(
    std::span<const float> query, const HeadState& state,
    std::span<const std::size_t> selected_middle_ids);
PQKV_CXX_API TensorF32 gqa_group_attention(const TensorF32& queries, const TensorF32& keys,
                                           const TensorF32& values);

// ---- runtime control -------------------------------------------------------------

/// The CUDA device this thread's API calls run on (default 0).
PQKV_CXX_API void set_device(int device);
/// The process-wide context used by the functions above on this thread.
PQKV_CXX_API pqkv_ctx* default_context();

}  // namespace pqkv
