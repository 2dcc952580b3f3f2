// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI shim over the UNMODIFIED reference library (the sources under
// /root/reference/proj/src, compiled by oracle/Makefile into
// oracle/_ref/libpqkv_ref.so with the namespace renamed pqkv -> pqkv_ref).
// Signatures mirror oracle/pqkv_oracle.h (ref_* instead of orc_*) so the C
// restatement can be pinned against the reference call for call.  It also
// exposes the multi-threaded CPU baseline used by bench.py (--impl reference
// and the cpu_baseline leg): the reference's own functions on a std::thread
// pool over all host cores, one (layer, kv_head) task per thread.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include "pqkv/attention.hpp"
#include "pqkv/kmeans.hpp"
#include "pqkv/kv_store.hpp"
#include "pqkv/pq.hpp"
#include "pqkv/rng.hpp"
#include "pqkv/topk.hpp"
#include "pqkv/workload.hpp"

using namespace pqkv;  // -Dpqkv=pqkv_ref on the command line

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 2;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

TensorF32 grid(const float* p, std::size_t rows, std::size_t cols) {
    return TensorF32({rows, cols}, std::vector<float>(p, p + rows * cols));
}

PqIndex make_index(const float* centroids, std::size_t m, std::size_t C, std::size_t d_m,
                   const std::uint16_t* codes, std::size_t s) {
    PqIndex index;
    std::size_t b = 0;
    for (std::size_t q = 1; q <= 16; ++q)
        if ((std::size_t{1} << q) == C) b = q;
    index.cfg = PqConfig::create(m, b, m * d_m);
    index.centroids = TensorF32({m, C, d_m}, std::vector<float>(centroids, centroids + m * C * d_m));
    index.codes.assign(codes, codes + s * m);
    return index;
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

uint64_t ref_rng_stream(uint64_t seed, uint64_t* out, size_t n, int kind) {
    Rng rng(seed);
    for (size_t i = 0; i < n; ++i) {
        if (kind == 0) out[i] = rng.next_u64();
        else if (kind == 1) { double u = rng.uniform(); std::memcpy(&out[i], &u, 8); }
        else if (kind == 2) { double u = rng.normal(); std::memcpy(&out[i], &u, 8); }
        else out[i] = rng.fork_seed();
    }
    return 0;
}

int ref_gen_workload(size_t s, size_t d_h, size_t h_kv, size_t g, int kind, size_t n_components,
                     double spread, double zipf, uint64_t seed, float* keys, float* values,
                     float* queries) {
    return guard([&] {
        WorkloadSpec spec;
        spec.s = s;
        spec.d_h = d_h;
        spec.h_kv = h_kv;
        spec.g = g;
        spec.kind = kind == 0 ? WorkloadKind::kGaussianMixture : WorkloadKind::kPowerlaw;
        spec.n_components = n_components;
        spec.spread = spread;
        spec.zipf_exponent = zipf;
        spec.seed = seed;
        Workload w = gen_workload(spec);
        std::copy(w.keys.data.begin(), w.keys.data.end(), keys);
        std::copy(w.values.data.begin(), w.values.data.end(), values);
        std::copy(w.queries.data.begin(), w.queries.data.end(), queries);
    });
}

int ref_kmeans_fit(const float* points, size_t n, size_t dim, size_t n_clusters, size_t max_iter,
                   uint64_t seed, float* centroids_out, uint64_t* assign_out,
                   double* inertia_trace, size_t* iterations_run) {
    return guard([&] {
        KmeansResult r = kmeans_fit(grid(points, n, dim), n_clusters, max_iter, seed);
        std::copy(r.centroids.data.begin(), r.centroids.data.end(), centroids_out);
        for (size_t i = 0; i < n; ++i) assign_out[i] = r.assignments[i];
        if (inertia_trace)
            std::copy(r.inertia_trace.begin(), r.inertia_trace.end(), inertia_trace);
        if (iterations_run) *iterations_run = r.iterations_run;
    });
}

int ref_assign_nearest(const float* points, size_t n, size_t dim, const float* centroids,
                       size_t k, uint64_t* assign_out) {
    return guard([&] {
        std::vector<std::size_t> a = assign_nearest(grid(points, n, dim), grid(centroids, k, dim));
        for (size_t i = 0; i < n; ++i) assign_out[i] = a[i];
    });
}

int ref_pq_construct(const float* keys, size_t s, size_t d_h, size_t m, size_t b,
                     size_t max_iter, uint64_t seed, float* centroids_out, uint16_t* codes_out) {
    return guard([&] {
        PqIndex idx = pq_construct(grid(keys, s, d_h), PqConfig::create(m, b, d_h), max_iter, seed);
        std::copy(idx.centroids.data.begin(), idx.centroids.data.end(), centroids_out);
        std::copy(idx.codes.begin(), idx.codes.end(), codes_out);
    });
}

int ref_pq_encode_one(const float* key, const float* centroids, size_t m, size_t C, size_t d_m,
                      uint16_t* code_out) {
    return guard([&] {
        std::uint16_t dummy[16] = {0};
        PqIndex idx = make_index(centroids, m, C, d_m, dummy, 0);
        std::vector<std::uint16_t> c = pq_encode_one({key, m * d_m}, idx);
        std::copy(c.begin(), c.end(), code_out);
    });
}

int ref_pq_score_gqa(const float* queries, size_t g, size_t d_h, const float* centroids,
                     size_t m, size_t C, const uint16_t* codes, size_t s, float* scores_out) {
    return guard([&] {
        PqIndex idx = make_index(centroids, m, C, d_h / m, codes, s);
        std::vector<float> sc = pq_score_gqa(grid(queries, g, d_h), idx);
        std::copy(sc.begin(), sc.end(), scores_out);
    });
}

int ref_top_k_desc(const float* scores, size_t n, size_t k, const uint8_t* excluded,
                   uint64_t* ids_out) {
    return guard([&] {
        std::unordered_set<std::size_t> ex;
        if (excluded)
            for (size_t i = 0; i < n; ++i)
                if (excluded[i]) ex.insert(i);
        std::vector<std::size_t> ids = top_k_desc({scores, n}, k, ex);
        for (size_t i = 0; i < ids.size(); ++i) ids_out[i] = ids[i];
    });
}

int ref_exact_scores(const float* query, const float* keys, size_t t, size_t d_h,
                     float* scores_out) {
    return guard([&] {
        std::vector<float> sc = exact_scores({query, d_h}, grid(keys, t, d_h));
        std::copy(sc.begin(), sc.end(), scores_out);
    });
}

int ref_softmax_rows(const float* query, const float* keys, const float* values, size_t d_h,
                     const uint64_t* rows, size_t t, float* out) {
    return guard([&] {
        std::vector<float> k(t * d_h), v(t * d_h);
        for (size_t i = 0; i < t; ++i) {
            size_t r = rows ? rows[i] : i;
            std::copy(keys + r * d_h, keys + (r + 1) * d_h, k.begin() + i * d_h);
            std::copy(values + r * d_h, values + (r + 1) * d_h, v.begin() + i * d_h);
        }
        std::vector<float> o = softmax_attention({query, d_h}, TensorF32({t, d_h}, std::move(k)),
                                                 TensorF32({t, d_h}, std::move(v)));
        std::copy(o.begin(), o.end(), out);
    });
}

// The reference's selective_attention reads a HeadState built by
// KvStore::offload_prefill; build one from the flat [total][d_h] rows.
int ref_selective_attention(const float* query, const float* keys, const float* values,
                            size_t d_h, size_t total, size_t n_init, size_t n_local,
                            const uint64_t* middle_ids, size_t n_ids, float* out) {
    return guard([&] {
        KvStore store(1, 1, 128, 4096, CachePolicy::kLru);
        SegmentConfig seg{n_init, n_local, 0};
        store.offload_prefill(0, 0, grid(keys, total, d_h), grid(values, total, d_h), seg);
        std::vector<std::size_t> ids(middle_ids, middle_ids + n_ids);
        std::vector<float> o = selective_attention({query, d_h}, store.state(0, 0), ids);
        std::copy(o.begin(), o.end(), out);
    });
}

// ---------------------------------------------------------------------------
// CPU baseline: the reference's decode retrieval for a batch of kv heads on a
// thread pool.  Per head (experiments.cpp:218-260): pq_score_gqa ->
// approx_topk -> middle row -> token id -> selective_attention per query row.
// Inputs are flat per head: keys/values [P][total][d_h], queries [P][g][d_h],
// centroids [P][m][C][d_m], codes [P][s_mid][m].  Returns wall seconds.
// ---------------------------------------------------------------------------
double ref_bench_decode_steps(size_t P, size_t total, size_t d_h, size_t g, size_t n_init,
                              size_t n_local, size_t m, size_t C, size_t k, const float* keys,
                              const float* values, const float* queries, size_t n_steps,
                              const float* centroids, const uint16_t* codes, float* out,
                              int n_threads, double* step_secs) {
    size_t s_mid = total - n_init - n_local, d_m = d_h / m;
    // HeadStates are built once, outside the timed steps (the reference keeps
    // them resident across decode steps, kv_store.cpp:32-74).  queries holds
    // n_steps x [P][g][d_h]; step t uses slice t.
    std::vector<KvStore> stores;
    std::vector<PqIndex> idx;
    stores.reserve(P);
    for (size_t p = 0; p < P; ++p) {
        stores.emplace_back(1, 1, 128, 4096, CachePolicy::kLru);
        stores.back().offload_prefill(0, 0, grid(keys + p * total * d_h, total, d_h),
                                      grid(values + p * total * d_h, total, d_h),
                                      SegmentConfig{n_init, n_local, k});
        idx.push_back(make_index(centroids + p * m * C * d_m, m, C, d_m, codes + p * s_mid * m, s_mid));
    }
    int nt = n_threads > 0 ? n_threads : (int)std::max(1u, std::thread::hardware_concurrency());
    double total_secs = 0.0;
    for (size_t step = 0; step < n_steps; ++step) {
        const float* qs = queries + step * P * g * d_h;
        std::atomic<size_t> next{0};
        auto worker = [&] {
            for (size_t p; (p = next.fetch_add(1)) < P;) {
                TensorF32 q = grid(qs + p * g * d_h, g, d_h);
                std::vector<float> scores = pq_score_gqa(q, idx[p]);
                std::vector<std::size_t> sel = approx_topk(scores, k);
                for (auto& r : sel) r += n_init;
                for (size_t r = 0; r < g; ++r) {
                    std::vector<float> o = selective_attention({q.row(r), d_h}, stores[p].state(0, 0), sel);
                    std::copy(o.begin(), o.end(), out + (p * g + r) * d_h);
                }
            }
        };
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int t = 0; t < nt; ++t) pool.emplace_back(worker);
        for (auto& t : pool) t.join();
        double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (step_secs) step_secs[step] = secs;
        total_secs += secs;
    }
    return total_secs;
}

double ref_bench_decode(size_t P, size_t total, size_t d_h, size_t g, size_t n_init,
                        size_t n_local, size_t m, size_t C, size_t k, const float* keys,
                        const float* values, const float* queries, const float* centroids,
                        const uint16_t* codes, float* out, int n_threads) {
    return ref_bench_decode_steps(P, total, d_h, g, n_init, n_local, m, C, k, keys, values, queries, 1,
                                  centroids, codes, out, n_threads, nullptr);
}

// CPU baseline for the prefill build: pq_construct per head on a thread pool.
double ref_bench_build(size_t P, size_t s, size_t d_h, size_t m, size_t b, size_t max_iter,
                       const float* keys, const uint64_t* seeds, float* centroids_out,
                       uint16_t* codes_out, int n_threads) {
    size_t C = size_t{1} << b, d_m = d_h / m;
    std::atomic<size_t> next{0};
    auto worker = [&] {
        for (size_t p; (p = next.fetch_add(1)) < P;) {
            PqIndex ix = pq_construct(grid(keys + p * s * d_h, s, d_h), PqConfig::create(m, b, d_h),
                                      max_iter, seeds[p]);
            std::copy(ix.centroids.data.begin(), ix.centroids.data.end(), centroids_out + p * m * C * d_m);
            std::copy(ix.codes.begin(), ix.codes.end(), codes_out + p * s * m);
        }
    };
    int nt = n_threads > 0 ? n_threads : (int)std::max(1u, std::thread::hardware_concurrency());
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t) pool.emplace_back(worker);
    for (auto& t : pool) t.join();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// Block-cache replay (kv_store.cpp:93-203): offload one (s, d_h) head, then
// for request r: if append_before[r], evict_local_append(fresh row r) against
// a pq_construct index (m = 2, b = 3) of the middle keys; then fetch_topk of
// ids[offs[r] .. offs[r+1]) with k_cache.  out[3r..3r+2] = hits, misses,
// bytes_from_slow_tier; out[3n..3n+3] = cache_stats hits, misses, requests,
// occupancy; cached block ids -> cache_out (up to cache_cap), count -> *n_cached.
int ref_fetch_replay(size_t s, size_t d_h, const float* keys, const float* values, size_t n_init,
                     size_t n_local, size_t block, size_t capacity, int lfu, size_t n_req,
                     const uint64_t* offs, const uint64_t* ids, const uint8_t* append_before,
                     const float* fresh, size_t k_cache, uint64_t* out, uint64_t* cache_out,
                     size_t cache_cap, size_t* n_cached) {
    return guard([&] {
        KvStore store(1, 1, block, capacity, lfu ? CachePolicy::kLfu : CachePolicy::kLru);
        store.offload_prefill(0, 0, grid(keys, s, d_h), grid(values, s, d_h), SegmentConfig{n_init, n_local, 0});
        std::size_t s_mid = s - n_init - n_local;
        PqIndex index = pq_construct(grid(keys + n_init * d_h, s_mid, d_h), PqConfig::create(2, 3, d_h), 4, 9);
        for (size_t r = 0; r < n_req; ++r) {
            if (append_before[r]) {
                KvEntry e;
                e.key.assign(fresh + r * 2 * d_h, fresh + r * 2 * d_h + d_h);
                e.value.assign(fresh + r * 2 * d_h + d_h, fresh + (r + 1) * 2 * d_h);
                store.evict_local_append(0, 0, std::move(e), index);
            }
            std::vector<std::size_t> req(ids + offs[r], ids + offs[r + 1]);
            FetchReport rep = store.fetch_topk(0, 0, req, k_cache);
            out[3 * r] = rep.hits;
            out[3 * r + 1] = rep.misses;
            out[3 * r + 2] = rep.bytes_from_slow_tier;
        }
        CacheStats cs = store.cache_stats(0, 0);
        out[3 * n_req] = cs.hits;
        out[3 * n_req + 1] = cs.misses;
        out[3 * n_req + 2] = cs.requests;
        out[3 * n_req + 3] = cs.occupancy_tokens;
        size_t n = 0;
        for (const auto& kv : store.state(0, 0).cache)
            if (n < cache_cap) cache_out[n++] = kv.first;
        *n_cached = store.state(0, 0).cache.size();
    });
}

// .pqt round trips through the reference's own writers / readers
// (tensor.cpp:110-150, pq.cpp:184-222).
int ref_save_index(const char* path, const float* centroids, size_t m, size_t C, size_t d_m,
                   const uint16_t* codes, size_t s) {
    return guard([&] { save_index(path, make_index(centroids, m, C, d_m, codes, s)); });
}

int ref_load_index(const char* path, size_t* m, size_t* C, size_t* d_m, size_t* s, float* centroids,
                   uint16_t* codes, size_t cen_cap, size_t code_cap) {
    return guard([&] {
        PqIndex ix = load_index(path);
        *m = ix.cfg.m;
        *C = ix.cfg.n_clusters;
        *d_m = ix.cfg.d_m;
        *s = ix.size();
        if (centroids && ix.centroids.data.size() <= cen_cap)
            std::copy(ix.centroids.data.begin(), ix.centroids.data.end(), centroids);
        if (codes && ix.codes.size() <= code_cap) std::copy(ix.codes.begin(), ix.codes.end(), codes);
    });
}

int ref_save_tensor(const char* path, const float* data, const size_t* dims, size_t ndim) {
    return guard([&] {
        std::vector<std::size_t> d(dims, dims + ndim);
        std::size_t n = 1;
        for (std::size_t x : d) n *= x;
        save_tensor(path, TensorF32(d, std::vector<float>(data, data + n)));
    });
}

}  // extern "C"
