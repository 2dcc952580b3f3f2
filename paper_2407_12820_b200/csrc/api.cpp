// api.cpp -- the C++ drop-in API (include/pqkv/pqkv.hpp) over the C ABI.
//
// Argument validation mirrors the reference's checks, order and exception
// types (tensor.cpp:86-98, kmeans.cpp:160-164, pq.cpp:13-177, topk.cpp:10-15,
// attention.cpp:11-104, kv_store.cpp:10-191); all arithmetic is delegated to
// the GPU through pqkv_c.h.  This layer owns no CUDA code: device buffers are
// obtained through pqkv_device_alloc / pqkv_copy.
#include "pqkv/pqkv.hpp"

#include <algorithm>
#include <bit>
#include <cstring>
#include <fstream>
#include <istream>
#include <ostream>
#include <cmath>
#include <limits>
#include <map>
#include <numeric>
#include <set>
#include <stdexcept>
#include <string>

namespace pqkv {

namespace {

[[noreturn]] void rethrow(int rc, const char* what) {
    std::string msg = what && *what ? what : "pqkv: error";
    switch (rc) {
        case PQKV_EINVAL: throw std::invalid_argument(msg);
        case PQKV_ERANGE: throw std::out_of_range(msg);
        case PQKV_ESTATE: throw std::logic_error(msg);
        default: throw std::runtime_error(msg);
    }
}

void check(int rc) {
    if (rc != PQKV_OK) rethrow(rc, pqkv_last_error());
}

thread_local int g_device = 0;
thread_local pqkv_ctx* g_ctx[64] = {};

// RAII device buffer through the C ABI.
template <typename T>
class Dev {
public:
    explicit Dev(std::size_t count) : n_(count) {
        void* p = nullptr;
        check(pqkv_device_alloc(default_context(), std::max<std::size_t>(1, n_) * sizeof(T), &p));
        p_ = static_cast<T*>(p);
    }
    Dev(const T* host, std::size_t count) : Dev(count) { upload(host, count); }
    ~Dev() { pqkv_device_free(default_context(), p_); }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    void upload(const T* host, std::size_t count) {
        if (count) check(pqkv_copy(default_context(), p_, host, count * sizeof(T), 0));
    }
    void download(T* host, std::size_t count) const {
        if (count) check(pqkv_copy(default_context(), host, p_, count * sizeof(T), 1));
    }
    std::vector<T> to_host() const {
        std::vector<T> v(n_);
        download(v.data(), n_);
        return v;
    }
    T* get() const { return p_; }

private:
    T* p_ = nullptr;
    std::size_t n_;
};

std::size_t checked_numel(const std::vector<std::size_t>& dims) {
    std::size_t n = 1;
    for (std::size_t d : dims) {
        if (d == 0) throw std::invalid_argument("tensor: zero-sized dimension");
        if (d > std::numeric_limits<std::size_t>::max() / n)
            throw std::invalid_argument("tensor: dimension product overflows");
        n *= d;
    }
    return n;
}

// Attention over explicit host rows (rows already in the reference's order).
std::vector<float> attend_host(const float* queries, std::size_t g, std::size_t d_h,
                               const std::vector<float>& keys, const std::vector<float>& values,
                               std::size_t t) {
    Dev<float> dq(queries, g * d_h), dk(keys.data(), t * d_h), dv(values.data(), t * d_h);
    std::vector<int64_t> rows(t);
    std::iota(rows.begin(), rows.end(), 0);
    Dev<int64_t> dr(rows.data(), t);
    Dev<float> dout(g * d_h);
    check(pqkv_attend_rows(default_context(), dq.get(), 1, g, d_h, dk.get(), dv.get(), t * d_h,
                           dr.get(), t, PQKV_PREC_F64, dout.get(), nullptr));
    return dout.to_host();
}

}  // namespace

// ---- runtime -----------------------------------------------------------------

void set_device(int device) {
    if (device < 0 || device >= 64) throw std::invalid_argument("pqkv: bad device");
    g_device = device;
}

pqkv_ctx* default_context() {
    pqkv_ctx*& c = g_ctx[g_device];
    if (!c) check(pqkv_ctx_create(g_device, &c));
    return c;
}

// ---- TensorF32 (tensor.hpp:13-29) -----------------------------------------------

TensorF32::TensorF32(std::vector<std::size_t> dims_, std::vector<float> data_)
    : dims(std::move(dims_)), data(std::move(data_)) {
    validate();
}

std::size_t TensorF32::numel() const { return checked_numel(dims); }

const float* TensorF32::row(std::size_t i) const {
    if (dims.size() != 2) throw std::invalid_argument("tensor: row() needs a 2-d tensor");
    if (i >= dims[0]) throw std::out_of_range("tensor: row index out of range");
    return data.data() + i * dims[1];
}

float* TensorF32::row(std::size_t i) {
    return const_cast<float*>(static_cast<const TensorF32*>(this)->row(i));
}

void TensorF32::validate() const {
    if (checked_numel(dims) != data.size())
        throw std::invalid_argument("tensor: data size does not match product of dims");
    for (float v : data)
        if (!std::isfinite(v)) throw std::invalid_argument("tensor: non-finite value");
}

double Rng::normal() {
    double u1 = uniform(), u2 = uniform();
    while (u1 == 0.0) u1 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
}

void SegmentConfig::validate() const {
    if (n_local < 1) throw std::invalid_argument("segments: n_local must be >= 1");
}

// ---- k-means (kmeans.hpp:24-30) ----------------------------------------------------

KmeansResult kmeans_fit(const TensorF32& points, std::size_t n_clusters, std::size_t max_iter,
                        std::uint64_t seed) {
    points.validate();
    if (points.ndim() != 2) throw std::invalid_argument("kmeans: points must be 2-d");
    if (n_clusters < 1) throw std::invalid_argument("kmeans: n_clusters must be >= 1");
    if (max_iter < 1) throw std::invalid_argument("kmeans: max_iter must be >= 1");
    const std::size_t n = points.dims[0], dim = points.dims[1];
    Dev<float> dp(points.data.data(), n * dim);
    Dev<float> dc(n_clusters * dim);
    Dev<uint32_t> da(n), di(1);
    Dev<double> dinert(max_iter);
    check(pqkv_kmeans_fit(default_context(), dp.get(), 1, n * dim, dim, n, dim, n_clusters, max_iter,
                          &seed, dc.get(), da.get(), di.get(), dinert.get(), nullptr));
    KmeansResult res;
    res.centroids = TensorF32({n_clusters, dim}, dc.to_host());
    std::vector<uint32_t> a = da.to_host();
    res.assignments.assign(a.begin(), a.end());
    res.iterations_run = di.to_host()[0];
    std::vector<double> tr = dinert.to_host();
    res.inertia_trace.assign(tr.begin(), tr.begin() + res.iterations_run);
    return res;
}

std::vector<std::size_t> assign_nearest(const TensorF32& points, const TensorF32& centroids) {
    if (points.ndim() != 2 || centroids.ndim() != 2)
        throw std::invalid_argument("assign_nearest: points and centroids must be 2-d");
    if (points.dims[1] != centroids.dims[1])
        throw std::invalid_argument("assign_nearest: dimension mismatch");
    const std::size_t n = points.dims[0], dim = points.dims[1], k = centroids.dims[0];
    Dev<float> dp(points.data.data(), n * dim), dc(centroids.data.data(), k * dim);
    Dev<uint32_t> da(n);
    check(pqkv_assign_nearest(default_context(), dp.get(), n, dim, dc.get(), k, da.get(), nullptr));
    std::vector<uint32_t> a = da.to_host();
    return std::vector<std::size_t>(a.begin(), a.end());
}

// ---- PQ (pq.hpp:16-67) ---------------------------------------------------------------

PqConfig PqConfig::create(std::size_t m, std::size_t b, std::size_t d_h) {
    std::size_t d_m = 0, c = 0;
    check(pqkv_pq_config(m, b, d_h, &d_m, &c));
    PqConfig cfg;
    cfg.m = m;
    cfg.b = b;
    cfg.d_m = d_m;
    cfg.n_clusters = c;
    return cfg;
}

void PqConfig::validate() const {
    if (m < 1 || d_m < 1) throw std::invalid_argument("pq: m and d_m must be >= 1");
    if (b < 1 || b > 16) throw std::invalid_argument("pq: b must be in [1, 16]");
    if (n_clusters != (std::size_t{1} << b))
        throw std::invalid_argument("pq: n_clusters must equal 2^b");
}

const float* PqIndex::centroid(std::size_t partition, std::size_t cluster) const {
    return centroids.data.data() + (partition * cfg.n_clusters + cluster) * cfg.d_m;
}

const std::uint16_t* PqIndex::code_row(std::size_t token) const {
    if (token >= size()) throw std::out_of_range("pq: token id out of range");
    return codes.data() + token * cfg.m;
}

PqIndex pq_construct(const TensorF32& keys, const PqConfig& cfg, std::size_t max_iter,
                     std::uint64_t seed) {
    cfg.validate();
    keys.validate();
    if (keys.ndim() != 2) throw std::invalid_argument("pq: keys must be 2-d");
    if (keys.dims[1] != cfg.head_dim()) throw std::invalid_argument("pq: key dim must equal m * d_m");
    const std::size_t s = keys.dims[0], d_h = keys.dims[1];
    if (s < 1) throw std::invalid_argument("pq: need at least one key");
    if (max_iter < 1) throw std::invalid_argument("kmeans: max_iter must be >= 1");
    Dev<float> dk(keys.data.data(), s * d_h);
    Dev<float> dc(cfg.m * cfg.n_clusters * cfg.d_m);
    Dev<uint16_t> dcodes(s * cfg.m);
    check(pqkv_pq_build(default_context(), dk.get(), 1, s * d_h, s, d_h, cfg.m, cfg.b, max_iter, &seed,
                        dc.get(), dcodes.get(), s * cfg.m, nullptr));
    PqIndex index;
    index.cfg = cfg;
    index.centroids = TensorF32({cfg.m, cfg.n_clusters, cfg.d_m}, dc.to_host());
    index.codes = dcodes.to_host();
    return index;
}

std::vector<std::uint16_t> pq_encode_one(std::span<const float> key, const PqIndex& index) {
    const PqConfig& cfg = index.cfg;
    if (key.size() != cfg.head_dim()) throw std::invalid_argument("pq: key dim must equal m * d_m");
    Dev<float> dk(key.data(), key.size());
    Dev<float> dc(index.centroids.data.data(), index.centroids.data.size());
    Dev<uint16_t> dcode(cfg.m);
    check(pqkv_pq_encode(default_context(), dk.get(), 1, key.size(), cfg.head_dim(), cfg.m, cfg.b,
                         dc.get(), dcode.get(), cfg.m, 0, nullptr));
    return dcode.to_host();
}

void append_code(PqIndex& index, std::span<const std::uint16_t> code) {
    if (code.size() != index.cfg.m) throw std::invalid_argument("pq: code must have m entries");
    for (std::uint16_t c : code)
        if (c >= index.cfg.n_clusters) throw std::invalid_argument("pq: code entry out of range");
    index.codes.insert(index.codes.end(), code.begin(), code.end());
}

static std::vector<float> score_rows(const float* q, std::size_t g, const PqIndex& index) {
    const PqConfig& cfg = index.cfg;
    const std::size_t s = index.size(), d_h = cfg.head_dim();
    std::vector<float> out(s);
    if (s == 0) return out;
    Dev<float> dq(q, g * d_h);
    Dev<float> dc(index.centroids.data.data(), index.centroids.data.size());
    Dev<uint16_t> dcodes(index.codes.data(), index.codes.size());
    Dev<float> ds(s);
    check(pqkv_pq_score(default_context(), dq.get(), 1, g, d_h, cfg.m, cfg.b, dc.get(), dcodes.get(),
                        s * cfg.m, s, ds.get(), s, nullptr));
    ds.download(out.data(), s);
    return out;
}

std::vector<float> pq_score(std::span<const float> query, const PqIndex& index) {
    if (query.size() != index.cfg.head_dim())
        throw std::invalid_argument("pq: query dim must equal m * d_m");
    return score_rows(query.data(), 1, index);
}

std::vector<float> pq_score_gqa(const TensorF32& queries, const PqIndex& index) {
    if (queries.ndim() != 2 || queries.dims[0] < 1)
        throw std::invalid_argument("pq: queries must be a non-empty 2-d grid");
    if (queries.dims[1] != index.cfg.head_dim())
        throw std::invalid_argument("pq: query dim must equal m * d_m");
    return score_rows(queries.data.data(), queries.dims[0], index);
}

std::vector<float> reconstruct(const PqIndex& index, std::size_t token) {
    const PqConfig& cfg = index.cfg;
    const std::uint16_t* code = index.code_row(token);
    std::vector<float> out(cfg.head_dim());
    for (std::size_t j = 0; j < cfg.m; ++j) {
        const float* cen = index.centroid(j, code[j]);
        std::copy(cen, cen + cfg.d_m, out.begin() + j * cfg.d_m);
    }
    return out;
}

std::vector<std::size_t> top_k_desc(std::span<const float> scores, std::size_t k,
                                    const std::unordered_set<std::size_t>& excluded) {
    const std::size_t n = scores.size();
    std::size_t n_ex = 0;
    for (std::size_t e : excluded) n_ex += e < n;
    if (k > n - n_ex) throw std::invalid_argument("top_k: k too large for the candidate set");
    if (k == 0) return {};
    Dev<float> ds(scores.data(), n);
    std::vector<uint8_t> mask;
    if (n_ex) {
        mask.assign(n, 0);
        for (std::size_t e : excluded)
            if (e < n) mask[e] = 1;
    }
    Dev<uint8_t> dm(mask.empty() ? nullptr : mask.data(), mask.size());
    Dev<int64_t> dids(k);
    check(pqkv_topk(default_context(), ds.get(), 1, n, n, k, mask.empty() ? nullptr : dm.get(),
                    dids.get(), nullptr));
    std::vector<int64_t> ids = dids.to_host();
    return std::vector<std::size_t>(ids.begin(), ids.end());
}

std::vector<std::size_t> approx_topk(std::span<const float> scores, std::size_t k,
                                     const std::unordered_set<std::size_t>& excluded) {
    return top_k_desc(scores, k, excluded);
}

double codes_memory_ratio(const PqConfig& cfg, std::size_t d_h) {
    double r = 0.0;
    check(pqkv_codes_memory_ratio(cfg.m, cfg.b, d_h, &r));
    return r;
}

// ---- attention (attention.hpp:13-32) ---------------------------------------------------

std::vector<float> exact_scores(std::span<const float> query, const TensorF32& keys) {
    if (keys.ndim() != 2) throw std::invalid_argument("attention: keys must be 2-d");
    if (keys.dims[1] != query.size())
        throw std::invalid_argument("attention: query dim must match key dim");
    const std::size_t t = keys.dims[0], d_h = keys.dims[1];
    Dev<float> dq(query.data(), d_h), dk(keys.data.data(), t * d_h);
    std::vector<int64_t> rows(t);
    std::iota(rows.begin(), rows.end(), 0);
    Dev<int64_t> dr(rows.data(), t);
    Dev<float> ds(t);
    check(pqkv_exact_scores(default_context(), dq.get(), 1, 1, d_h, dk.get(), t * d_h, dr.get(), t,
                            ds.get(), nullptr));
    return ds.to_host();
}

std::vector<std::size_t> exact_topk(std::span<const float> query, const TensorF32& keys,
                                    std::size_t k,
                                    const std::unordered_set<std::size_t>& excluded) {
    std::vector<float> scores = exact_scores(query, keys);
    return top_k_desc(scores, k, excluded);
}

std::vector<float> softmax_attention(std::span<const float> query, const TensorF32& keys,
                                     const TensorF32& values) {
    if (values.ndim() != 2 || values.dims != keys.dims)
        throw std::invalid_argument("attention: values must match key dims");
    if (keys.dims[0] < 1) throw std::invalid_argument("attention: need at least one token");
    if (keys.ndim() != 2) throw std::invalid_argument("attention: keys must be 2-d");
    if (keys.dims[1] != query.size())
        throw std::invalid_argument("attention: query dim must match key dim");
    return attend_host(query.data(), 1, keys.dims[1], keys.data, values.data, keys.dims[0]);
}

std::vector<float> selective_attention(std::span<const float> query, const HeadState& state,
                                       std::span<const std::size_t> selected_middle_ids) {
    std::vector<std::size_t> ids(selected_middle_ids.begin(), selected_middle_ids.end());
    std::sort(ids.begin(), ids.end());
    if (std::adjacent_find(ids.begin(), ids.end()) != ids.end())
        throw std::invalid_argument("attention: duplicate middle token id");
    const std::size_t d_h = query.size();
    const std::size_t t = state.init_entries.size() + ids.size() + state.local.size();
    std::vector<float> keys(t * d_h), values(t * d_h);
    std::size_t row = 0;
    auto put = [&](const KvEntry& e) {
        if (e.key.size() != d_h) throw std::invalid_argument("attention: entry dim mismatch");
        std::copy(e.key.begin(), e.key.end(), keys.begin() + row * d_h);
        std::copy(e.value.begin(), e.value.end(), values.begin() + row * d_h);
        ++row;
    };
    for (const KvEntry& e : state.init_entries) put(e);
    for (std::size_t id : ids) {
        auto it = state.middle.find(id);
        if (it == state.middle.end())
            throw std::out_of_range("attention: token " + std::to_string(id) + " is not a middle token");
        put(it->second);
    }
    for (const auto& [id, e] : state.local) put(e);
    if (t < 1 || d_h < 1) throw std::invalid_argument("tensor: zero-sized dimension");
    return attend_host(query.data(), 1, d_h, keys, values, t);
}

TensorF32 gqa_group_attention(const TensorF32& queries, const TensorF32& keys,
                              const TensorF32& values) {
    if (queries.ndim() != 2 || queries.dims[0] < 1)
        throw std::invalid_argument("attention: queries must be a non-empty 2-d grid");
    if (values.ndim() != 2 || values.dims != keys.dims)
        throw std::invalid_argument("attention: values must match key dims");
    if (keys.dims[0] < 1) throw std::invalid_argument("attention: need at least one token");
    if (keys.ndim() != 2) throw std::invalid_argument("attention: keys must be 2-d");
    const std::size_t g = queries.dims[0], d_h = queries.dims[1];
    if (keys.dims[1] != d_h) throw std::invalid_argument("attention: query dim must match key dim");
    std::vector<float> o = attend_host(queries.data.data(), g, d_h, keys.data, values.data, keys.dims[0]);
    return TensorF32({g, d_h}, std::move(o));
}

// ---- KvStore data path (kv_store.cpp:10-153) ------------------------------------------

KvStore::KvStore(std::size_t num_layers, std::size_t num_kv_heads, std::size_t block_size,
                 std::size_t cache_capacity_tokens, CachePolicy policy)
    : num_layers_(num_layers), num_kv_heads_(num_kv_heads), block_size_(block_size),
      cache_capacity_(cache_capacity_tokens), policy_(policy) {
    if (num_layers < 1 || num_kv_heads < 1)
        throw std::invalid_argument("kv_store: need at least one layer and kv head");
    if (block_size < 1) throw std::invalid_argument("kv_store: block_size must be >= 1");
    states_.resize(num_layers * num_kv_heads);
}

HeadState& KvStore::state_mut(std::size_t layer, std::size_t kv_head) {
    if (layer >= num_layers_ || kv_head >= num_kv_heads_)
        throw std::out_of_range("kv_store: layer or kv_head out of range");
    return states_[layer * num_kv_heads_ + kv_head];
}

const HeadState& KvStore::state(std::size_t layer, std::size_t kv_head) const {
    if (layer >= num_layers_ || kv_head >= num_kv_heads_)
        throw std::out_of_range("kv_store: layer or kv_head out of range");
    return states_[layer * num_kv_heads_ + kv_head];
}

OffloadReport KvStore::offload_prefill(std::size_t layer, std::size_t kv_head,
                                       const TensorF32& keys, const TensorF32& values,
                                       const SegmentConfig& seg) {
    HeadState& st = state_mut(layer, kv_head);
    if (st.prefilled) throw std::logic_error("kv_store: state already prefilled");
    seg.validate();
    keys.validate();
    values.validate();
    if (keys.ndim() != 2 || values.ndim() != 2 || keys.dims != values.dims)
        throw std::invalid_argument("kv_store: keys and values must be 2-d with equal dims");
    const std::size_t s = keys.dims[0], d_h = keys.dims[1];
    if (seg.n_init + seg.n_local > s)
        throw std::invalid_argument("kv_store: segment overflow, n_init + n_local > s");
    if (head_dim_ == 0) head_dim_ = d_h;
    if (d_h != head_dim_) throw std::invalid_argument("kv_store: head_dim mismatch");
    auto entry_at = [&](std::size_t i) {
        KvEntry e;
        e.key.assign(keys.row(i), keys.row(i) + d_h);
        e.value.assign(values.row(i), values.row(i) + d_h);
        return e;
    };
    OffloadReport rep;
    std::set<std::size_t> blocks;
    for (std::size_t i = 0; i < s; ++i) {
        if (i < seg.n_init) {
            st.init_entries.push_back(entry_at(i));
            ++rep.init_tokens;
        } else if (i >= s - seg.n_local) {
            st.local.emplace_back(i, entry_at(i));
            ++rep.local_tokens;
        } else {
            st.middle.emplace(i, entry_at(i));
            blocks.insert(i / block_size_);
            ++rep.middle_tokens;
        }
    }
    st.total_tokens = s;
    st.prefilled = true;
    rep.middle_blocks = blocks.size();
    rep.bytes_offloaded = rep.middle_tokens * 2 * 2 * head_dim_;
    return rep;
}

std::size_t KvStore::evict_local_append(std::size_t layer, std::size_t kv_head, KvEntry new_entry,
                                        PqIndex& index) {
    HeadState& st = state_mut(layer, kv_head);
    if (st.local.empty()) throw std::logic_error("kv_store: local segment is empty");
    if (new_entry.key.size() != head_dim_ || new_entry.value.size() != head_dim_)
        throw std::invalid_argument("kv_store: entry dim mismatch");
    auto [evicted_id, entry] = std::move(st.local.front());
    st.local.pop_front();
    append_code(index, pq_encode_one(entry.key, index));
    st.middle.emplace(evicted_id, std::move(entry));
    st.local.emplace_back(st.total_tokens++, std::move(new_entry));
    return evicted_id;
}

// LRU evicts the stalest block; LFU the least frequent, ties by least recent
// use, then the lower block id (kv_store.cpp:93-113).
void KvStore::evict_until_fits(HeadState& st, std::size_t incoming_tokens) {
    while (!st.cache.empty() && st.occupancy_tokens + incoming_tokens > cache_capacity_) {
        auto victim = st.cache.begin();
        for (auto it = std::next(st.cache.begin()); it != st.cache.end(); ++it) {
            bool worse;
            if (policy_ == CachePolicy::kLru) {
                worse = it->second.last_used < victim->second.last_used;
            } else {
                worse = it->second.freq < victim->second.freq ||
                        (it->second.freq == victim->second.freq && it->second.last_used < victim->second.last_used);
            }
            if (worse) victim = it;
        }
        st.occupancy_tokens -= victim->second.snapshot.size();
        st.cache.erase(victim);
    }
}

// fetch_topk (kv_store.cpp:115-191).  The per-request work -- distinct
// tokens, distinct tokens per block and the top-k_cache block ranking -- runs
// on the GPU (pqkv_block_rank); the lookups and the LRU/LFU cache refresh are
// the reference's sequential state machine.
FetchReport KvStore::fetch_topk(std::size_t layer, std::size_t kv_head, std::span<const std::size_t> token_ids,
                                std::size_t k_cache) {
    HeadState& st = state_mut(layer, kv_head);
    for (std::size_t id : token_ids)
        if (!st.middle.contains(id))
            throw std::out_of_range("kv_store: token " + std::to_string(id) + " is not a middle token");
    ++st.fetch_calls;

    const std::size_t n_tokens = st.total_tokens, bs = block_size_;
    const std::size_t n_blocks = std::max<std::size_t>(1, (n_tokens + bs - 1) / bs);
    const std::size_t words = (n_tokens + 31) / 32;
    const std::size_t k_rank = std::min(k_cache, n_blocks);
    std::vector<std::int64_t> ids(token_ids.begin(), token_ids.end());
    std::vector<std::uint32_t> bits(words), counts(n_blocks);
    std::vector<std::int64_t> ranked(k_rank);
    {
        Dev<std::int64_t> d_ids(ids.data(), ids.size());
        Dev<std::uint32_t> d_bits(words), d_counts(n_blocks);
        Dev<std::int64_t> d_ranked(k_rank);
        check(pqkv_block_rank(default_context(), d_ids.get(), 1, ids.size(), ids.size(), n_tokens, bs, k_rank,
                              d_bits.get(), d_counts.get(), d_ranked.get(), nullptr, nullptr));
        d_bits.download(bits.data(), words);
        d_counts.download(counts.data(), n_blocks);
        d_ranked.download(ranked.data(), k_rank);
    }

    FetchReport rep;
    std::size_t touched = 0;
    for (std::size_t b = 0; b < n_blocks; ++b) {  // distinct blocks, ascending id (a std::map in the reference)
        if (!counts[b]) continue;
        ++touched;
        auto it = st.cache.find(b);
        const bool hit = it != st.cache.end();
        if (hit) {
            ++rep.hits;
            it->second.freq += 1;
            it->second.last_used = ++st.tick;
            const std::size_t hi = std::min(n_tokens, (b + 1) * bs);
            for (std::size_t id = b * bs; id < hi; ++id)
                if (((bits[id >> 5] >> (id & 31)) & 1u) && !it->second.snapshot.contains(id))
                    rep.bytes_from_slow_tier += token_bytes();  // appended after caching
        } else {
            ++rep.misses;
            rep.bytes_from_slow_tier += counts[b] * token_bytes();
        }
        if (trace_enabled_) trace_.push_back({st.fetch_calls, layer, kv_head, b, hit});
    }
    st.hits += rep.hits;
    st.misses += rep.misses;
    st.requests += touched;

    // the middle segment is authoritative; cached copies are bit-identical
    rep.entries.reserve(token_ids.size());
    for (std::size_t id : token_ids) rep.entries.push_back(st.middle.at(id));

    // cache update: top-k_cache blocks of this request by requested-token count,
    // ties toward the lower block id
    for (std::int64_t rb : ranked) {
        if (rb < 0) break;
        const std::size_t block_id = static_cast<std::size_t>(rb);
        std::map<std::size_t, KvEntry> snapshot;
        for (std::size_t id = block_id * bs; id < (block_id + 1) * bs; ++id) {
            auto mit = st.middle.find(id);
            if (mit != st.middle.end()) snapshot.emplace(id, mit->second);
        }
        // a refresh re-inserts with its counters kept, so stale snapshots heal
        std::size_t freq = 1;
        std::uint64_t last = 0;
        auto it = st.cache.find(block_id);
        const bool was_cached = it != st.cache.end();
        if (was_cached) {
            freq = it->second.freq;
            last = it->second.last_used;
            st.occupancy_tokens -= it->second.snapshot.size();
            st.cache.erase(it);
        }
        if (snapshot.size() > cache_capacity_) continue;  // cannot fit even alone
        evict_until_fits(st, snapshot.size());
        const std::size_t tokens = snapshot.size();
        st.cache.emplace(block_id, HeadState::CachedBlock{std::move(snapshot), freq, was_cached ? last : ++st.tick});
        st.occupancy_tokens += tokens;
    }
    return rep;
}

CacheStats KvStore::cache_stats(std::size_t layer, std::size_t kv_head) const {
    const HeadState& st = state(layer, kv_head);
    CacheStats cs;
    cs.hits = st.hits;
    cs.misses = st.misses;
    cs.requests = st.requests;
    cs.occupancy_tokens = st.occupancy_tokens;
    cs.hit_rate = st.requests ? static_cast<double>(st.hits) / st.requests : 0.0;
    return cs;
}

// ---- .pqt file format (tensor.cpp:46-150, pq.cpp:184-222) -----------------------

static_assert(std::endian::native == std::endian::little, ".pqt I/O assumes a little-endian host");

namespace {

constexpr char kPqtMagic[4] = {'P', 'Q', 'K', 'V'};
constexpr std::uint8_t kPqtF32 = 0, kPqtU16 = 1;

template <typename T>
void put(std::ostream& out, const T& v) {
    out.write(reinterpret_cast<const char*>(&v), sizeof(T));
}

template <typename T>
T get(std::istream& in) {
    T v{};
    in.read(reinterpret_cast<char*>(&v), sizeof(T));
    if (!in) throw std::runtime_error("tensor: truncated file");
    return v;
}

void put_header(std::ostream& out, std::uint8_t dtype, const std::vector<std::size_t>& dims) {
    if (dims.empty()) throw std::invalid_argument("tensor: ndim must be >= 1");
    if (dims.size() > 255) throw std::invalid_argument("tensor: too many dimensions");
    out.write(kPqtMagic, 4);
    put(out, kTensorFormatVersion);
    put(out, dtype);
    put(out, static_cast<std::uint8_t>(dims.size()));
    for (std::size_t d : dims) put(out, static_cast<std::uint64_t>(d));
}

std::vector<std::size_t> get_header(std::istream& in, std::uint8_t want) {
    char magic[4];
    in.read(magic, 4);
    if (!in || std::memcmp(magic, kPqtMagic, 4) != 0) throw std::runtime_error("tensor: bad magic");
    if (get<std::uint32_t>(in) != kTensorFormatVersion) throw std::runtime_error("tensor: unsupported format version");
    if (get<std::uint8_t>(in) != want) throw std::runtime_error("tensor: unexpected dtype");
    const auto ndim = get<std::uint8_t>(in);
    if (ndim == 0) throw std::runtime_error("tensor: ndim must be >= 1");
    std::vector<std::size_t> dims(ndim);
    for (auto& d : dims) d = static_cast<std::size_t>(get<std::uint64_t>(in));
    return dims;
}

}  // namespace

void write_tensor(std::ostream& out, const TensorF32& t) {
    t.validate();
    put_header(out, kPqtF32, t.dims);
    out.write(reinterpret_cast<const char*>(t.data.data()), static_cast<std::streamsize>(t.data.size() * 4));
    if (!out) throw std::runtime_error("tensor: write failed");
}

TensorF32 read_tensor(std::istream& in) {
    TensorF32 t;
    t.dims = get_header(in, kPqtF32);
    t.data.resize(checked_numel(t.dims));
    in.read(reinterpret_cast<char*>(t.data.data()), static_cast<std::streamsize>(t.data.size() * 4));
    if (!in) throw std::runtime_error("tensor: truncated payload");
    t.validate();
    return t;
}

void write_grid_u16(std::ostream& out, const std::vector<std::size_t>& dims, const std::vector<std::uint16_t>& data) {
    if (checked_numel(dims) != data.size()) throw std::invalid_argument("grid: data size does not match product of dims");
    put_header(out, kPqtU16, dims);
    out.write(reinterpret_cast<const char*>(data.data()), static_cast<std::streamsize>(data.size() * 2));
    if (!out) throw std::runtime_error("grid: write failed");
}

void read_grid_u16(std::istream& in, std::vector<std::size_t>& dims, std::vector<std::uint16_t>& data) {
    dims = get_header(in, kPqtU16);
    data.resize(checked_numel(dims));
    in.read(reinterpret_cast<char*>(data.data()), static_cast<std::streamsize>(data.size() * 2));
    if (!in) throw std::runtime_error("grid: truncated payload");
}

void save_tensor(const std::string& path, const TensorF32& t) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("tensor: cannot open " + path);
    write_tensor(out, t);
}

TensorF32 load_tensor(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("tensor: cannot open " + path);
    return read_tensor(in);
}

void write_index(std::ostream& out, const PqIndex& index) {
    index.cfg.validate();
    write_tensor(out, index.centroids);
    write_grid_u16(out, {index.size(), index.cfg.m}, index.codes);
}

PqIndex read_index(std::istream& in) {
    PqIndex index;
    index.centroids = read_tensor(in);
    if (index.centroids.ndim() != 3) throw std::runtime_error("pq: centroid tensor must be 3-d");
    index.cfg.m = index.centroids.dims[0];
    index.cfg.n_clusters = index.centroids.dims[1];
    index.cfg.d_m = index.centroids.dims[2];
    index.cfg.b = 0;
    for (std::size_t b = 1; b <= 16; ++b)
        if ((std::size_t{1} << b) == index.cfg.n_clusters) index.cfg.b = b;
    index.cfg.validate();
    std::vector<std::size_t> dims;
    read_grid_u16(in, dims, index.codes);
    if (dims.size() != 2 || dims[1] != index.cfg.m) throw std::runtime_error("pq: code grid shape mismatch");
    for (std::uint16_t c : index.codes)
        if (c >= index.cfg.n_clusters) throw std::runtime_error("pq: code entry out of range");
    return index;
}

void save_index(const std::string& path, const PqIndex& index) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("pq: cannot open " + path);
    write_index(out, index);
}

PqIndex load_index(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("pq: cannot open " + path);
    return read_index(in);
}

}  // namespace pqkv
