// api.cpp -- the C++ drop-in API (include/pqkv/*.hpp) over the C ABI.
//
// Argument validation follows the reference's checks, order and exception
// types (kmeans.cpp:160-164, pq.cpp:13-177, topk.cpp:10-15,
// attention.cpp:11-104); every computation runs on the GPU through
// pqkv_c.h.  The host side here is the runtime that makes a value-semantics
// API cheap to call repeatedly (runtime_internal.hpp):
//   * one pqkv_ctx per (thread, device), destroyed with the thread;
//   * call scratch: a grow-only device stack, no cudaMalloc per call;
//   * device mirrors of PqIndex (codes uploaded once, appends incrementally)
//     and HeadState (a token's K/V row uploaded once), so a decode loop in
//     the reference's style (run_e2e, experiments.cpp:197-273) moves only the
//     new rows and each call's query/result across PCIe.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <list>
#include <numeric>
#include <stdexcept>
#include <string>

#include "pqkv/pqkv.hpp"
#include "runtime_internal.hpp"

namespace pqkv {

namespace detail {

[[noreturn]] void rethrow(int rc, const char* what) {
    const std::string msg = what && *what ? what : "pqkv: error";
    switch (rc) {
        case PQKV_EINVAL: throw std::invalid_argument(msg);
        case PQKV_ERANGE: throw std::out_of_range(msg);
        case PQKV_ESTATE: throw std::logic_error(msg);
        default: throw std::runtime_error(msg);
    }
}

namespace {

constexpr int kMaxDevices = 64;
constexpr std::size_t kMaxMirrors = 256;  // per (thread, device) and kind

struct DevBuf {
    void* p = nullptr;
    std::size_t bytes = 0;
};

struct IndexMirror {
    const PqIndex* owner = nullptr;
    std::vector<float> centroids;              // host copy (identity check)
    std::vector<std::uint16_t> first_row, last_row;
    std::size_t m = 0, rows = 0;
    DevBuf d_cen, d_codes;
    std::uint64_t stamp = 0;
};

struct StateMirror {
    const HeadState* owner = nullptr;
    std::size_t d_h = 0;
    std::vector<float> fingerprint;  // init keys (or the first local key)
    DevBuf d_k, d_v;
    std::size_t cap_tokens = 0;
    std::vector<std::uint8_t> resident;  // per token id
    std::uint64_t stamp = 0;
};

struct DeviceSlot {
    pqkv_ctx* ctx = nullptr;
    // call scratch: a stack of chunks; `top` = (chunk, offset) of the next byte
    std::vector<DevBuf> chunks;
    std::size_t chunk = 0, offset = 0;
    int depth = 0;
    std::list<IndexMirror> indexes;
    std::list<StateMirror> states;
    std::uint64_t clock = 0;
};

void free_buf(pqkv_ctx* ctx, DevBuf& b) {
    if (b.p) pqkv_device_free(ctx, b.p);
    b = DevBuf{};
}

void alloc_buf(pqkv_ctx* ctx, DevBuf& b, std::size_t bytes) {
    free_buf(ctx, b);
    check(pqkv_device_alloc(ctx, std::max<std::size_t>(bytes, 256), &b.p));
    b.bytes = std::max<std::size_t>(bytes, 256);
}

// Grows `b` to at least `bytes`, keeping its first `keep` bytes.
void grow_buf(pqkv_ctx* ctx, DevBuf& b, std::size_t bytes, std::size_t keep) {
    if (b.bytes >= bytes) return;
    DevBuf nb;
    check(pqkv_device_alloc(ctx, bytes, &nb.p));
    nb.bytes = bytes;
    if (keep && b.p) check(pqkv_copy(ctx, nb.p, b.p, keep, 2));
    free_buf(ctx, b);
    b = nb;
}

struct ThreadRuntime {
    int device = 0;
    DeviceSlot slots[kMaxDevices];

    ~ThreadRuntime() { release(); }

    void release() {
        for (DeviceSlot& s : slots) {
            if (!s.ctx) continue;
            for (DevBuf& c : s.chunks) free_buf(s.ctx, c);
            for (IndexMirror& m : s.indexes) {
                free_buf(s.ctx, m.d_cen);
                free_buf(s.ctx, m.d_codes);
            }
            for (StateMirror& m : s.states) {
                free_buf(s.ctx, m.d_k);
                free_buf(s.ctx, m.d_v);
            }
            s.chunks.clear();
            s.indexes.clear();
            s.states.clear();
            pqkv_ctx_destroy(s.ctx);
            s.ctx = nullptr;
        }
    }

    DeviceSlot& slot() {
        DeviceSlot& s = slots[device];
        if (!s.ctx) check(pqkv_ctx_create(device, &s.ctx));
        return s;
    }
};

thread_local ThreadRuntime t_rt;

}  // namespace

// ---- call scratch -----------------------------------------------------------

CallScratch::CallScratch() : slot_(t_rt.device) {
    DeviceSlot& s = t_rt.slot();
    if (s.depth++ == 0 && s.chunks.size() > 1) {
        // consolidate the chunks of the last call into one
        std::size_t total = 0;
        for (DevBuf& c : s.chunks) {
            total += c.bytes;
            free_buf(s.ctx, c);
        }
        s.chunks.assign(1, DevBuf{});
        alloc_buf(s.ctx, s.chunks[0], total);
    }
    // this frame's allocations start at the current top
    chunk_ = s.chunk;
    offset_ = s.offset;
}

CallScratch::~CallScratch() {
    DeviceSlot& s = t_rt.slots[slot_];
    s.chunk = chunk_;
    s.offset = offset_;
    --s.depth;
}

void* CallScratch::raw(std::size_t bytes) {
    DeviceSlot& s = t_rt.slots[slot_];
    bytes = (std::max<std::size_t>(bytes, 1) + 255) & ~std::size_t{255};
    while (true) {
        if (s.chunk < s.chunks.size() && s.offset + bytes <= s.chunks[s.chunk].bytes) {
            void* p = static_cast<char*>(s.chunks[s.chunk].p) + s.offset;
            s.offset += bytes;
            return p;
        }
        if (s.chunk + 1 < s.chunks.size() || (s.chunk < s.chunks.size() && s.offset > 0)) {
            if (s.chunk + 1 >= s.chunks.size()) {
                DevBuf nb;
                alloc_buf(s.ctx, nb, std::max(bytes, 2 * s.chunks[s.chunk].bytes));
                s.chunks.push_back(nb);
            }
            ++s.chunk;
            s.offset = 0;
            continue;
        }
        // empty or too-small first chunk that nothing lives in: replace it
        if (s.chunks.empty()) s.chunks.push_back(DevBuf{});
        alloc_buf(s.ctx, s.chunks[s.chunk], std::max<std::size_t>(bytes, 1 << 20));
        s.offset = 0;
    }
}

void CallScratch::copy_h2d(void* d, const void* h, std::size_t bytes) {
    if (bytes) check(pqkv_copy(t_rt.slots[slot_].ctx, d, h, bytes, 0));
}

namespace {
struct PhaseTotals {
    double us[kPhases] = {};
    long calls[kPhases] = {};
    ~PhaseTotals() {
        if (!api_profile()) return;
        static const char* names[kPhases] = {"sa_prep", "sa_mirror", "sa_compute", "ft_rank",
                                             "ft_account", "ft_entries", "ft_admit"};
        std::fprintf(stderr, "{\"api_profile_us\": {");
        for (int i = 0; i < kPhases; ++i)
            std::fprintf(stderr, "%s\"%s\": [%.1f, %ld]", i ? ", " : "", names[i], us[i], calls[i]);
        std::fprintf(stderr, "}}\n");
    }
};
PhaseTotals g_phases;
}  // namespace

bool api_profile() {
    static const bool on = [] {
        const char* e = std::getenv("PQKV_API_PROFILE");
        return e && *e && *e != '0';
    }();
    return on;
}

void phase_add(Phase p, double us) {
    g_phases.us[p] += us;
    ++g_phases.calls[p];
}

void copy_to_host(void* host, const void* dev, std::size_t bytes) {
    if (bytes) check(pqkv_copy(t_rt.slot().ctx, host, dev, bytes, 1));
}

// ---- PqIndex mirror ------------------------------------------------------------

IndexView mirror(const PqIndex& index) {
    DeviceSlot& s = t_rt.slot();
    const std::size_t m = index.cfg.m, rows = index.size();
    const std::vector<float>& cen = index.centroids.data;
    auto row_of = [&](std::size_t r) {
        return std::vector<std::uint16_t>(index.codes.begin() + r * m, index.codes.begin() + (r + 1) * m);
    };
    auto it = std::find_if(s.indexes.begin(), s.indexes.end(), [&](const IndexMirror& x) { return x.owner == &index; });
    if (it == s.indexes.end()) {
        if (s.indexes.size() >= kMaxMirrors) {  // drop the least recently used
            auto lru = std::min_element(s.indexes.begin(), s.indexes.end(),
                                        [](const IndexMirror& a, const IndexMirror& b) { return a.stamp < b.stamp; });
            free_buf(s.ctx, lru->d_cen);
            free_buf(s.ctx, lru->d_codes);
            s.indexes.erase(lru);
        }
        s.indexes.emplace_front();
        it = s.indexes.begin();
        it->owner = &index;
    }
    IndexMirror& mr = *it;
    mr.stamp = ++s.clock;
    // identity: same codebook, and the mirrored rows are still a prefix
    const bool same = mr.m == m && mr.centroids.size() == cen.size() &&
                      std::equal(cen.begin(), cen.end(), mr.centroids.begin(),
                                 [](float a, float b) { return std::memcmp(&a, &b, 4) == 0; }) &&
                      rows >= mr.rows && (mr.rows == 0 || (row_of(0) == mr.first_row && row_of(mr.rows - 1) == mr.last_row));
    if (!same) {
        mr.m = m;
        mr.rows = 0;
        mr.centroids = cen;
        alloc_buf(s.ctx, mr.d_cen, cen.size() * sizeof(float));
        if (!cen.empty()) check(pqkv_copy(s.ctx, mr.d_cen.p, cen.data(), cen.size() * sizeof(float), 0));
    }
    if (rows > mr.rows) {
        const std::size_t row_bytes = m * sizeof(std::uint16_t);
        if (mr.d_codes.bytes < rows * row_bytes)
            grow_buf(s.ctx, mr.d_codes, std::max((rows + rows / 4 + 4096) * row_bytes, 2 * mr.d_codes.bytes),
                     mr.rows * row_bytes);
        check(pqkv_copy(s.ctx, static_cast<char*>(mr.d_codes.p) + mr.rows * row_bytes,
                        index.codes.data() + mr.rows * m, (rows - mr.rows) * row_bytes, 0));
        mr.rows = rows;
        mr.first_row = row_of(0);
        mr.last_row = row_of(rows - 1);
    }
    return IndexView{static_cast<const float*>(mr.d_cen.p), static_cast<const std::uint16_t*>(mr.d_codes.p), rows};
}

// ---- HeadState mirror ------------------------------------------------------------

namespace {

const KvEntry* entry_of(const HeadState& st, std::size_t id) {
    if (id < st.init_entries.size()) return &st.init_entries[id];
    if (!st.local.empty() && id >= st.local.front().first) {
        const std::size_t off = id - st.local.front().first;
        if (off < st.local.size() && st.local[off].first == id) return &st.local[off].second;
        for (const auto& [lid, e] : st.local)
            if (lid == id) return &e;
    }
    auto it = st.middle.find(id);
    return it == st.middle.end() ? nullptr : &it->second;
}

std::vector<float> state_fingerprint(const HeadState& st) {
    std::vector<float> f;
    for (const KvEntry& e : st.init_entries) f.insert(f.end(), e.key.begin(), e.key.end());
    if (f.empty() && !st.middle.empty()) {
        const std::size_t lo = st.local.empty() ? 0 : st.local.front().first;
        if (const KvEntry* e = entry_of(st, lo >= st.middle.size() ? lo - st.middle.size() : 0))
            f = e->key;
    }
    return f;
}

}  // namespace

StateView mirror(const HeadState& st, std::size_t d_h, std::span<const std::int64_t> ids) {
    DeviceSlot& s = t_rt.slot();
    auto it = std::find_if(s.states.begin(), s.states.end(), [&](const StateMirror& x) { return x.owner == &st; });
    if (it == s.states.end()) {
        if (s.states.size() >= kMaxMirrors) {
            auto lru = std::min_element(s.states.begin(), s.states.end(),
                                        [](const StateMirror& a, const StateMirror& b) { return a.stamp < b.stamp; });
            free_buf(s.ctx, lru->d_k);
            free_buf(s.ctx, lru->d_v);
            s.states.erase(lru);
        }
        s.states.emplace_front();
        it = s.states.begin();
        it->owner = &st;
    }
    StateMirror& mr = *it;
    mr.stamp = ++s.clock;
    std::vector<float> fp = state_fingerprint(st);
    if (mr.d_h != d_h || fp.size() != mr.fingerprint.size() ||
        std::memcmp(fp.data(), mr.fingerprint.data(), fp.size() * sizeof(float)) != 0) {
        // another state (or another head_dim) at this address: start over
        mr.d_h = d_h;
        mr.fingerprint = std::move(fp);
        free_buf(s.ctx, mr.d_k);
        free_buf(s.ctx, mr.d_v);
        mr.cap_tokens = 0;
        mr.resident.clear();
    }
    const std::size_t need = st.total_tokens;
    if (mr.cap_tokens < need) {
        // headroom: decode appends one token per step; a regrow is a
        // cudaMalloc + D2D copy + cudaFree of the whole mirror
        const std::size_t cap = std::max(need + need / 4 + 1024, mr.cap_tokens + mr.cap_tokens / 2);
        grow_buf(s.ctx, mr.d_k, cap * d_h * sizeof(float), mr.cap_tokens * d_h * sizeof(float));
        grow_buf(s.ctx, mr.d_v, cap * d_h * sizeof(float), mr.cap_tokens * d_h * sizeof(float));
        mr.cap_tokens = cap;
        mr.resident.resize(cap, 0);
    }
    // rows not yet on the device: packed on the host, one copy, one scatter
    std::vector<std::int64_t> missing;
    for (std::int64_t id : ids)
        if (!mr.resident[static_cast<std::size_t>(id)]) {
            missing.push_back(id);
            mr.resident[static_cast<std::size_t>(id)] = 1;
        }
    if (!missing.empty()) {
        std::vector<float> pk(missing.size() * d_h), pv(missing.size() * d_h);
        for (std::size_t i = 0; i < missing.size(); ++i) {
            const KvEntry* e = entry_of(st, static_cast<std::size_t>(missing[i]));
            if (!e || e->key.size() != d_h || e->value.size() != d_h) {
                for (std::int64_t id : missing) mr.resident[static_cast<std::size_t>(id)] = 0;
                if (!e) throw std::out_of_range("attention: token " + std::to_string(missing[i]) + " is not stored");
                throw std::invalid_argument("attention: entry dim mismatch");
            }
            std::copy(e->key.begin(), e->key.end(), pk.begin() + i * d_h);
            std::copy(e->value.begin(), e->value.end(), pv.begin() + i * d_h);
        }
        CallScratch sc;
        const std::int64_t* d_ids = sc.upload(missing.data(), missing.size());
        const float* d_pk = sc.upload(pk.data(), pk.size());
        const float* d_pv = sc.upload(pv.data(), pv.size());
        check(pqkv_scatter_rows(s.ctx, d_pk, d_pv, d_ids, missing.size(), d_h, static_cast<float*>(mr.d_k.p),
                                static_cast<float*>(mr.d_v.p), nullptr));
    }
    return StateView{static_cast<const float*>(mr.d_k.p), static_cast<const float*>(mr.d_v.p), d_h};
}

// ---- block ranking of a fetch -------------------------------------------------

BlockRanking rank_blocks(std::span<const std::size_t> ids, std::size_t n_tokens, std::size_t block_size,
                         std::size_t k_cache) {
    const std::size_t n_blocks = std::max<std::size_t>(1, (n_tokens + block_size - 1) / block_size);
    const std::size_t words = (n_tokens + 31) / 32, k_rank = std::min(k_cache, n_blocks);
    BlockRanking br;
    br.bits.resize(words);
    br.counts.resize(n_blocks);
    br.ranked.resize(k_rank);
    CallScratch sc;
    std::vector<std::int64_t> h_ids(ids.begin(), ids.end());
    const std::int64_t* d_ids = sc.upload(h_ids.data(), h_ids.size());
    // the three results packed in one scratch span: one device->host copy
    const std::size_t o_counts = (words * 4 + 255) & ~std::size_t{255};
    const std::size_t o_ranked = o_counts + ((n_blocks * 4 + 255) & ~std::size_t{255});
    const std::size_t span = o_ranked + k_rank * 8;
    char* d_out = sc.alloc<char>(span);
    auto* d_bits = reinterpret_cast<std::uint32_t*>(d_out);
    auto* d_counts = reinterpret_cast<std::uint32_t*>(d_out + o_counts);
    auto* d_ranked = reinterpret_cast<std::int64_t*>(d_out + o_ranked);
    check(pqkv_block_rank(t_rt.slot().ctx, d_ids, 1, h_ids.size(), h_ids.size(), n_tokens, block_size, k_rank,
                          d_bits, d_counts, d_ranked, nullptr, nullptr));
    std::vector<char> h_out(span);
    copy_to_host(h_out.data(), d_out, span);
    std::memcpy(br.bits.data(), h_out.data(), words * 4);
    std::memcpy(br.counts.data(), h_out.data() + o_counts, n_blocks * 4);
    std::memcpy(br.ranked.data(), h_out.data() + o_ranked, k_rank * 8);
    return br;
}

}  // namespace detail

using detail::CallScratch;
using detail::check;
using detail::copy_to_host;

// ---- runtime control ------------------------------------------------------------

void set_device(int device) {
    if (device < 0 || device >= detail::kMaxDevices) throw std::invalid_argument("pqkv: bad device");
    detail::t_rt.device = device;
}

pqkv_ctx* default_context() { return detail::t_rt.slot().ctx; }

void forget_mirrors() {
    detail::DeviceSlot& s = detail::t_rt.slot();
    for (auto& m : s.indexes) {
        detail::free_buf(s.ctx, m.d_cen);
        detail::free_buf(s.ctx, m.d_codes);
    }
    for (auto& m : s.states) {
        detail::free_buf(s.ctx, m.d_k);
        detail::free_buf(s.ctx, m.d_v);
    }
    s.indexes.clear();
    s.states.clear();
}

// ---- k-means (kmeans.hpp) ------------------------------------------------------------

KmeansResult kmeans_fit(const TensorF32& points, std::size_t n_clusters, std::size_t max_iter, std::uint64_t seed) {
    points.validate();
    if (points.ndim() != 2) throw std::invalid_argument("kmeans: points must be 2-d");
    if (n_clusters < 1) throw std::invalid_argument("kmeans: n_clusters must be >= 1");
    if (max_iter < 1) throw std::invalid_argument("kmeans: max_iter must be >= 1");
    const std::size_t n = points.dims[0], dim = points.dims[1];
    CallScratch sc;
    const float* dp = sc.upload(points.data.data(), n * dim);
    float* dc = sc.alloc<float>(n_clusters * dim);
    auto* da = sc.alloc<std::uint32_t>(n);
    auto* di = sc.alloc<std::uint32_t>(1);
    auto* dinert = sc.alloc<double>(max_iter);
    check(pqkv_kmeans_fit(default_context(), dp, 1, n * dim, dim, n, dim, n_clusters, max_iter, &seed, dc, da, di,
                          dinert, nullptr));
    KmeansResult res;
    std::vector<float> cen(n_clusters * dim);
    copy_to_host(cen.data(), dc, cen.size() * 4);
    res.centroids = TensorF32({n_clusters, dim}, std::move(cen));
    std::vector<std::uint32_t> a(n);
    copy_to_host(a.data(), da, n * 4);
    res.assignments.assign(a.begin(), a.end());
    std::uint32_t its = 0;
    copy_to_host(&its, di, 4);
    res.iterations_run = its;
    res.inertia_trace.resize(its);
    copy_to_host(res.inertia_trace.data(), dinert, its * 8);
    return res;
}

std::vector<std::size_t> assign_nearest(const TensorF32& points, const TensorF32& centroids) {
    if (points.ndim() != 2 || centroids.ndim() != 2)
        throw std::invalid_argument("assign_nearest: points and centroids must be 2-d");
    if (points.dims[1] != centroids.dims[1]) throw std::invalid_argument("assign_nearest: dimension mismatch");
    const std::size_t n = points.dims[0], dim = points.dims[1], k = centroids.dims[0];
    CallScratch sc;
    const float* dp = sc.upload(points.data.data(), n * dim);
    const float* dc = sc.upload(centroids.data.data(), k * dim);
    auto* da = sc.alloc<std::uint32_t>(n);
    check(pqkv_assign_nearest(default_context(), dp, n, dim, dc, k, da, nullptr));
    std::vector<std::uint32_t> a(n);
    copy_to_host(a.data(), da, n * 4);
    return std::vector<std::size_t>(a.begin(), a.end());
}

// ---- PQ (pq.hpp) ------------------------------------------------------------------

PqConfig PqConfig::create(std::size_t m, std::size_t b, std::size_t d_h) {
    PqConfig cfg;
    check(pqkv_pq_config(m, b, d_h, &cfg.d_m, &cfg.n_clusters));
    cfg.m = m;
    cfg.b = b;
    return cfg;
}

void PqConfig::validate() const {
    if (m < 1 || d_m < 1) throw std::invalid_argument("pq: m and d_m must be >= 1");
    if (b < 1 || b > 16) throw std::invalid_argument("pq: b must be in [1, 16]");
    if (n_clusters != (std::size_t{1} << b)) throw std::invalid_argument("pq: n_clusters must equal 2^b");
}

const float* PqIndex::centroid(std::size_t partition, std::size_t cluster) const {
    return centroids.data.data() + (partition * cfg.n_clusters + cluster) * cfg.d_m;
}

const std::uint16_t* PqIndex::code_row(std::size_t token) const {
    if (token >= size()) throw std::out_of_range("pq: token id out of range");
    return codes.data() + token * cfg.m;
}

PqIndex pq_construct(const TensorF32& keys, const PqConfig& cfg, std::size_t max_iter, std::uint64_t seed) {
    cfg.validate();
    keys.validate();
    if (keys.ndim() != 2) throw std::invalid_argument("pq: keys must be 2-d");
    if (keys.dims[1] != cfg.head_dim()) throw std::invalid_argument("pq: key dim must equal m * d_m");
    const std::size_t s = keys.dims[0], d_h = keys.dims[1];
    if (s < 1) throw std::invalid_argument("pq: need at least one key");
    if (max_iter < 1) throw std::invalid_argument("kmeans: max_iter must be >= 1");
    CallScratch sc;
    const float* dk = sc.upload(keys.data.data(), s * d_h);
    float* dc = sc.alloc<float>(cfg.m * cfg.n_clusters * cfg.d_m);
    auto* dcodes = sc.alloc<std::uint16_t>(s * cfg.m);
    check(pqkv_pq_build(default_context(), dk, 1, s * d_h, s, d_h, cfg.m, cfg.b, max_iter, &seed, dc, dcodes,
                        s * cfg.m, nullptr));
    PqIndex index;
    index.cfg = cfg;
    std::vector<float> cen(cfg.m * cfg.n_clusters * cfg.d_m);
    copy_to_host(cen.data(), dc, cen.size() * 4);
    index.centroids = TensorF32({cfg.m, cfg.n_clusters, cfg.d_m}, std::move(cen));
    index.codes.resize(s * cfg.m);
    copy_to_host(index.codes.data(), dcodes, index.codes.size() * 2);
    return index;
}

std::vector<std::uint16_t> pq_encode_one(std::span<const float> key, const PqIndex& index) {
    const PqConfig& cfg = index.cfg;
    if (key.size() != cfg.head_dim()) throw std::invalid_argument("pq: key dim must equal m * d_m");
    const detail::IndexView iv = detail::mirror(index);
    CallScratch sc;
    const float* dk = sc.upload(key.data(), key.size());
    auto* dcode = sc.alloc<std::uint16_t>(cfg.m);
    check(pqkv_pq_encode(default_context(), dk, 1, key.size(), cfg.head_dim(), cfg.m, cfg.b, iv.centroids, dcode,
                         cfg.m, 0, nullptr));
    std::vector<std::uint16_t> code(cfg.m);
    copy_to_host(code.data(), dcode, cfg.m * 2);
    return code;
}

void append_code(PqIndex& index, std::span<const std::uint16_t> code) {
    if (code.size() != index.cfg.m) throw std::invalid_argument("pq: code must have m entries");
    if (std::any_of(code.begin(), code.end(), [&](std::uint16_t c) { return c >= index.cfg.n_clusters; }))
        throw std::invalid_argument("pq: code entry out of range");
    index.codes.insert(index.codes.end(), code.begin(), code.end());
}

namespace {

std::vector<float> adc_scores(const float* queries, std::size_t g, const PqIndex& index) {
    const PqConfig& cfg = index.cfg;
    const std::size_t s = index.size(), d_h = cfg.head_dim();
    std::vector<float> out(s);
    if (s == 0) return out;
    const detail::IndexView iv = detail::mirror(index);
    CallScratch sc;
    const float* dq = sc.upload(queries, g * d_h);
    float* ds = sc.alloc<float>(s);
    check(pqkv_pq_score(default_context(), dq, 1, g, d_h, cfg.m, cfg.b, iv.centroids, iv.codes, s * cfg.m, s, ds, s,
                        nullptr));
    copy_to_host(out.data(), ds, s * 4);
    return out;
}

}  // namespace

std::vector<float> pq_score(std::span<const float> query, const PqIndex& index) {
    if (query.size() != index.cfg.head_dim()) throw std::invalid_argument("pq: query dim must equal m * d_m");
    return adc_scores(query.data(), 1, index);
}

std::vector<float> pq_score_gqa(const TensorF32& queries, const PqIndex& index) {
    if (queries.ndim() != 2 || queries.dims[0] < 1)
        throw std::invalid_argument("pq: queries must be a non-empty 2-d grid");
    if (queries.dims[1] != index.cfg.head_dim()) throw std::invalid_argument("pq: query dim must equal m * d_m");
    return adc_scores(queries.data.data(), queries.dims[0], index);
}

std::vector<float> reconstruct(const PqIndex& index, std::size_t token) {
    const PqConfig& cfg = index.cfg;
    const std::uint16_t* code = index.code_row(token);
    std::vector<float> out;
    out.reserve(cfg.head_dim());
    for (std::size_t j = 0; j < cfg.m; ++j) {
        const float* c = index.centroid(j, code[j]);
        out.insert(out.end(), c, c + cfg.d_m);
    }
    return out;
}

std::vector<std::size_t> top_k_desc(std::span<const float> scores, std::size_t k,
                                    const std::unordered_set<std::size_t>& excluded) {
    const std::size_t n = scores.size();
    const std::size_t n_ex = std::count_if(excluded.begin(), excluded.end(), [n](std::size_t e) { return e < n; });
    if (k > n - n_ex) throw std::invalid_argument("top_k: k too large for the candidate set");
    if (k == 0) return {};
    CallScratch sc;
    const float* ds = sc.upload(scores.data(), n);
    const std::uint8_t* dm = nullptr;
    if (n_ex) {
        std::vector<std::uint8_t> mask(n, 0);
        for (std::size_t e : excluded)
            if (e < n) mask[e] = 1;
        dm = sc.upload(mask.data(), n);
    }
    auto* dids = sc.alloc<std::int64_t>(k);
    check(pqkv_topk(default_context(), ds, 1, n, n, k, dm, dids, nullptr));
    std::vector<std::int64_t> ids(k);
    copy_to_host(ids.data(), dids, k * 8);
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

// ---- attention (attention.hpp) ------------------------------------------------------
//
// The reference's fp64 order (PQKV_PREC_F64: exact_scores bit-identical,
// serial total, row-ordered accumulation), so outputs round to the
// reference's f32 values.

namespace {

// g query rows over t contiguous host K/V rows.
std::vector<float> attend_dense(const float* queries, std::size_t g, std::size_t d_h, const float* keys,
                                const float* values, std::size_t t) {
    CallScratch sc;
    const float* dq = sc.upload(queries, g * d_h);
    const float* dk = sc.upload(keys, t * d_h);
    const float* dv = sc.upload(values, t * d_h);
    std::vector<std::int64_t> rows(t);
    std::iota(rows.begin(), rows.end(), 0);
    const std::int64_t* dr = sc.upload(rows.data(), t);
    float* dout = sc.alloc<float>(g * d_h);
    check(pqkv_attend_rows(default_context(), dq, 1, g, d_h, dk, dv, t * d_h, dr, t, PQKV_PREC_F64, dout, nullptr));
    std::vector<float> out(g * d_h);
    copy_to_host(out.data(), dout, out.size() * 4);
    return out;
}

void check_kv(const TensorF32& keys, const TensorF32& values) {
    if (values.ndim() != 2 || values.dims != keys.dims)
        throw std::invalid_argument("attention: values must match key dims");
    if (keys.dims[0] < 1) throw std::invalid_argument("attention: need at least one token");
}

}  // namespace

std::vector<float> exact_scores(std::span<const float> query, const TensorF32& keys) {
    if (keys.ndim() != 2) throw std::invalid_argument("attention: keys must be 2-d");
    if (keys.dims[1] != query.size()) throw std::invalid_argument("attention: query dim must match key dim");
    const std::size_t t = keys.dims[0], d_h = keys.dims[1];
    std::vector<float> out(t);
    if (t == 0) return out;
    CallScratch sc;
    const float* dq = sc.upload(query.data(), d_h);
    const float* dk = sc.upload(keys.data.data(), t * d_h);
    std::vector<std::int64_t> rows(t);
    std::iota(rows.begin(), rows.end(), 0);
    const std::int64_t* dr = sc.upload(rows.data(), t);
    float* ds = sc.alloc<float>(t);
    check(pqkv_exact_scores(default_context(), dq, 1, 1, d_h, dk, t * d_h, dr, t, ds, nullptr));
    copy_to_host(out.data(), ds, t * 4);
    return out;
}

std::vector<std::size_t> exact_topk(std::span<const float> query, const TensorF32& keys, std::size_t k,
                                    const std::unordered_set<std::size_t>& excluded) {
    return top_k_desc(exact_scores(query, keys), k, excluded);
}

std::vector<float> softmax_attention(std::span<const float> query, const TensorF32& keys, const TensorF32& values) {
    check_kv(keys, values);
    if (keys.ndim() != 2) throw std::invalid_argument("attention: keys must be 2-d");
    if (keys.dims[1] != query.size()) throw std::invalid_argument("attention: query dim must match key dim");
    return attend_dense(query.data(), 1, keys.dims[1], keys.data.data(), values.data.data(), keys.dims[0]);
}

std::vector<float> selective_attention(std::span<const float> query, const HeadState& state,
                                       std::span<const std::size_t> selected_middle_ids) {
    detail::PhaseTimer pt;
    // ascending, duplicate-free ids: a bitmap over the token ids (all ids are
    // < total_tokens in any valid call; otherwise sort)
    std::vector<std::size_t> ids;
    ids.reserve(selected_middle_ids.size());
    const std::size_t n_tok = state.total_tokens;
    if (std::all_of(selected_middle_ids.begin(), selected_middle_ids.end(),
                    [&](std::size_t id) { return id < n_tok; })) {
        std::vector<std::uint64_t> seen((n_tok + 63) / 64, 0);
        for (std::size_t id : selected_middle_ids) {
            std::uint64_t& w = seen[id >> 6];
            const std::uint64_t bit = std::uint64_t{1} << (id & 63);
            if (w & bit) throw std::invalid_argument("attention: duplicate middle token id");
            w |= bit;
        }
        for (std::size_t wi = 0; wi < seen.size(); ++wi)
            for (std::uint64_t w = seen[wi]; w; w &= w - 1)
                ids.push_back(wi * 64 + static_cast<std::size_t>(__builtin_ctzll(w)));
    } else {
        ids.assign(selected_middle_ids.begin(), selected_middle_ids.end());
        std::sort(ids.begin(), ids.end());
        if (std::adjacent_find(ids.begin(), ids.end()) != ids.end())
            throw std::invalid_argument("attention: duplicate middle token id");
    }
    const std::size_t d_h = query.size();
    const std::size_t t = state.init_entries.size() + ids.size() + state.local.size();
    if (t == 0 || d_h == 0) throw std::invalid_argument("tensor: zero-sized dimension");
    // middle membership: O(1) when the middle segment is the contiguous id
    // range [n_init, first local id) that offload_prefill + evict_local_append
    // maintain (checked), else a lookup per id
    const std::size_t n_init = state.init_entries.size();
    const std::size_t hi = state.local.empty() ? state.total_tokens : state.local.front().first;
    const bool contiguous = hi >= n_init && state.middle.size() == hi - n_init &&
                            (hi == n_init || (state.middle.contains(n_init) && state.middle.contains(hi - 1)));
    std::vector<std::int64_t> rows;
    rows.reserve(t);
    for (std::size_t i = 0; i < n_init; ++i) rows.push_back(static_cast<std::int64_t>(i));
    for (std::size_t id : ids) {
        const bool is_mid = contiguous ? (id >= n_init && id < hi) : state.middle.contains(id);
        if (!is_mid) throw std::out_of_range("attention: token " + std::to_string(id) + " is not a middle token");
        rows.push_back(static_cast<std::int64_t>(id));
    }
    for (const auto& lt : state.local) rows.push_back(static_cast<std::int64_t>(lt.first));
    // entry dims (the reference checks every entry it copies; middle rows are
    // checked when first mirrored)
    auto bad_dim = [&](const KvEntry& e) { return e.key.size() != d_h || e.value.size() != d_h; };
    if (std::any_of(state.init_entries.begin(), state.init_entries.end(), bad_dim) ||
        std::any_of(state.local.begin(), state.local.end(), [&](const auto& lt) { return bad_dim(lt.second); }))
        throw std::invalid_argument("attention: entry dim mismatch");
    pt.lap(detail::kSaPrep);
    const detail::StateView sv = detail::mirror(state, d_h, rows);
    pt.lap(detail::kSaMirror);
    CallScratch sc;
    const float* dq = sc.upload(query.data(), d_h);
    const std::int64_t* dr = sc.upload(rows.data(), t);
    float* dout = sc.alloc<float>(d_h);
    check(pqkv_attend_rows(default_context(), dq, 1, 1, d_h, sv.keys, sv.values, 0, dr, t, PQKV_PREC_F64, dout,
                           nullptr));
    std::vector<float> out(d_h);
    copy_to_host(out.data(), dout, d_h * 4);
    pt.lap(detail::kSaCompute);
    return out;
}

TensorF32 gqa_group_attention(const TensorF32& queries, const TensorF32& keys, const TensorF32& values) {
    if (queries.ndim() != 2 || queries.dims[0] < 1)
        throw std::invalid_argument("attention: queries must be a non-empty 2-d grid");
    check_kv(keys, values);
    if (keys.ndim() != 2) throw std::invalid_argument("attention: keys must be 2-d");
    const std::size_t g = queries.dims[0], d_h = queries.dims[1];
    if (keys.dims[1] != d_h) throw std::invalid_argument("attention: query dim must match key dim");
    return TensorF32({g, d_h}, attend_dense(queries.data.data(), g, d_h, keys.data.data(), values.data.data(),
                                            keys.dims[0]));
}

}  // namespace pqkv

// run_recall's seeder stream (experiments.cpp:90-113): host arithmetic on
// the reference's Rng, exported for device-side recall drivers.
extern "C" PQKV_CXX_API int pqkv_recall_seeds(uint64_t seed, size_t h_kv, const size_t* ks, size_t n_k, size_t s,
                                              uint64_t* fork_seeds, int64_t* random_ids) {
    try {
        if ((n_k && !ks) || (h_kv && !fork_seeds)) throw std::invalid_argument("recall_seeds: NULL buffer");
        std::size_t total = 0;
        for (std::size_t i = 0; i < n_k; ++i) {
            if (ks[i] < 1 || ks[i] > s) throw std::invalid_argument("recall: k must be in [1, s]");
            total += ks[i];
        }
        if (h_kv && total && !random_ids) throw std::invalid_argument("recall_seeds: NULL buffer");
        pqkv::Rng rng(seed);
        std::vector<std::size_t> pool(s);
        for (std::size_t h = 0; h < h_kv; ++h) {
            fork_seeds[h] = rng.fork_seed();
            std::size_t off = h * total;
            for (std::size_t ki = 0; ki < n_k; ++ki) {
                std::iota(pool.begin(), pool.end(), std::size_t{0});
                for (std::size_t i = 0; i < ks[ki]; ++i) std::swap(pool[i], pool[i + rng.index(s - i)]);
                for (std::size_t i = 0; i < ks[ki]; ++i) random_ids[off + i] = static_cast<int64_t>(pool[i]);
                off += ks[ki];
            }
        }
        return PQKV_OK;
    } catch (const std::invalid_argument&) {
        return PQKV_EINVAL;
    } catch (...) {
        return PQKV_ERUNTIME;
    }
}
