// kv_store_host.cpp -- KvStore (reference kv_store.cpp:10-211): the
// three-segment token layout, evict-and-encode, and block-granular fetches
// with the fast-tier block cache.
//
// Structure here: a fetch is (1) the per-request analysis -- distinct tokens
// per block and the (count desc, block asc) ranking -- computed on the GPU by
// pqkv_block_rank (blocks.cu), then (2) a host pass over the touched blocks
// for hit/miss accounting, then (3) admission of the ranked blocks into the
// cache (admit_block), evicting by policy (make_room).  Only (2) and (3), a
// small sequential state machine, run on the host.
#include <algorithm>
#include <ostream>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "pqkv/kv_store.hpp"
#include "pqkv/runtime.hpp"
#include "pqkv_c.h"
#include "runtime_internal.hpp"

namespace pqkv {

KvStore::KvStore(std::size_t num_layers, std::size_t num_kv_heads, std::size_t block_size,
                 std::size_t cache_capacity_tokens, CachePolicy policy)
    : num_layers_(num_layers), num_kv_heads_(num_kv_heads), block_size_(block_size),
      cache_capacity_(cache_capacity_tokens), policy_(policy) {
    if (num_layers == 0 || num_kv_heads == 0)
        throw std::invalid_argument("kv_store: need at least one layer and kv head");
    if (block_size == 0) throw std::invalid_argument("kv_store: block_size must be >= 1");
    states_.resize(num_layers * num_kv_heads);
}

std::size_t KvStore::slot(std::size_t layer, std::size_t kv_head) const {
    if (layer >= num_layers_ || kv_head >= num_kv_heads_)
        throw std::out_of_range("kv_store: layer or kv_head out of range");
    return layer * num_kv_heads_ + kv_head;
}

const HeadState& KvStore::state(std::size_t layer, std::size_t kv_head) const {
    return states_[slot(layer, kv_head)];
}

OffloadReport KvStore::offload_prefill(std::size_t layer, std::size_t kv_head, const TensorF32& keys,
                                       const TensorF32& values, const SegmentConfig& seg) {
    HeadState& st = states_[slot(layer, kv_head)];
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

    auto entry = [&](std::size_t i) {
        return KvEntry{std::vector<float>(keys.row(i), keys.row(i) + d_h),
                       std::vector<float>(values.row(i), values.row(i) + d_h)};
    };
    // segments are contiguous id ranges: [0, lo) init, [lo, hi) middle, [hi, s) local
    const std::size_t lo = seg.n_init, hi = s - seg.n_local;
    for (std::size_t i = 0; i < lo; ++i) st.init_entries.push_back(entry(i));
    for (std::size_t i = lo; i < hi; ++i) st.middle.emplace(i, entry(i));
    for (std::size_t i = hi; i < s; ++i) st.local.emplace_back(i, entry(i));
    st.total_tokens = s;
    st.prefilled = true;

    OffloadReport rep;
    rep.init_tokens = lo;
    rep.middle_tokens = hi - lo;
    rep.local_tokens = s - hi;
    rep.middle_blocks = hi > lo ? (hi - 1) / block_size_ - lo / block_size_ + 1 : 0;
    rep.bytes_offloaded = rep.middle_tokens * entry_bytes();
    return rep;
}

std::size_t KvStore::evict_local_append(std::size_t layer, std::size_t kv_head, KvEntry new_entry,
                                        PqIndex& index) {
    HeadState& st = states_[slot(layer, kv_head)];
    if (st.local.empty()) throw std::logic_error("kv_store: local segment is empty");
    if (new_entry.key.size() != head_dim_ || new_entry.value.size() != head_dim_)
        throw std::invalid_argument("kv_store: entry dim mismatch");
    auto oldest = std::move(st.local.front());
    st.local.pop_front();
    // the evicted key is encoded against the (device-resident) codebook and
    // its code row appended: it is now a middle token
    append_code(index, pq_encode_one(oldest.second.key, index));
    const std::size_t evicted = oldest.first;
    st.middle.emplace(evicted, std::move(oldest.second));
    st.local.emplace_back(st.total_tokens++, std::move(new_entry));
    return evicted;
}

// Evicts cached blocks until `incoming_tokens` fit: LRU by last use; LFU by
// frequency, then last use; remaining ties to the lowest block id (the first
// minimum in the map's id order).
void KvStore::make_room(HeadState& st, std::size_t incoming_tokens) {
    auto rank = [this](const auto& kv) {
        const HeadState::CachedBlock& b = kv.second;
        return policy_ == CachePolicy::kLru ? std::make_tuple(std::size_t{0}, b.last_used)
                                            : std::make_tuple(b.freq, b.last_used);
    };
    while (!st.cache.empty() && st.occupancy_tokens + incoming_tokens > cache_capacity_) {
        auto victim = std::min_element(st.cache.begin(), st.cache.end(),
                                       [&](const auto& a, const auto& b) { return rank(a) < rank(b); });
        st.occupancy_tokens -= victim->second.snapshot.size();
        retired_.push_back(std::move(victim->second.snapshot));
        st.cache.erase(victim);
    }
}

// (Re)admits one ranked block: a fresh snapshot of its middle tokens; a block
// already cached keeps its counters (so a stale snapshot heals); a block
// larger than the whole cache is dropped.
void KvStore::admit_block(HeadState& st, std::size_t block_id, std::map<std::size_t, KvEntry>&& snapshot) {
    HeadState::CachedBlock blk;
    blk.snapshot = std::move(snapshot);
    bool refreshed = false;
    if (auto old = st.cache.find(block_id); old != st.cache.end()) {
        blk.freq = old->second.freq;
        blk.last_used = old->second.last_used;
        st.occupancy_tokens -= old->second.snapshot.size();
        retired_.push_back(std::move(old->second.snapshot));
        st.cache.erase(old);
        refreshed = true;
    }
    const std::size_t tokens = blk.snapshot.size();
    if (tokens > cache_capacity_) {
        retired_.push_back(std::move(blk.snapshot));
        return;
    }
    make_room(st, tokens);
    if (!refreshed) {
        blk.freq = 1;
        blk.last_used = ++st.tick;
    }
    st.cache.emplace(block_id, std::move(blk));
    st.occupancy_tokens += tokens;
}

FetchReport KvStore::fetch_topk(std::size_t layer, std::size_t kv_head, std::span<const std::size_t> token_ids,
                                std::size_t k_cache) {
    detail::PhaseTimer pt;
    HeadState& st = states_[slot(layer, kv_head)];
    for (std::size_t id : token_ids)
        if (!st.middle.contains(id))
            throw std::out_of_range("kv_store: token " + std::to_string(id) + " is not a middle token");
    ++st.fetch_calls;

    // (1) request analysis on the GPU
    const std::size_t bs = block_size_, n_tokens = st.total_tokens;
    const detail::BlockRanking br = detail::rank_blocks(token_ids, n_tokens, bs, k_cache);
    pt.lap(detail::kFtRank);

    // (2) one lookup per touched block, ascending block id
    FetchReport rep;
    std::size_t touched = 0;
    for (std::size_t b = 0; b < br.counts.size(); ++b) {
        if (br.counts[b] == 0) continue;
        ++touched;
        auto cached = st.cache.find(b);
        const bool hit = cached != st.cache.end();
        if (hit) {
            ++rep.hits;
            ++cached->second.freq;
            cached->second.last_used = ++st.tick;
            // requested tokens appended to the middle after the block was cached
            const auto& snap = cached->second.snapshot;
            for (std::size_t id = b * bs, end = std::min(n_tokens, id + bs); id < end; ++id)
                if (br.requested(id) && !snap.contains(id)) rep.bytes_from_slow_tier += entry_bytes();
        } else {
            ++rep.misses;
            rep.bytes_from_slow_tier += br.counts[b] * entry_bytes();
        }
        if (trace_enabled_) trace_.push_back(TraceRow{st.fetch_calls, layer, kv_head, b, hit});
    }
    st.hits += rep.hits;
    st.misses += rep.misses;
    st.requests += touched;

    pt.lap(detail::kFtAccount);
    // entries come from the middle segment (cache snapshots are copies of it)
    // (thousands of KvEntry copies: spread over the host worker pool)
    rep.entries.resize(token_ids.size());
    detail::parallel_for(token_ids.size(), 256, [&](std::size_t lo, std::size_t hi) {
        for (std::size_t i = lo; i < hi; ++i) rep.entries[i] = st.middle.find(token_ids[i])->second;  // ids checked above
    });

    pt.lap(detail::kFtEntries);
    // (3) admission of this request's top-k_cache blocks
    // snapshots first (copies of the middle tokens, built in parallel), then
    // the sequential cache-state updates in rank order
    std::size_t n_ranked = 0;
    while (n_ranked < br.ranked.size() && br.ranked[n_ranked] >= 0) ++n_ranked;
    std::vector<std::map<std::size_t, KvEntry>> snaps(n_ranked);
    detail::parallel_for(n_ranked, 1, [&](std::size_t lo, std::size_t hi) {
        for (std::size_t r = lo; r < hi; ++r) {
            const std::size_t b0 = static_cast<std::size_t>(br.ranked[r]) * bs;
            for (std::size_t id = b0; id < b0 + bs; ++id)
                if (auto m = st.middle.find(id); m != st.middle.end()) snaps[r].emplace_hint(snaps[r].end(), id, m->second);
        }
    });
    for (std::size_t r = 0; r < n_ranked; ++r)
        admit_block(st, static_cast<std::size_t>(br.ranked[r]), std::move(snaps[r]));
    // snapshots replaced or evicted above: thousands of KvEntry frees, spread
    // over the host worker pool
    detail::parallel_for(retired_.size(), 1, [&](std::size_t lo, std::size_t hi) {
        for (std::size_t i = lo; i < hi; ++i) retired_[i].clear();
    });
    retired_.clear();
    pt.lap(detail::kFtAdmit);
    return rep;
}

CacheStats KvStore::cache_stats(std::size_t layer, std::size_t kv_head) const {
    const HeadState& st = states_[slot(layer, kv_head)];
    CacheStats cs;
    cs.hits = st.hits;
    cs.misses = st.misses;
    cs.requests = st.requests;
    cs.occupancy_tokens = st.occupancy_tokens;
    cs.hit_rate = st.requests ? static_cast<double>(st.hits) / static_cast<double>(st.requests) : 0.0;
    return cs;
}

void write_trace_csv(std::ostream& out, const std::vector<TraceRow>& rows) {
    out << "step,layer,kv_head,block_id,hit\n";
    for (const TraceRow& r : rows)
        out << r.step << ',' << r.layer << ',' << r.kv_head << ',' << r.block_id << ',' << (r.hit ? 1 : 0) << '\n';
}

}  // namespace pqkv
