// runtime_internal.hpp -- host-side runtime of the C++ drop-in API (not
// installed): per-thread contexts, reusable device scratch and the device
// mirrors of long-lived reference objects (PqIndex, HeadState).
#pragma once

#include <chrono>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <span>
#include <vector>

#include "pqkv/kv_store.hpp"
#include "pqkv/pq.hpp"
#include "pqkv_c.h"

namespace pqkv::detail {

// fn(begin, end) over [0, n) in chunks of >= grain on the host worker pool
// (host_pool.cpp); the calling thread takes chunks too.
void parallel_for(std::size_t n, std::size_t grain, const std::function<void(std::size_t, std::size_t)>& fn);

// Host-side phase timing of the drop-in calls (PQKV_API_PROFILE=1: per-phase
// totals in microseconds printed to stderr at exit).  Diagnostics only.
enum Phase { kSaPrep, kSaMirror, kSaCompute, kFtRank, kFtAccount, kFtEntries, kFtAdmit, kPhases };
bool api_profile();
void phase_add(Phase p, double us);
class PhaseTimer {
public:
    PhaseTimer() : on_(api_profile()) {
        if (on_) t_ = std::chrono::steady_clock::now();
    }
    void lap(Phase p) {
        if (!on_) return;
        const auto now = std::chrono::steady_clock::now();
        phase_add(p, std::chrono::duration<double, std::micro>(now - t_).count());
        t_ = now;
    }

private:
    bool on_;
    std::chrono::steady_clock::time_point t_;
};

[[noreturn]] void rethrow(int rc, const char* what);
inline void check(int rc) {
    if (rc != PQKV_OK) rethrow(rc, pqkv_last_error());
}

// Device scratch of the current API call: bump-allocated from per-thread,
// per-device buffers that only grow; valid until the next API call on this
// thread (every call ends by copying its result to the host, which
// synchronizes, so reuse across calls is safe).
class CallScratch {
public:
    CallScratch();
    ~CallScratch();
    template <typename T>
    T* alloc(std::size_t count) {
        return static_cast<T*>(raw(count * sizeof(T)));
    }
    template <typename T>
    T* upload(const T* host, std::size_t count) {
        T* d = alloc<T>(count);
        copy_h2d(d, host, count * sizeof(T));
        return d;
    }

private:
    void* raw(std::size_t bytes);
    void copy_h2d(void* d, const void* h, std::size_t bytes);
    int slot_;
    std::size_t chunk_, offset_;  // stack top when this frame opened
};

void copy_to_host(void* host, const void* dev, std::size_t bytes);

// Device view of a PqIndex: centroids [m][C][d_m] f32 + codes [rows][m] u16.
struct IndexView {
    const float* centroids;
    const std::uint16_t* codes;
    std::size_t rows;
};
IndexView mirror(const PqIndex& index);

// Device K/V of a HeadState by token id: row t at keys + t * d_h; rows of
// the ids passed to ensure_rows are resident afterwards.
struct StateView {
    const float* keys;
    const float* values;
    std::size_t d_h;
};
StateView mirror(const HeadState& state, std::size_t d_h, std::span<const std::int64_t> ids);

// Block analysis of one fetch (pqkv_block_rank).
struct BlockRanking {
    std::vector<std::uint32_t> bits;    // distinct requested tokens
    std::vector<std::uint32_t> counts;  // per block
    std::vector<std::int64_t> ranked;   // top-k_cache blocks, -1 padded
    bool requested(std::size_t id) const { return (bits[id >> 5] >> (id & 31)) & 1u; }
};
BlockRanking rank_blocks(std::span<const std::size_t> ids, std::size_t n_tokens, std::size_t block_size,
                         std::size_t k_cache);

}  // namespace pqkv::detail
