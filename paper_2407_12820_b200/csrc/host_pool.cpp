// host_pool.cpp -- a small persistent worker pool for the host-side copies
// the drop-in API's value semantics require (FetchReport::entries, cache
// snapshots: thousands of KvEntry allocations + copies per fetch).  The
// caller runs chunks too; a second concurrent caller runs serially rather
// than queueing behind the first.
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <exception>
#include <mutex>
#include <thread>
#include <vector>

#include "runtime_internal.hpp"

namespace pqkv::detail {
namespace {

class Pool {
public:
    Pool() {
        unsigned n = std::max(1u, std::thread::hardware_concurrency());
        if (const char* e = std::getenv("PQKV_HOST_THREADS")) n = std::max(1, std::atoi(e));
        n = std::min(n, 16u);
        for (unsigned i = 1; i < n; ++i) workers_.emplace_back([this] { work(); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }

    std::size_t width() const { return workers_.size() + 1; }

    void run(std::size_t n_chunks, const std::function<void(std::size_t)>& fn) {
        std::unique_lock<std::mutex> busy(busy_, std::try_to_lock);
        if (!busy.owns_lock() || workers_.empty() || n_chunks < 2) {
            for (std::size_t c = 0; c < n_chunks; ++c) fn(c);
            return;
        }
        {
            std::lock_guard<std::mutex> g(m_);
            fn_ = &fn;
            n_chunks_ = n_chunks;
            next_.store(0);
            pending_ = workers_.size();
            ++gen_;
        }
        cv_.notify_all();
        drain();
        std::unique_lock<std::mutex> g(m_);
        done_.wait(g, [&] { return pending_ == 0; });
        fn_ = nullptr;
    }

private:
    void drain() {
        for (std::size_t c; (c = next_.fetch_add(1)) < n_chunks_;) (*fn_)(c);
    }
    void work() {
        std::uint64_t seen = 0;
        while (true) {
            {
                std::unique_lock<std::mutex> g(m_);
                cv_.wait(g, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
            }
            drain();
            std::lock_guard<std::mutex> g(m_);
            if (--pending_ == 0) done_.notify_one();
        }
    }

    std::vector<std::thread> workers_;
    std::mutex m_, busy_;
    std::condition_variable cv_, done_;
    const std::function<void(std::size_t)>* fn_ = nullptr;
    std::size_t n_chunks_ = 0, pending_ = 0;
    std::atomic<std::size_t> next_{0};
    std::uint64_t gen_ = 0;
    bool stop_ = false;
};

Pool& pool() {
    static Pool p;
    return p;
}

}  // namespace

void parallel_for(std::size_t n, std::size_t grain, const std::function<void(std::size_t, std::size_t)>& fn) {
    if (n == 0) return;
    grain = std::max<std::size_t>(grain, 1);
    if (n <= grain) {
        fn(0, n);
        return;
    }
    Pool& p = pool();
    const std::size_t chunk = std::max(grain, (n + 4 * p.width() - 1) / (4 * p.width()));
    const std::size_t n_chunks = (n + chunk - 1) / chunk;
    // the first exception of any chunk is rethrown on the calling thread
    std::exception_ptr err;
    std::mutex err_m;
    p.run(n_chunks, [&](std::size_t c) {
        try {
            fn(c * chunk, std::min(n, (c + 1) * chunk));
        } catch (...) {
            std::lock_guard<std::mutex> g(err_m);
            if (!err) err = std::current_exception();
        }
    });
    if (err) std::rethrow_exception(err);
}

}  // namespace pqkv::detail
