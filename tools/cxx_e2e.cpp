// cxx_e2e -- the decode loop of the reference's run_e2e (experiments.cpp:
// 197-273, data path only: evict_local_append -> pq_score_gqa -> approx_topk
// -> fetch_topk -> selective_attention per query row) written against the
// C++ drop-in API (include/pqkv/*.hpp) and timed per layer-step.  Every call
// is the reference's value-semantics API; the runtime's device mirrors keep
// the index and the K/V rows on the GPU between calls.  Prints one JSON line.
//   pqkv_cxx_e2e [heads=8] [s=32768] [g=1] [ratio=5] [steps=4]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "pqkv/attention.hpp"
#include "pqkv/kv_store.hpp"
#include "pqkv/model.hpp"
#include "pqkv/pq.hpp"
#include "pqkv/tensor.hpp"
#include "pqkv/topk.hpp"

using namespace pqkv;

int main(int argc, char** argv) {
    const std::size_t H = argc > 1 ? std::strtoul(argv[1], nullptr, 10) : 8;
    const std::size_t S = argc > 2 ? std::strtoul(argv[2], nullptr, 10) : 32768;
    const std::size_t G = argc > 3 ? std::strtoul(argv[3], nullptr, 10) : 1;
    const std::size_t ratio = argc > 4 ? std::strtoul(argv[4], nullptr, 10) : 5;
    const std::size_t steps = argc > 5 ? std::strtoul(argv[5], nullptr, 10) : 4;
    const std::size_t D = 128, n_init = 4, n_local = 64, s_mid = S - n_init - n_local;
    const std::size_t k = (S + ratio / 2) / ratio;
    std::mt19937 rng(7);
    std::normal_distribution<float> nd;
    KvStore store(1, H, 128, 4096, CachePolicy::kLru);
    std::vector<PqIndex> idx;
    std::vector<TensorF32> qs;
    auto t_build = std::chrono::steady_clock::now();
    for (std::size_t h = 0; h < H; ++h) {
        std::vector<float> kv(S * D), vv(S * D), qv(G * D);
        for (auto& x : kv) x = nd(rng);
        for (auto& x : vv) x = nd(rng);
        for (auto& x : qv) x = nd(rng);
        TensorF32 keys({S, D}, kv), vals({S, D}, vv);
        store.offload_prefill(0, h, keys, vals, SegmentConfig{n_init, n_local, k});
        TensorF32 mids({s_mid, D}, std::vector<float>(kv.begin() + n_init * D, kv.begin() + (n_init + s_mid) * D));
        idx.push_back(pq_construct(mids, PqConfig::create(2, 6, D), 10, 100 + h));
        qs.push_back(TensorF32({G, D}, qv));
    }
    const double build_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_build).count();
    double total_us = 0.0;
    std::size_t timed = 0;
    double t_evict = 0, t_score = 0, t_topk = 0, t_fetch = 0, t_attn = 0;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto us_since = [&](auto t) { return std::chrono::duration<double, std::micro>(now() - t).count(); };
    for (std::size_t step = 0; step < steps + 1; ++step) {  // step 0 warms the mirrors
        auto t0 = std::chrono::steady_clock::now();
        for (std::size_t h = 0; h < H; ++h) {
            KvEntry fresh;
            fresh.key.resize(D);
            fresh.value.resize(D);
            for (auto& x : fresh.key) x = nd(rng);
            for (auto& x : fresh.value) x = nd(rng);
            auto t = now();
            store.evict_local_append(0, h, std::move(fresh), idx[h]);
            if (step) t_evict += us_since(t);
            t = now();
            const std::vector<float> scores = pq_score_gqa(qs[h], idx[h]);
            if (step) t_score += us_since(t);
            t = now();
            std::vector<std::size_t> ids = approx_topk(scores, k);
            for (auto& id : ids) id += n_init;
            if (step) t_topk += us_since(t);
            t = now();
            const FetchReport rep = store.fetch_topk(0, h, ids, 32);
            (void)rep;
            if (step) t_fetch += us_since(t);
            t = now();
            for (std::size_t r = 0; r < G; ++r) {
                const std::vector<float> o = selective_attention({qs[h].row(r), D}, store.state(0, h), ids);
                (void)o;
            }
            if (step) t_attn += us_since(t);
        }
        const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
        if (step > 0) {
            total_us += us;
            ++timed;
        }
    }
    std::printf("{\"heads\": %zu, \"s\": %zu, \"g\": %zu, \"k\": %zu, \"steps\": %zu, \"us_per_layer_step\": %.1f, "
                "\"us_per_head_step\": %.1f, \"prefill_s\": %.3f, \"per_call_us\": {\"evict_local_append\": %.1f, "
                "\"pq_score_gqa\": %.1f, \"approx_topk\": %.1f, \"fetch_topk\": %.1f, \"selective_attention\": %.1f}}\n",
                H, S, G, k, timed, total_us / timed, total_us / timed / H, build_s, t_evict / timed / H,
                t_score / timed / H, t_topk / timed / H, t_fetch / timed / H, t_attn / timed / H);
    return 0;
}
