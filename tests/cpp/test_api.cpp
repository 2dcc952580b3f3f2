// C++ drop-in API parity: the reference's own unit-test cases (tests/*.cpp in
// the reference: test_pq, test_kmeans, test_attention, test_model), rewritten
// against include/pqkv/pqkv.hpp (every computing call runs on the GPU through
// libpqkv.so), plus call-for-call equality with the reference library
// (oracle/_ref/libpqkv_ref.so, C shim ref_*).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "pqkv/pqkv.hpp"

extern "C" {
int ref_pq_construct(const float*, size_t, size_t, size_t, size_t, size_t, uint64_t, float*, uint16_t*);
int ref_kmeans_fit(const float*, size_t, size_t, size_t, size_t, uint64_t, float*, uint64_t*, double*, size_t*);
int ref_pq_score_gqa(const float*, size_t, size_t, const float*, size_t, size_t, const uint16_t*, size_t, float*);
int ref_top_k_desc(const float*, size_t, size_t, const uint8_t*, uint64_t*);
int ref_selective_attention(const float*, const float*, const float*, size_t, size_t, size_t, size_t,
                            const uint64_t*, size_t, float*);
int ref_save_index(const char*, const float*, size_t, size_t, size_t, const uint16_t*, size_t);
int ref_load_index(const char*, size_t*, size_t*, size_t*, size_t*, float*, uint16_t*, size_t, size_t);
int ref_fetch_replay(size_t, size_t, const float*, const float*, size_t, size_t, size_t, size_t, int, size_t,
                     const uint64_t*, const uint64_t*, const uint8_t*, const float*, size_t, uint64_t*, uint64_t*,
                     size_t, size_t*);
}

using namespace pqkv;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                                  \
    do {                                                                          \
        ++g_checks;                                                               \
        if (!(c)) {                                                               \
            ++g_fail;                                                             \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);              \
        }                                                                         \
    } while (0)
template <class E, class F>
bool throws_as(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}
#define CHECK_THROWS_AS(expr, E) CHECK(throws_as<E>([&] { (void)(expr); }))
// doctest::Approx(want).epsilon(e): |a - w| < e * (1 + max(|a|, |w|))
static bool approx(double a, double w, double e) { return std::fabs(a - w) < e * (1.0 + std::max(std::fabs(a), std::fabs(w))); }

static TensorF32 random_grid(std::uint64_t seed, std::size_t r, std::size_t c, double scale = 1.0) {
    Rng rng(seed);
    std::vector<float> d(r * c);
    for (float& x : d) x = static_cast<float>(scale * rng.normal());
    return TensorF32({r, c}, std::move(d));
}
static std::vector<float> random_vec(std::uint64_t seed, std::size_t n) {
    Rng rng(seed);
    std::vector<float> v(n);
    for (float& x : v) x = static_cast<float>(rng.normal());
    return v;
}
static double dot(std::span<const float> a, std::span<const float> b) {
    double acc = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) acc += static_cast<double>(a[i]) * static_cast<double>(b[i]);
    return acc;
}

static void pq_cases() {
    PqConfig cfg = PqConfig::create(2, 6, 128);
    CHECK(cfg.d_m == 64 && cfg.n_clusters == 64 && cfg.head_dim() == 128);
    CHECK_THROWS_AS(PqConfig::create(3, 6, 128), std::invalid_argument);
    CHECK_THROWS_AS(PqConfig::create(0, 6, 128), std::invalid_argument);
    CHECK_THROWS_AS(PqConfig::create(2, 0, 128), std::invalid_argument);
    CHECK_THROWS_AS(PqConfig::create(2, 17, 128), std::invalid_argument);

    PqIndex tiny;
    tiny.cfg = PqConfig::create(2, 1, 4);
    tiny.centroids = TensorF32({2, 2, 2}, {1, 0, 0, 1, 1, 0, 0, 1});
    tiny.codes = {0, 1};
    std::vector<float> ones{1, 1, 1, 1};
    std::vector<float> sc = pq_score(ones, tiny);
    CHECK(sc.size() == 1 && sc[0] == 2.0f);
    CHECK((reconstruct(tiny, 0) == std::vector<float>{1, 0, 0, 1}));

    for (std::size_t m : {1u, 2u, 4u}) {
        TensorF32 keys = random_grid(50 + m, 96, 32);
        PqIndex index = pq_construct(keys, PqConfig::create(m, 4, 32), 10, 7);
        std::vector<float> q = random_vec(m, 32);
        std::vector<float> s = pq_score(q, index);
        CHECK(s.size() == 96);
        for (std::size_t t = 0; t < 96; ++t) CHECK(approx(s[t], dot(q, reconstruct(index, t)), 1e-5));
    }
    {
        TensorF32 keys = random_grid(3, 64, 16);
        PqIndex index = pq_construct(keys, PqConfig::create(4, 3, 16), 8, 21);
        TensorF32 queries = random_grid(11, 4, 16);
        std::vector<float> qsum(16, 0.0f);
        for (std::size_t r = 0; r < 4; ++r)
            for (std::size_t j = 0; j < 16; ++j) qsum[j] += queries.row(r)[j];
        std::vector<float> a = pq_score_gqa(queries, index), b = pq_score(qsum, index);
        for (std::size_t t = 0; t < a.size(); ++t) CHECK(approx(a[t], b[t], 1e-4));
    }
    {
        TensorF32 keys = random_grid(4, 32, 8);
        PqIndex index = pq_construct(keys, PqConfig::create(2, 3, 8), 8, 3);
        std::vector<float> q = random_vec(19, 8);
        TensorF32 qq({2, 8}, std::vector<float>(16));
        for (int j = 0; j < 8; ++j) { qq.data[j] = q[j]; qq.data[8 + j] = -q[j]; }
        for (float v : pq_score_gqa(qq, index)) CHECK(v == 0.0f);
    }
    {
        PqIndex index = pq_construct(random_grid(8, 1, 8), PqConfig::create(2, 4, 8), 5, 1);
        CHECK(index.size() == 1 && (index.codes == std::vector<std::uint16_t>{0, 0}));
    }
    {
        TensorF32 keys = random_grid(12, 16, 8);
        PqIndex index = pq_construct(keys, PqConfig::create(2, 4, 8), 10, 2);
        for (std::size_t t = 0; t < 16; ++t)
            CHECK(std::memcmp(reconstruct(index, t).data(), keys.row(t), 8 * sizeof(float)) == 0);
    }
    {
        TensorF32 keys = random_grid(23, 60, 12);
        PqIndex index = pq_construct(keys, PqConfig::create(3, 3, 12), 10, 5);
        std::size_t before = index.size();
        std::vector<float> probe(keys.row(7), keys.row(7) + 12);
        std::vector<std::uint16_t> code = pq_encode_one(probe, index);
        CHECK(code.size() == 3);
        for (auto c : code) CHECK(c < 8);
        append_code(index, code);
        CHECK(index.size() == before + 1);
        CHECK(std::memcmp(index.code_row(before), code.data(), 3 * 2) == 0);
        std::vector<float> q = random_vec(4, 12);
        CHECK(approx(pq_score(q, index)[before], dot(q, reconstruct(index, before)), 1e-5));
    }
    {
        std::vector<std::uint16_t> short_code{0}, bad{0, 2};
        CHECK_THROWS_AS(append_code(tiny, short_code), std::invalid_argument);
        CHECK_THROWS_AS(append_code(tiny, bad), std::invalid_argument);
    }
    CHECK(codes_memory_ratio(PqConfig::create(2, 6, 128), 128) == 12.0 / 2048.0);
    CHECK(codes_memory_ratio(PqConfig::create(4, 8, 128), 128) == 1.0 / 64.0);
    {
        TensorF32 keys = random_grid(5, 128, 16);
        PqConfig c = PqConfig::create(2, 5, 16);
        PqIndex a = pq_construct(keys, c, 15, 7), b = pq_construct(keys, c, 15, 7), d = pq_construct(keys, c, 15, 8);
        CHECK(a.codes == b.codes);
        CHECK(std::memcmp(a.centroids.data.data(), b.centroids.data.data(), a.centroids.data.size() * 4) == 0);
        CHECK(a.codes != d.codes);
    }
    std::vector<float> s4{0.1f, 0.9f, 0.5f, 0.9f};
    CHECK((approx_topk(s4, 2) == std::vector<std::size_t>{1, 3}));
    CHECK((approx_topk(s4, 2, {1}) == std::vector<std::size_t>{3, 2}));
}

static void topk_cases() {
    std::vector<float> s{3.0f, 1.0f, 3.0f, 0.0f};
    CHECK((top_k_desc(s, 2) == std::vector<std::size_t>{0, 2}));
    Rng rng(7);
    for (int trial = 0; trial < 20; ++trial) {
        std::vector<float> sc(100);
        for (float& x : sc) x = static_cast<float>(rng.index(17));
        std::size_t k = 1 + rng.index(99);
        std::vector<std::size_t> ids(100);
        std::iota(ids.begin(), ids.end(), 0);
        std::sort(ids.begin(), ids.end(), [&](std::size_t a, std::size_t b) { return sc[a] != sc[b] ? sc[a] > sc[b] : a < b; });
        ids.resize(k);
        CHECK(top_k_desc(sc, k) == ids);
    }
    std::vector<float> f{5, 4, 3, 2, 1};
    std::unordered_set<std::size_t> ex{0, 2};
    CHECK((top_k_desc(f, 2, ex) == std::vector<std::size_t>{1, 3}));
    CHECK(top_k_desc(f, 0).empty());
    CHECK_THROWS_AS(top_k_desc(f, 4, ex), std::invalid_argument);
    CHECK_THROWS_AS(top_k_desc(f, 6), std::invalid_argument);
}

static void kmeans_cases() {
    for (std::uint64_t seed = 0; seed < 12; ++seed) {
        KmeansResult r = kmeans_fit(random_grid(seed, 200, 4), 8, 25, seed * 11 + 1);
        CHECK(!r.inertia_trace.empty());
        for (std::size_t i = 1; i < r.inertia_trace.size(); ++i) CHECK(r.inertia_trace[i] <= r.inertia_trace[i - 1]);
        CHECK(r.iterations_run == r.inertia_trace.size() && r.iterations_run <= 25);
    }
    for (std::uint64_t seed = 0; seed < 8; ++seed) {
        KmeansResult r = kmeans_fit(random_grid(seed + 100, 64, 3), 16, 20, seed);
        std::vector<std::size_t> cnt(16, 0);
        for (auto a : r.assignments) ++cnt[a];
        for (auto c : cnt) CHECK(c > 0);
    }
    {
        TensorF32 pts({3, 2}, {0, 0, 5, 1, -2, 4});
        KmeansResult r = kmeans_fit(pts, 4, 10, 99);
        CHECK(r.inertia_trace.back() == 0.0);
        for (std::size_t i = 0; i < 3; ++i) CHECK(std::memcmp(r.centroids.row(r.assignments[i]), pts.row(i), 8) == 0);
    }
    {
        KmeansResult r = kmeans_fit(TensorF32({4, 1}, {2.0f, 2.0f, 7.0f, 7.0f}), 2, 10, 5);
        CHECK(r.inertia_trace.back() == 0.0);
        CHECK(r.assignments[0] == r.assignments[1] && r.assignments[2] == r.assignments[3]);
    }
    {
        TensorF32 pts = random_grid(77, 300, 5);
        KmeansResult a = kmeans_fit(pts, 10, 30, 1234), b = kmeans_fit(pts, 10, 30, 1234), c = kmeans_fit(pts, 10, 30, 1235);
        CHECK(a.assignments == b.assignments && a.inertia_trace == b.inertia_trace);
        CHECK(a.assignments != c.assignments);
    }
    CHECK((assign_nearest(TensorF32({2, 1}, {1.0f, 3.0f}), TensorF32({3, 1}, {0.0f, 2.0f, 2.0f})) ==
           std::vector<std::size_t>{0, 1}));
    CHECK((assign_nearest(TensorF32({1, 1}, {1.0f}), TensorF32({2, 1}, {0.0f, 2.0f})) == std::vector<std::size_t>{0}));
    TensorF32 pts({2, 2}, {0, 0, 1, 1});
    CHECK_THROWS_AS(kmeans_fit(pts, 0, 5, 1), std::invalid_argument);
    CHECK_THROWS_AS(kmeans_fit(pts, 2, 0, 1), std::invalid_argument);
    CHECK_THROWS_AS(kmeans_fit(TensorF32({2, 2, 1}, {0, 0, 1, 1}), 2, 5, 1), std::invalid_argument);
    CHECK_THROWS_AS(assign_nearest(pts, TensorF32({1, 3}, {0, 0, 0})), std::invalid_argument);
    // two blobs (test_kmeans.cpp:73-90): assignments split the blobs exactly
    Rng rng(31);
    std::vector<float> d(200 * 6);
    for (std::size_t i = 0; i < 200; ++i)
        for (std::size_t j = 0; j < 6; ++j) d[i * 6 + j] = static_cast<float>((i < 100 ? 3.0 : -3.0) + 0.4 * rng.normal());
    KmeansResult r = kmeans_fit(TensorF32({200, 6}, d), 2, 50, 17);
    for (std::size_t i = 1; i < 100; ++i) CHECK(r.assignments[i] == r.assignments[0]);
    for (std::size_t i = 101; i < 200; ++i) CHECK(r.assignments[i] == r.assignments[100]);
    CHECK(r.assignments[0] != r.assignments[100]);
}

static void attention_cases() {
    TensorF32 id({4, 4}, {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1});
    std::vector<float> q{1, 2, 3, 4};
    CHECK((exact_scores(q, id) == std::vector<float>{0.5f, 1.0f, 1.5f, 2.0f}));
    TensorF32 k23({2, 3}, {1, 2, 3, 4, 5, 6});
    std::vector<float> q2{1, 2}, q3{1, 2, 3};
    CHECK_THROWS_AS(exact_scores(q2, k23), std::invalid_argument);
    CHECK_THROWS_AS(softmax_attention(q3, k23, TensorF32({3, 3}, std::vector<float>(9, 0.0f))), std::invalid_argument);
    for (std::uint64_t seed = 0; seed < 6; ++seed) {
        TensorF32 keys = random_grid(seed, 50, 8), values = random_grid(seed + 100, 50, 8);
        std::vector<float> qq = random_vec(seed + 200, 8);
        std::vector<float> got = softmax_attention(qq, keys, values);
        long double scale = 1.0L / std::sqrt(8.0L);
        std::vector<long double> s(50);
        long double mx = -1e300L;
        for (int i = 0; i < 50; ++i) {
            long double acc = 0;
            for (int j = 0; j < 8; ++j) acc += (long double)qq[j] * keys.row(i)[j];
            s[i] = static_cast<float>(static_cast<double>(acc * scale));
            mx = std::max(mx, s[i]);
        }
        long double tot = 0;
        for (auto& v : s) { v = std::exp(v - mx); tot += v; }
        for (int j = 0; j < 8; ++j) {
            long double o = 0;
            for (int i = 0; i < 50; ++i) o += s[i] / tot * values.row(i)[j];
            CHECK(approx(got[j], (double)o, 1e-6));
        }
    }
    {
        TensorF32 keys = random_grid(7, 30, 6);
        std::vector<float> row{1.5f, -2.0f, 0.25f, 8.0f, -0.5f, 3.0f}, flat;
        for (int i = 0; i < 30; ++i) flat.insert(flat.end(), row.begin(), row.end());
        std::vector<float> ones(6, 1.0f);
        std::vector<float> out = softmax_attention(ones, keys, TensorF32({30, 6}, flat));
        for (int j = 0; j < 6; ++j) CHECK(approx(out[j], row[j], 1e-6));
    }
    CHECK((softmax_attention(std::vector<float>{0.5, 0.5, 0.5}, TensorF32({1, 3}, {4, 5, 6}), TensorF32({1, 3}, {-1, 2, 7})) ==
           std::vector<float>{-1, 2, 7}));
    for (float v : softmax_attention(random_vec(10, 4), random_grid(8, 20, 4, 100.0), random_grid(9, 20, 4))) CHECK(std::isfinite(v));
    {
        TensorF32 keys = random_grid(11, 64, 8);
        std::vector<float> qq = random_vec(12, 8);
        std::vector<float> scores = exact_scores(qq, keys);
        std::vector<std::size_t> got = exact_topk(qq, keys, 10);
        CHECK(got.size() == 10);
        float cut = scores[got.back()];
        std::size_t better = 0;
        for (float s : scores) better += s > cut;
        CHECK(better < 10);
        for (std::size_t i = 1; i < got.size(); ++i) CHECK(scores[got[i - 1]] >= scores[got[i]]);
    }
    TensorF32 keys = random_grid(21, 40, 8), values = random_grid(22, 40, 8);
    KvStore store(1, 1, 8, 4096, CachePolicy::kLru);
    store.offload_prefill(0, 0, keys, values, SegmentConfig{4, 6, 0});
    {
        std::vector<float> qq(8, 0.3f);
        std::vector<std::size_t> picked{25, 7, 18};
        std::vector<std::size_t> order{0, 1, 2, 3, 7, 18, 25, 34, 35, 36, 37, 38, 39};
        TensorF32 sk({order.size(), 8}, std::vector<float>(order.size() * 8)), sv = sk;
        for (std::size_t i = 0; i < order.size(); ++i) {
            std::copy(keys.row(order[i]), keys.row(order[i]) + 8, sk.row(i));
            std::copy(values.row(order[i]), values.row(order[i]) + 8, sv.row(i));
        }
        CHECK(selective_attention(qq, store.state(0, 0), picked) == softmax_attention(qq, sk, sv));
    }
    {
        std::vector<std::size_t> all;
        for (std::size_t id = 4; id < 34; ++id) all.push_back(id);
        std::vector<float> qq = random_vec(23, 8);
        CHECK(selective_attention(qq, store.state(0, 0), all) == softmax_attention(qq, keys, values));
    }
    {
        std::vector<float> qq(8, 0.1f);
        std::vector<std::size_t> dup{7, 7}, loc{35}, ini{1};
        CHECK_THROWS_AS(selective_attention(qq, store.state(0, 0), dup), std::invalid_argument);
        CHECK_THROWS_AS(selective_attention(qq, store.state(0, 0), loc), std::out_of_range);
        CHECK_THROWS_AS(selective_attention(qq, store.state(0, 0), ini), std::out_of_range);
    }
    {
        TensorF32 kk = random_grid(31, 24, 6), vv = random_grid(32, 24, 6), qq = random_grid(33, 3, 6);
        TensorF32 out = gqa_group_attention(qq, kk, vv);
        CHECK((out.dims == std::vector<std::size_t>{3, 6}));
        for (std::size_t r = 0; r < 3; ++r) {
            std::vector<float> want = softmax_attention({qq.row(r), 6}, kk, vv);
            CHECK(std::memcmp(out.row(r), want.data(), 24) == 0);
        }
    }
    {  // lossless fetch + evict/append code consistency (test_kv_store.cpp)
        std::vector<std::size_t> ids{10, 5, 20};
        FetchReport rep = store.fetch_topk(0, 0, ids, 4);
        for (std::size_t i = 0; i < ids.size(); ++i)
            CHECK(std::memcmp(rep.entries[i].key.data(), keys.row(ids[i]), 32) == 0 &&
                  std::memcmp(rep.entries[i].value.data(), values.row(ids[i]), 32) == 0);
        CHECK_THROWS_AS(store.fetch_topk(0, 0, std::vector<std::size_t>{2}, 4), std::out_of_range);
        TensorF32 mid({30, 8}, std::vector<float>(keys.data.begin() + 32, keys.data.begin() + 32 + 240));
        PqIndex index = pq_construct(mid, PqConfig::create(2, 3, 8), 10, 4);
        KvEntry fresh{random_vec(50, 8), random_vec(51, 8)};
        std::size_t ev = store.evict_local_append(0, 0, fresh, index);
        CHECK(ev == 34 && index.size() == 31);
        CHECK((std::vector<std::uint16_t>(index.code_row(30), index.code_row(30) + 2) ==
               pq_encode_one(std::vector<float>(keys.row(34), keys.row(34) + 8), index)));
        CHECK(store.state(0, 0).total_tokens == 41 && store.state(0, 0).middle.count(34) == 1);
    }
}

static void reference_equality() {
    TensorF32 keys = random_grid(900, 2048, 128);
    PqIndex idx = pq_construct(keys, PqConfig::create(2, 6, 128), 10, 4242);
    std::vector<float> cen(2 * 64 * 64);
    std::vector<std::uint16_t> codes(2048 * 2);
    CHECK(ref_pq_construct(keys.data.data(), 2048, 128, 2, 6, 10, 4242, cen.data(), codes.data()) == 0);
    CHECK(idx.codes == codes);
    CHECK(std::memcmp(idx.centroids.data.data(), cen.data(), cen.size() * 4) == 0);
    TensorF32 q = random_grid(901, 4, 128);
    std::vector<float> s = pq_score_gqa(q, idx), rs(2048);
    CHECK(ref_pq_score_gqa(q.data.data(), 4, 128, cen.data(), 2, 64, codes.data(), 2048, rs.data()) == 0);
    CHECK(std::memcmp(s.data(), rs.data(), rs.size() * 4) == 0);
    std::vector<std::size_t> ids = approx_topk(s, 410);
    std::vector<uint64_t> rid(410);
    CHECK(ref_top_k_desc(rs.data(), 2048, 410, nullptr, rid.data()) == 0);
    CHECK(std::equal(ids.begin(), ids.end(), rid.begin()));
    TensorF32 pts = random_grid(902, 3000, 16);
    KmeansResult km = kmeans_fit(pts, 64, 20, 77);
    std::vector<float> rc(64 * 16);
    std::vector<uint64_t> ra(3000);
    std::vector<double> rt(20);
    size_t rit = 0;
    CHECK(ref_kmeans_fit(pts.data.data(), 3000, 16, 64, 20, 77, rc.data(), ra.data(), rt.data(), &rit) == 0);
    CHECK(km.iterations_run == rit);
    CHECK(std::equal(km.assignments.begin(), km.assignments.end(), ra.begin()));
    CHECK(std::memcmp(km.inertia_trace.data(), rt.data(), rit * 8) == 0);
    CHECK(std::memcmp(km.centroids.data.data(), rc.data(), rc.size() * 4) == 0);
    // selective attention vs the reference within the fp64 path's exp tolerance
    TensorF32 kv = random_grid(903, 300, 32), vv = random_grid(904, 300, 32);
    KvStore st(1, 1, 64, 4096, CachePolicy::kLfu);
    st.offload_prefill(0, 0, kv, vv, SegmentConfig{4, 16, 0});
    std::vector<std::size_t> sel{10, 200, 57, 133, 4, 279};
    std::vector<uint64_t> sel64(sel.begin(), sel.end());
    std::vector<float> qq = random_vec(905, 32), want(32);
    std::vector<float> got = selective_attention(qq, st.state(0, 0), sel);
    CHECK(ref_selective_attention(qq.data(), kv.data.data(), vv.data.data(), 32, 300, 4, 16, sel64.data(), sel.size(),
                                  want.data()) == 0);
    for (int j = 0; j < 32; ++j) CHECK(approx(got[j], want[j], 1e-6));
}

// .pqt index files: ours and the reference's are interchangeable
static void io_cases() {
    TensorF32 keys = random_grid(77, 600, 16);
    PqIndex idx = pq_construct(keys, PqConfig::create(2, 3, 16), 5, 3);
    const std::string a = "/tmp/pqkv_io_ours.pqt", b = "/tmp/pqkv_io_ref.pqt";
    save_index(a, idx);
    size_t m = 0, C = 0, d_m = 0, n = 0;
    std::vector<float> cen(2 * 8 * 8);
    std::vector<uint16_t> codes(600 * 2);
    CHECK(ref_load_index(a.c_str(), &m, &C, &d_m, &n, cen.data(), codes.data(), cen.size(), codes.size()) == 0);
    CHECK(m == 2 && C == 8 && d_m == 8 && n == 600);
    CHECK(cen == idx.centroids.data && codes == idx.codes);
    CHECK(ref_save_index(b.c_str(), idx.centroids.data.data(), 2, 8, 8, idx.codes.data(), 600) == 0);
    PqIndex back = load_index(b);
    CHECK(back.codes == idx.codes && back.centroids.data == idx.centroids.data && back.cfg.b == 3 &&
          back.centroids.dims == idx.centroids.dims);
    TensorF32 t = random_grid(78, 4, 9);
    save_tensor(a, t);
    TensorF32 t2 = load_tensor(a);
    CHECK(t2.dims == t.dims && t2.data == t.data);
    CHECK_THROWS_AS(load_index(a), std::runtime_error);  // a 2-d tensor is not a centroid grid
    CHECK_THROWS_AS(load_tensor("/tmp/pqkv_io_missing.pqt"), std::runtime_error);
    std::remove(a.c_str());
    std::remove(b.c_str());
}

// Block-cache accounting (test_kv_store.cpp cases + a randomized replay
// against the reference library, appends included).
static void kv_cache_cases() {
    {  // tokens sharing a block count as one lookup
        TensorF32 k = random_grid(4, 256, 4), v = random_grid(5, 256, 4);
        KvStore store(1, 1, 128, 1024, CachePolicy::kLru);
        store.offload_prefill(0, 0, k, v, SegmentConfig{8, 8, 0});
        FetchReport rep = store.fetch_topk(0, 0, std::vector<std::size_t>{100, 101, 200, 100}, 4);
        CHECK(rep.entries.size() == 4);
        CHECK(rep.hits + rep.misses == 2);
        CHECK(rep.bytes_from_slow_tier == 3 * 2 * 2 * 4);
        CHECK(store.cache_stats(0, 0).requests == 2);
    }
    {  // a warm block hits on the second request
        TensorF32 k = random_grid(6, 256, 4), v = random_grid(7, 256, 4);
        KvStore store(1, 1, 32, 1024, CachePolicy::kLru);
        store.offload_prefill(0, 0, k, v, SegmentConfig{8, 8, 0});
        CHECK(store.fetch_topk(0, 0, std::vector<std::size_t>{40}, 1).misses == 1);
        FetchReport again = store.fetch_topk(0, 0, std::vector<std::size_t>{40}, 1);
        CHECK(again.hits == 1);
        CHECK(again.bytes_from_slow_tier == 0);
    }
    {  // zero capacity never caches
        TensorF32 k = random_grid(8, 128, 4), v = random_grid(9, 128, 4);
        KvStore store(1, 1, 16, 0, CachePolicy::kLfu);
        store.offload_prefill(0, 0, k, v, SegmentConfig{4, 4, 0});
        for (int i = 0; i < 5; ++i) {
            FetchReport rep = store.fetch_topk(0, 0, std::vector<std::size_t>{60}, 2);
            CHECK(rep.hits == 0 && rep.misses == 1);
        }
        CHECK(store.cache_stats(0, 0).occupancy_tokens == 0);
        CHECK(store.fetch_topk(0, 0, std::vector<std::size_t>{}, 1).entries.empty());
    }
    {  // the cache keeps the most requested blocks, ties toward the lower id
        TensorF32 k = random_grid(10, 512, 4), v = random_grid(11, 512, 4);
        KvStore store(1, 1, 64, 4096, CachePolicy::kLru);
        store.offload_prefill(0, 0, k, v, SegmentConfig{8, 8, 0});
        store.enable_trace();
        store.fetch_topk(0, 0, std::vector<std::size_t>{130, 140, 70, 280}, 2);
        const HeadState& st = store.state(0, 0);
        CHECK(st.cache.size() == 2 && st.cache.contains(2) && st.cache.contains(1) && !st.cache.contains(4));
        CHECK(store.trace().size() == 3 && store.trace()[0].block_id == 1 && store.trace()[2].block_id == 4);
    }
    {  // eviction follows the policy
        auto run = [&](CachePolicy policy) {
            TensorF32 k = random_grid(12, 10, 4), v = random_grid(13, 10, 4);
            KvStore store(1, 1, 1, 2, policy);
            store.offload_prefill(0, 0, k, v, SegmentConfig{0, 1, 0});
            auto touch = [&](std::size_t id) {
                return store.fetch_topk(0, 0, std::vector<std::size_t>{id}, 1).hits == 1;
            };
            touch(0);
            touch(0);
            touch(1);
            touch(2);
            return touch(0);
        };
        CHECK(run(CachePolicy::kLru) == false);
        CHECK(run(CachePolicy::kLfu) == true);
    }
    // randomized replay against the reference library
    for (int trial = 0; trial < 6; ++trial) {
        const std::size_t s = 700, d = 8, n_init = 4, n_local = 16;
        const std::size_t block = trial % 3 == 0 ? 16 : (trial % 3 == 1 ? 32 : 7);
        const std::size_t cap = trial < 3 ? 96 : 200;
        const bool lfu = trial & 1;
        const std::size_t k_cache = 1 + trial % 4, n_req = 120;
        TensorF32 k = random_grid(100 + trial, s, d), v = random_grid(200 + trial, s, d);
        Rng rng(300 + trial);
        std::vector<uint64_t> offs{0}, ids;
        std::vector<uint8_t> app(n_req);
        std::vector<float> fresh(n_req * 2 * d);
        for (float& x : fresh) x = static_cast<float>(rng.normal());
        KvStore store(1, 1, block, cap, lfu ? CachePolicy::kLfu : CachePolicy::kLru);
        store.offload_prefill(0, 0, k, v, SegmentConfig{n_init, n_local, 0});
        TensorF32 mid({s - n_init - n_local, d},
                      std::vector<float>(k.data.begin() + n_init * d, k.data.begin() + (s - n_local) * d));
        PqIndex index = pq_construct(mid, PqConfig::create(2, 3, d), 4, 9);
        std::size_t mid_end = s - n_local;  // middle ids [n_init, mid_end)
        std::vector<uint64_t> got;
        for (std::size_t r = 0; r < n_req; ++r) {
            app[r] = rng.index(4) == 0;
            if (app[r]) {
                KvEntry e;
                e.key.assign(fresh.begin() + r * 2 * d, fresh.begin() + r * 2 * d + d);
                e.value.assign(fresh.begin() + r * 2 * d + d, fresh.begin() + (r + 1) * 2 * d);
                store.evict_local_append(0, 0, std::move(e), index);
                ++mid_end;
            }
            std::size_t n = 1 + rng.index(12);
            std::vector<std::size_t> req;
            std::size_t hot = n_init + rng.index(mid_end - n_init);
            for (std::size_t i = 0; i < n; ++i) {
                // clustered around a hot token (repeats and the newest rows included)
                std::size_t id = rng.index(3) == 0 ? mid_end - 1 - rng.index(std::min<std::size_t>(8, mid_end - n_init))
                                                  : hot + rng.index(40);
                req.push_back(std::min(id, mid_end - 1));
            }
            for (std::size_t id : req) ids.push_back(id);
            offs.push_back(ids.size());
            FetchReport rep = store.fetch_topk(0, 0, req, k_cache);
            got.push_back(rep.hits);
            got.push_back(rep.misses);
            got.push_back(rep.bytes_from_slow_tier);
        }
        CacheStats cs = store.cache_stats(0, 0);
        got.push_back(cs.hits);
        got.push_back(cs.misses);
        got.push_back(cs.requests);
        got.push_back(cs.occupancy_tokens);
        std::vector<uint64_t> want(3 * n_req + 4), cache_ids(4096);
        size_t n_cached = 0;
        CHECK(ref_fetch_replay(s, d, k.data.data(), v.data.data(), n_init, n_local, block, cap, lfu ? 1 : 0, n_req,
                               offs.data(), ids.data(), app.data(), fresh.data(), k_cache, want.data(),
                               cache_ids.data(), cache_ids.size(), &n_cached) == 0);
        CHECK(got == want);
        std::vector<uint64_t> mine;
        for (const auto& kv : store.state(0, 0).cache) mine.push_back(kv.first);
        CHECK(mine.size() == n_cached && std::equal(mine.begin(), mine.end(), cache_ids.begin()));
        CHECK(cs.hit_rate == (cs.requests ? static_cast<double>(cs.hits) / cs.requests : 0.0));
    }
}

int main() {
    struct { const char* name; void (*fn)(); } suites[] = {
        {"pq", pq_cases}, {"topk", topk_cases}, {"kmeans", kmeans_cases}, {"attention", attention_cases},
        {"reference_equality", reference_equality}, {"kv_cache", kv_cache_cases}, {"io", io_cases}};
    for (auto& s : suites) {
        int before = g_fail;
        try {
            s.fn();
        } catch (const std::exception& e) {
            ++g_fail;
            std::printf("FAIL %s threw: %s\n", s.name, e.what());
        }
        std::printf("suite %s: %s\n", s.name, g_fail == before ? "ok" : "FAILED");
    }
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
