// select_common.cuh -- device building blocks shared by the selection
// kernels (select.cu) and the fused decode kernel (attend.cu).
#pragma once

#include "common.cuh"

namespace pqkv_dev {

constexpr int NB = 2048;  // bins of the two 11-bit radix digits

// Phase timestamps (profiling): tp[ph] = clock64() from thread 0 when tp != null.
#define PQKV_T(ph) do { if (tp && threadIdx.x == 0) tp[ph] = clock64(); } while (0)

// Builds T[j][c] (pq.cpp:113-126, rows accumulated as in pq.cpp:157-159).
// One thread per (j, c); the t-chain stays sequential (reference order) while
// the centroid row is prefetched 16 floats at a time so the chain is not
// serialised on L2 latency.
template <int DM>
__device__ __forceinline__ void lut_entry_vec(double* lut, const float* q, const float* cen, int g, int d_h,
                                              int e, int j) {
    // centroid row and query slice as 128-bit loads, all issued before the
    // sequential fp64 chain (t ascending, products exact => DFMA == mul+add)
    const float4* cc4 = reinterpret_cast<const float4*>(cen + (long long)e * DM);
    float4 cv[DM / 4];
#pragma unroll
    for (int u = 0; u < DM / 4; ++u) cv[u] = __ldg(cc4 + u);
    double t = 0.0;
    for (int r = 0; r < g; ++r) {
        const float4* q4 = reinterpret_cast<const float4*>(q + (long long)r * d_h + j * DM);
        float4 qv[DM / 4];
#pragma unroll
        for (int u = 0; u < DM / 4; ++u) qv[u] = q4[u];  // q may be in shared memory
        double acc = 0.0;
#pragma unroll
        for (int u = 0; u < DM / 4; ++u) {
            acc = __fma_rn((double)qv[u].x, (double)cv[u].x, acc);
            acc = __fma_rn((double)qv[u].y, (double)cv[u].y, acc);
            acc = __fma_rn((double)qv[u].z, (double)cv[u].z, acc);
            acc = __fma_rn((double)qv[u].w, (double)cv[u].w, acc);
        }
        t = __dadd_rn(t, acc);
    }
    lut[e] = t;
}

// g > 1: the per-query dot products are independent chains (only their sum
// t = ((0 + d_0) + d_1) + ... is ordered), so up to four run interleaved --
// the serial latency is one d_m-long chain instead of g of them.
template <int DM>
__device__ __forceinline__ void lut_entry_multi(double* lut, const float* q, const float* cen, int g, int d_h,
                                                int e, int j) {
    const float4* cc4 = reinterpret_cast<const float4*>(cen + (long long)e * DM);
    double t = 0.0;
    for (int r0 = 0; r0 < g; r0 += 4) {
        const int rn = min(4, g - r0);
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 4
        for (int u = 0; u < DM / 4; ++u) {
            const float4 cv = __ldg(cc4 + u);
#pragma unroll
            for (int rr = 0; rr < 4; ++rr) {
                if (rr < rn) {
                    const float4 qv = reinterpret_cast<const float4*>(q + (long long)(r0 + rr) * d_h + j * DM)[u];
                    acc[rr] = __fma_rn((double)qv.x, (double)cv.x, acc[rr]);
                    acc[rr] = __fma_rn((double)qv.y, (double)cv.y, acc[rr]);
                    acc[rr] = __fma_rn((double)qv.z, (double)cv.z, acc[rr]);
                    acc[rr] = __fma_rn((double)qv.w, (double)cv.w, acc[rr]);
                }
            }
        }
#pragma unroll
        for (int rr = 0; rr < 4; ++rr)
            if (rr < rn) t = __dadd_rn(t, acc[rr]);
    }
    lut[e] = t;
}

// One ADC table entry e (pq.cpp:113-126; subspace j = e / C), written to
// lut[e] -- lut may be a distributed-shared-memory pointer.
__device__ __forceinline__ void lut_entry(double* lut, const float* q, const float* cen, int g, int d_h, int m,
                                          int C, int e) {
    const int dm = d_h / m, j = e / C;
    const bool aligned = ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(cen)) & 15) == 0 &&
                         (d_h % 4) == 0;
    if (aligned && dm == 64) {
        if (g > 1) lut_entry_multi<64>(lut, q, cen, g, d_h, e, j);
        else lut_entry_vec<64>(lut, q, cen, g, d_h, e, j);
        return;
    }
    if (aligned && dm == 32) {
        if (g > 1) lut_entry_multi<32>(lut, q, cen, g, d_h, e, j);
        else lut_entry_vec<32>(lut, q, cen, g, d_h, e, j);
        return;
    }
    const float* cc = cen + (long long)e * dm;
    double t = 0.0;
    for (int r = 0; r < g; ++r) {
        const float* qq = q + (long long)r * d_h + j * dm;
        double acc = 0.0;
        for (int u = 0; u < dm; ++u) acc = __fma_rn((double)qq[u], (double)__ldg(cc + u), acc);
        t = __dadd_rn(t, acc);
    }
    lut[e] = t;
}

// LUT entry from a centroid row staged in shared memory (16-byte chunk u of
// row e at e * DM/4 + (u ^ (e & 7)): the 8 lanes of a 128-bit access phase
// hit 8 distinct bank groups).  Same products, same order as lut_entry_vec /
// lut_entry_multi.
template <int DM>
__device__ __forceinline__ void lut_entry_staged(double* lut, const float* q, const float4* stage, int g, int d_h,
                                                 int e, int j) {
    const float4* row = stage + (long long)e * (DM / 4);
    double t = 0.0;
    if (g == 1) {  // one chain; a partial unroll keeps the query loads from
                   // crowding the registers (the fused decode runs at 64)
        const float4* q4 = reinterpret_cast<const float4*>(q + j * DM);
        double acc = 0.0;
#pragma unroll 4
        for (int u = 0; u < DM / 4; ++u) {
            const float4 cv = row[u ^ (e & 7)], qv = q4[u];
            acc = __fma_rn((double)qv.x, (double)cv.x, acc);
            acc = __fma_rn((double)qv.y, (double)cv.y, acc);
            acc = __fma_rn((double)qv.z, (double)cv.z, acc);
            acc = __fma_rn((double)qv.w, (double)cv.w, acc);
        }
        lut[e] = __dadd_rn(t, acc);
        return;
    }
    for (int r0 = 0; r0 < g; r0 += 4) {
        const int rn = min(4, g - r0);
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 4
        for (int u = 0; u < DM / 4; ++u) {
            const float4 cv = row[u ^ (e & 7)];
#pragma unroll
            for (int rr = 0; rr < 4; ++rr) {
                if (rr < rn) {
                    const float4 qv = reinterpret_cast<const float4*>(q + (long long)(r0 + rr) * d_h + j * DM)[u];
                    acc[rr] = __fma_rn((double)qv.x, (double)cv.x, acc[rr]);
                    acc[rr] = __fma_rn((double)qv.y, (double)cv.y, acc[rr]);
                    acc[rr] = __fma_rn((double)qv.z, (double)cv.z, acc[rr]);
                    acc[rr] = __fma_rn((double)qv.w, (double)cv.w, acc[rr]);
                }
            }
        }
#pragma unroll
        for (int rr = 0; rr < 4; ++rr)
            if (rr < rn) t = __dadd_rn(t, acc[rr]);
    }
    lut[e] = t;
}

// `stage` (nullable, 16-byte aligned, m*C*d_m floats): the centroid table is
// first copied there with coalesced cp.async (a lane per 16-byte chunk) --
// one CTA pulling a 32 KB table with per-lane row loads (256 B apart) was the
// slowest part of the pair select (tools/microbench/lut_probe.cu: 3.2 ->
// 1.9 us warm).
// Whether build_lut stages the centroid table (in `stage`) for these inputs.
__device__ __forceinline__ bool lut_staged(const float* q, const float* cen, int d_h, int m, const void* stage) {
    const int dm = d_h / m;
    return stage && (dm == 64 || dm == 32) &&
           ((reinterpret_cast<uintptr_t>(cen) | reinterpret_cast<uintptr_t>(q)) & 15) == 0 && (d_h % 4) == 0;
}

// The centroid-table staging copies of build_lut (cp.async, one commit group).
__device__ inline void stage_centroids(const float* cen, int d_h, int m, int C, float4* stage) {
    const int cpr = d_h / m / 4, n = m * C * cpr;  // 16-byte chunks per row, in total
    for (int f = threadIdx.x; f < n; f += blockDim.x) {
        const int e = f / cpr, u = f % cpr;
        cp_async16(stage + (long long)e * cpr + (u ^ (e & 7)), cen + 4LL * f);
    }
    cp_async_commit();
}

// prestaged: the caller already issued stage_centroids (e.g. before its
// griddepcontrol.wait: the centroids are not written by a kernel that lets
// this one launch early)
__device__ inline void build_lut(double* lut, const float* q, const float* cen, int g, int d_h, int m,
                          int C, float4* stage = nullptr, bool prestaged = false) {
    const int dm = d_h / m;
    if (lut_staged(q, cen, d_h, m, stage)) {
        if (!prestaged) stage_centroids(cen, d_h, m, C, stage);
        cp_async_wait_all();
        __syncthreads();
        for (int e = threadIdx.x; e < m * C; e += blockDim.x) {
            if (dm == 64) lut_entry_staged<64>(lut, q, stage, g, d_h, e, e / C);
            else lut_entry_staged<32>(lut, q, stage, g, d_h, e, e / C);
        }
        __syncthreads();  // the stage may be reused right after
        return;
    }
    const int d_m = d_h / m;
    const bool aligned = ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(cen)) & 15) == 0 &&
                         (d_h % 4) == 0;
    if (aligned && (d_m == 64 || d_m == 32)) {
        for (int e = threadIdx.x; e < m * C; e += blockDim.x) {
            if (g > 1) {
                if (d_m == 64) lut_entry_multi<64>(lut, q, cen, g, d_h, e, e / C);
                else lut_entry_multi<32>(lut, q, cen, g, d_h, e, e / C);
            } else if (d_m == 64) {
                lut_entry_vec<64>(lut, q, cen, g, d_h, e, e / C);
            } else {
                lut_entry_vec<32>(lut, q, cen, g, d_h, e, e / C);
            }
        }
        return;
    }
    for (int e = threadIdx.x; e < m * C; e += blockDim.x) {
        const int j = e / C;
        const float* cc = cen + (long long)e * d_m;
        double t = 0.0;
        for (int r0 = 0; r0 < g; r0 += 4) {
            const int rn = min(4, g - r0);
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            for (int t0 = 0; t0 < d_m; t0 += 16) {
                float cv[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) cv[u] = (t0 + u < d_m) ? __ldg(cc + t0 + u) : 0.0f;
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    if (r >= rn) break;
                    const float* qq = q + (long long)(r0 + r) * d_h + j * d_m + t0;
                    float qv[16];
#pragma unroll
                    for (int u = 0; u < 16; ++u) qv[u] = (t0 + u < d_m) ? qq[u] : 0.0f;
#pragma unroll
                    for (int u = 0; u < 16; ++u)
                        if (t0 + u < d_m) acc[r] = __fma_rn((double)qv[u], (double)cv[u], acc[r]);
                }
            }
#pragma unroll
            for (int r = 0; r < 4; ++r)
                if (r < rn) t = __dadd_rn(t, acc[r]);
        }
        lut[e] = t;
    }
}

// Block-wide exclusive scan (NT threads) of one u32 per thread.
template <int NT>
__device__ uint32_t block_excl_scan(uint32_t v, uint32_t* wsum, uint32_t* total) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < NW ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(FULL, w, o);
            if (lane >= o) w += y;
        }
        if (lane < NW) wsum[lane] = w;  // inclusive
    }
    __syncthreads();
    uint32_t before = (warp ? wsum[warp - 1] : 0) + x - v;
    if (total) *total = wsum[NW - 1];
    __syncthreads();
    return before;
}

// Finds the digit holding the k_rem-th largest element of hist[0..nb).
// Returns (digit, count strictly above it) via out[0], out[1].
template <int NT>
__device__ void find_digit(const uint32_t* hist, int nb, uint32_t k_rem, uint32_t* wsum,
                           uint32_t* out) {
    const int per = nb / NT;  // bins per thread (>= 1)
    const int hi = nb - per * (int)threadIdx.x;  // this thread owns [hi-per, hi), from the top
    uint32_t local = 0;
    for (int b = hi - 1; b >= hi - per; --b) local += hist[b];
    uint32_t above = block_excl_scan<NT>(local, wsum, nullptr);
    if (above < k_rem && k_rem <= above + local) {
        uint32_t acc = above;
        for (int b = hi - 1; b >= hi - per; --b) {
            if (k_rem <= acc + hist[b]) {
                out[0] = (uint32_t)b;
                out[1] = acc;
                break;
            }
            acc += hist[b];
        }
    }
    __syncthreads();
}


// Where pair_select stages the centroid table: hist[] .. lst[] (2 NB + C^2
// words, unused before its compaction) when it fits.
__device__ __forceinline__ float4* pair_lut_stage(int C, int d_h, uint32_t* hist) {
    return 2 * C * (d_h / 2) <= 2 * NB + C * C ? reinterpret_cast<float4*>(hist) : nullptr;
}

// Pair-level exact top-k for one head (m == 2): builds the ADC table, the
// keys of the code pairs that occur (thist > 0), selects the k-th
// largest key weighted by the pair histogram thist, classifies every pair
// (0 below or absent, 1 above, 2 equal) into cls[], and finds the
// PQKV_TUPLE_CHUNK chunk c* holding the k_rem-th equal token in id order plus
// how many of c*'s equal tokens are taken.  Pairs that never occur are
// compacted away first (block scan), so the select costs O(distinct pairs),
// not O(C^2).  On return (after a barrier) sh[3] = c*, sh[4] = take,
// sh[5] = K*.  All scratch is shared memory owned by the caller (see
// pair_select_scratch): lut[2C] f64, hist[NB], cnt[NB], lst[C*C], ceq[n_chunks]
// u32, wsum[64], sh[8].  Requires C*C <= NT*WMAX and thist entries below
// 2^(32 - log2(C*C)) (a list entry packs pair << wbits | weight).
// tkey_out (nullable) receives the key of every pair.
template <int NT, int WMAX>
__device__ void pair_select(const float* q, int g, int d_h, const float* cen, int C,
                            const uint32_t* thist, const uint16_t* chist, int n_chunks, int k,
                            double* lut, uint32_t* hist, uint32_t* cnt, uint32_t* lst, uint32_t* ceq,
                            uint32_t* wsum, uint32_t* sh, uint8_t* cls, uint32_t* tkey_out,
                            unsigned long long* tp = nullptr, bool cen_prestaged = false) {
    const int tid = threadIdx.x, C2 = C * C, lane = tid & 31, warp = tid >> 5;
    const int wbits = 32 - (32 - __clz((unsigned)(C2 - 1) | 1u));  // weight bits of a list entry
    const uint32_t wmask = (1u << wbits) - 1u;
    // pair weights: loaded once into registers (WMAX * NT >= C2), in flight
    // while the ADC table is built
    PQKV_T(0);
    uint32_t w[WMAX];
#pragma unroll
    for (int u = 0; u < WMAX; ++u) {
        const int t = tid + u * NT;
        w[u] = t < C2 ? __ldg(thist + t) : 0u;
    }
    // the centroid table is staged in hist[] .. lst[] (2 NB + C^2 words, not
    // used before the compaction below) when it fits
    build_lut(lut, q, cen, g, d_h, 2, C, pair_lut_stage(C, d_h, hist), cen_prestaged);
    for (int c = tid; c < n_chunks; c += NT) ceq[c] = 0;
    for (int e = tid; e < (C2 + 3) / 4; e += NT) reinterpret_cast<uint32_t*>(cls)[e] = 0u;
    PQKV_T(1);
    // ---- compaction: lst[] = (pair << wbits | weight) of the pairs present ----
    uint32_t nz = 0;
#pragma unroll
    for (int u = 0; u < WMAX; ++u) nz += w[u] != 0u;
    uint32_t nnz;
    uint32_t pos = block_excl_scan<NT>(nz, wsum, &nnz);  // ends with a barrier
#pragma unroll
    for (int u = 0; u < WMAX; ++u)
        if (w[u]) lst[pos++] = (uint32_t)(tid + u * NT) << wbits | w[u];
    for (int b = tid; b < NB; b += NT) { hist[b] = 0; cnt[b] = 0; }
    __syncthreads();
    PQKV_T(2);
    // this thread's items: lst[tid + u*NT], u < per (block-uniform)
    const int per = (int)((nnz + NT - 1) / NT);
    uint32_t it[WMAX], kr[WMAX];
    uint32_t kmin = 0xffffffffu, kmax = 0u;
#pragma unroll
    for (int u = 0; u < WMAX; ++u) {
        it[u] = 0u;
        kr[u] = 0u;
        if (u < per) {
            const int i = tid + u * NT;
            if (i < (int)nnz) {
                it[u] = lst[i];
                const int t = (int)(it[u] >> wbits);
                double acc = __dadd_rn(0.0, lut[t / C]);
                acc = __dadd_rn(acc, lut[C + t % C]);
                kr[u] = score_key((float)acc);
                kmin = min(kmin, kr[u]);
                kmax = max(kmax, kr[u]);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(FULL, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(FULL, kmax, o));
    }
    if (lane == 0) { wsum[warp] = kmin; wsum[32 + warp] = kmax; }
    if (tkey_out)
        for (int t = tid; t < C2; t += NT) {
            double acc = __dadd_rn(0.0, lut[t / C]);
            acc = __dadd_rn(acc, lut[C + t % C]);
            tkey_out[t] = score_key((float)acc);
        }
    __syncthreads();
    if (tid < 32) {
        uint32_t a = lane < NT / 32 ? wsum[lane] : 0xffffffffu, z = lane < NT / 32 ? wsum[32 + lane] : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a = min(a, __shfl_xor_sync(FULL, a, o));
            z = max(z, __shfl_xor_sync(FULL, z, o));
        }
        if (lane == 0) { sh[6] = a; sh[7] = z; }
    }
    __syncthreads();
    kmin = sh[6];
    kmax = sh[7];
    PQKV_T(3);
    // ---- weighted select over the present pair keys ----
    // Each pass bins the candidate pairs linearly by score value over the
    // candidates' [lo, hi] (a monotone map, so bins are ordered like keys;
    // score-value bins spread the bulk of a score distribution, where the
    // k-th largest sits, far better than key-bit digits, which split it by
    // sign and exponent), finds the bin holding the k_rem-th largest weight
    // and keeps its pairs.  It ends when one pair is left, when all the
    // candidates share one key, or -- usually after the first pass -- when
    // at most 32 pairs are left: one warp sorts them and walks their weights.
    // On exit k_rem is the rank of the threshold among tokens with key K*.
    uint32_t k_rem = (uint32_t)k;
    uint32_t kstar = 0;
    uint32_t alive = 0;  // bit u: item u is still a candidate
#pragma unroll
    for (int u = 0; u < WMAX; ++u)
        if (u < per && (it[u] & wmask)) alive |= 1u << u;
    double lo = (double)key_score(kmin), hi = (double)key_score(kmax);
    // The first pass bins on the order-preserving key bits -- the top 11
    // bits of key - kmin over this head's [kmin, kmax] -- i.e. on sign,
    // exponent and leading mantissa bits: a fixed fraction of a binade per bin
    // (1/64 for a 36-binade range) wherever the bulk of the scores sits.
    // Value-linear bins put a heavy-tailed bulk (powerlaw keys: a few pair
    // scores near 8, thousands near 1e-3) into one bin, whose items then also
    // collide on one shared-memory atomic.  Later passes bin the survivors
    // linearly by value over their own [min, max].
    const bool key_bins = true;
    const int kshift = max(0, (32 - __clz((kmax - kmin) | 1u)) - 11);
    for (int pass = 0;; ++pass) {
#ifdef PQKV_PASS_STAMPS  // tools/microbench/pair_select_probe.cu: per-pass clocks + survivor counts
        if (tp && tid == 0 && pass < 4) tp[8 + pass] = clock64();
#endif
        if (lo == hi) {  // every candidate has the same key
            kstar = score_key((float)lo);
            break;
        }
        const double scale = (double)NB / (hi - lo);
        const bool kb = pass == 0 && key_bins;
        auto bin_of = [&](uint32_t key) {
            return kb ? (int)((key - kmin) >> kshift) : min(NB - 1, (int)(((double)key_score(key) - lo) * scale));
        };
#pragma unroll
        for (int u = 0; u < WMAX; ++u) {
            if (u >= per) break;
            if ((alive >> u) & 1u) {
                const int b = bin_of(kr[u]);
                atomicAdd(&hist[b], it[u] & wmask);
                atomicAdd(&cnt[b], 1u);
            }
        }
        __syncthreads();
#ifdef PQKV_PASS_STAMPS
        if (tp && tid == 0 && pass < 4) tp[21 + pass] = clock64();
#endif
        find_digit<NT>(hist, NB, k_rem, wsum, sh);
#ifdef PQKV_PASS_STAMPS
        if (tp && tid == 0 && pass < 4) tp[25 + pass] = clock64();
#endif
        const int bsel = (int)sh[0];
        k_rem -= sh[1];
        const uint32_t items = cnt[bsel];
#ifdef PQKV_PASS_STAMPS
        if (tp && tid == 0 && pass < 4) tp[12 + pass] = items;
#endif
        float vmin = INFINITY, vmax = -INFINITY;
#pragma unroll
        for (int u = 0; u < WMAX; ++u) {
            if (u >= per) break;
            if ((alive >> u) & 1u) {
                const float f = key_score(kr[u]);
                const int b = bin_of(kr[u]);
                if (b != bsel) alive &= ~(1u << u);
                else { vmin = fminf(vmin, f); vmax = fmaxf(vmax, f); }
            }
        }
        __syncthreads();  // hist / cnt / sh reads done
        if (items <= 32) {
            // one warp sorts the (key, weight) of the survivors, descending
            unsigned long long* small = reinterpret_cast<unsigned long long*>(hist);
            if (tid == 0) sh[2] = 0;
            __syncthreads();
#pragma unroll
            for (int u = 0; u < WMAX; ++u) {
                if (u >= per) break;
                if ((alive >> u) & 1u) small[atomicAdd(&sh[2], 1u)] = (unsigned long long)kr[u] << 32 | (it[u] & wmask);
            }
            __syncthreads();
            if (warp == 0) {
                const int n = (int)sh[2];
                unsigned long long v = lane < n ? small[lane] : 0ull;
#pragma unroll
                for (int sz = 2; sz <= 32; sz <<= 1)
#pragma unroll
                    for (int st = sz >> 1; st > 0; st >>= 1) {
                        const unsigned long long o = __shfl_xor_sync(FULL, v, st);
                        const bool keep_max = ((lane & sz) == 0) == ((lane & st) == 0);
                        v = keep_max ? (v > o ? v : o) : (v < o ? v : o);
                    }
                const uint32_t key = (uint32_t)(v >> 32), wt = (uint32_t)v;
                uint32_t x = wt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(FULL, x, o);
                    if (lane >= o) x += y;
                }
                const unsigned hm = __ballot_sync(FULL, lane < n && x >= k_rem);
                const uint32_t ks = __shfl_sync(FULL, key, __ffs(hm) - 1);
                const uint32_t above = warp_sum(lane < n && key > ks ? wt : 0u);
                if (lane == 0) { sh[5] = ks; sh[6] = above; }
            }
            __syncthreads();
            kstar = sh[5];
            k_rem -= sh[6];
            break;
        }
        if (items <= 128) {
            // up to 128 survivors: rank them directly (a survivor's rank =
            // survivors with a larger (key, weight) word, ties by list slot),
            // scatter into rank order and scan the weights -- replaces another
            // histogram pass plus the warp sort (powerlaw keys: ~100
            // survivors after the first pass; select 6.7 -> 5.6 us in
            // tools/microbench/pair_select_probe.cu; the quadratic ranking
            // loses above ~200 survivors)
            unsigned long long* small = reinterpret_cast<unsigned long long*>(hist);   // [items]
            unsigned long long* srt = reinterpret_cast<unsigned long long*>(cnt);      // [items] rank order
            if (tid == 0) sh[2] = 0;
            __syncthreads();
#pragma unroll
            for (int u = 0; u < WMAX; ++u) {
                if (u >= per) break;
                if ((alive >> u) & 1u) small[atomicAdd(&sh[2], 1u)] = (unsigned long long)kr[u] << 32 | (it[u] & wmask);
            }
            __syncthreads();
            const int n = (int)sh[2];
            for (int i = tid; i < n; i += NT) {
                const unsigned long long v = small[i];
                int rank = 0;
                for (int j = 0; j < n; ++j) {
                    const unsigned long long o = small[j];
                    rank += (o > v) || (o == v && j < i);
                }
                srt[rank] = v;
            }
            __syncthreads();
            // thread t owns ranks 2t, 2t+1
            const int r0 = 2 * tid;
            const uint32_t w0 = r0 < n ? (uint32_t)srt[r0] : 0u, w1 = r0 + 1 < n ? (uint32_t)srt[r0 + 1] : 0u;
            const uint32_t before = block_excl_scan<NT>(w0 + w1, wsum, nullptr);
            if (r0 < n && before < k_rem && k_rem <= before + w0) sh[5] = (uint32_t)(srt[r0] >> 32);
            if (r0 + 1 < n && before + w0 < k_rem && k_rem <= before + w0 + w1) sh[5] = (uint32_t)(srt[r0 + 1] >> 32);
            __syncthreads();
            const uint32_t ks = sh[5];
            // weight above K*: the cumulative weight before the first rank with key K*
            if (r0 < n && (uint32_t)(srt[r0] >> 32) == ks && (r0 == 0 || (uint32_t)(srt[r0 - 1] >> 32) != ks))
                sh[6] = before;
            if (r0 + 1 < n && (uint32_t)(srt[r0 + 1] >> 32) == ks && (uint32_t)(srt[r0] >> 32) != ks)
                sh[6] = before + w0;
            __syncthreads();
            kstar = ks;
            k_rem -= sh[6];
            break;
        }
        // more than 128 pairs left: next pass over their [min, max]
        vmin = warp_min(vmin);
        vmax = warp_max(vmax);
        if (lane == 0) { reinterpret_cast<float*>(wsum)[warp] = vmin; reinterpret_cast<float*>(wsum)[32 + warp] = vmax; }
        for (int e = tid; e < NB; e += NT) { hist[e] = 0; cnt[e] = 0; }
        __syncthreads();
        float a = INFINITY, z = -INFINITY;
#pragma unroll
        for (int w2 = 0; w2 < NT / 32; ++w2) {
            a = fminf(a, reinterpret_cast<float*>(wsum)[w2]);
            z = fmaxf(z, reinterpret_cast<float*>(wsum)[32 + w2]);
        }
        lo = (double)a;
        hi = (double)z;
        __syncthreads();  // wsum reads done before find_digit reuses it
    }
    PQKV_T(4);
    // ---- classification of the present pairs; equal pairs -> eql (= lst) ----
    uint32_t* eql = lst;  // every thread has its items in registers
    if (tid == 0) sh[2] = 0;
    __syncthreads();
#pragma unroll
    for (int u = 0; u < WMAX; ++u) {
        if (u >= per) break;
        if (!(it[u] & wmask)) continue;
        const uint32_t t = it[u] >> wbits, kk = kr[u];
        const uint8_t c = kk > kstar ? 1 : (kk == kstar ? 2 : 0);
        cls[t] = c;
        if (c == 2) eql[atomicAdd(&sh[2], 1u)] = t;
    }
    __syncthreads();
    PQKV_T(5);
    const int neq = (int)sh[2];
    for (int e = tid; e < neq * n_chunks; e += NT) {
        int c = e / neq, t = (int)eql[e % neq];
        uint32_t v = chist[(long long)c * C2 + t];
        if (v) atomicAdd(&ceq[c], v);
    }
    __syncthreads();
    PQKV_T(6);
    if (tid < 32) {  // chunk holding the k_rem-th equal token (warp scan over chunks)
        uint32_t run = 0;
        int cstar = -1;
        uint32_t take = 0;
        for (int c0 = 0; c0 < n_chunks && cstar < 0; c0 += 32) {
            const int c = c0 + lane;
            uint32_t v = c < n_chunks ? ceq[c] : 0u, x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(FULL, x, o);
                if (lane >= o) x += y;
            }
            const bool hit = c < n_chunks && run + x >= k_rem;
            const unsigned hm = __ballot_sync(FULL, hit);
            if (hm) {
                const int l = __ffs(hm) - 1;
                const uint32_t xl = __shfl_sync(FULL, x, l), vl = __shfl_sync(FULL, v, l);
                cstar = c0 + l;
                take = k_rem - (run + xl - vl);
            }
            run += __shfl_sync(FULL, x, 31);
        }
        if (lane == 0) {
            sh[3] = (uint32_t)(cstar < 0 ? n_chunks - 1 : cstar);
            sh[4] = take;
            sh[5] = kstar;
        }
    }
    __syncthreads();
}

// Shared-memory bytes of pair_select's scratch for C centroids and n_chunks
// tuple chunks (lut | hist | cnt | lst | ceq | wsum | sh).
__host__ __device__ constexpr size_t pair_select_scratch(int C, int n_chunks) {
    return (size_t)16 * C + (size_t)4 * (2 * NB + (size_t)C * C + n_chunks + 72);
}

// Carves pair_select's scratch out of z (8-byte aligned).
struct PairScratch {
    double* lut;
    uint32_t *hist, *cnt, *lst, *ceq, *wsum, *sh;
    __device__ PairScratch(unsigned char* z, int C, int n_chunks) {
        lut = reinterpret_cast<double*>(z);
        hist = reinterpret_cast<uint32_t*>(lut + 2 * C);
        cnt = hist + NB;
        lst = cnt + NB;
        ceq = lst + C * C;
        wsum = ceq + n_chunks;
        sh = wsum + 64;
    }
};

}  // namespace pqkv_dev
