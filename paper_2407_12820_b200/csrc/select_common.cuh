// select_common.cuh -- device building blocks shared by the selection
// kernels (select.cu) and the fused decode kernel (attend.cu).
#pragma once

#include "common.cuh"

namespace pqkv_dev {

constexpr int NB = 2048;  // bins of the two 11-bit radix digits

// Builds T[j][c] (pq.cpp:113-126, rows accumulated as in pq.cpp:157-159).
// One thread per (j, c); the t-chain stays sequential (reference order) while
// the centroid row is prefetched 16 floats at a time so the chain is not
// serialised on L2 latency.
__device__ inline void build_lut(double* lut, const float* q, const float* cen, int g, int d_h, int m,
                          int C) {
    const int d_m = d_h / m;
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
                    for (int u = 0; u < 16; ++u) qv[u] = (t0 + u < d_m) ? __ldg(qq + u) : 0.0f;
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


// Pair-level exact top-k for one head (m == 2): builds the ADC table, the
// C*C pair keys, radix-selects the k-th largest key weighted by the pair
// histogram thist, classifies every pair (0 below, 1 above, 2 equal) into
// cls[], and finds the PQKV_TUPLE_CHUNK chunk c* holding the k_rem-th equal
// token in id order plus how many of c*'s equal tokens are taken.  On return
// (after a barrier) sh[3] = c*, sh[4] = take, sh[5] = K*.  All scratch is
// shared memory owned by the caller: lut[2C] f64, key[C*C], hist[NB],
// eql[C*C], ceq[n_chunks], wsum[32], sh[8].
template <int NT>
__device__ void pair_select(const float* q, int g, int d_h, const float* cen, int C,
                            const uint32_t* thist, const uint16_t* chist, int n_chunks, int k,
                            double* lut, uint32_t* key, uint32_t* hist, uint32_t* eql, uint32_t* ceq,
                            uint32_t* wsum, uint32_t* sh, uint8_t* cls, uint32_t* tkey_out) {
    const int tid = threadIdx.x, C2 = C * C;
    build_lut(lut, q, cen, g, d_h, 2, C);
    for (int c = tid; c < n_chunks; c += NT) ceq[c] = 0;
    if (tid == 0) sh[2] = 0;
    __syncthreads();
    for (int t = tid; t < C2; t += NT) {
        double acc = __dadd_rn(0.0, lut[t / C]);
        acc = __dadd_rn(acc, lut[C + t % C]);
        key[t] = score_key((float)acc);
    }
    uint32_t k_rem = (uint32_t)k, prefix = 0;
    const int shifts[3] = {21, 10, 0};
    const int nbins[3] = {2048, 2048, 1024};
    for (int pass = 0; pass < 3; ++pass) {
        for (int b = tid; b < NB; b += NT) hist[b] = 0;
        __syncthreads();
        const uint32_t mask = (uint32_t)(nbins[pass] - 1);
        for (int t = tid; t < C2; t += NT) {
            uint32_t kk = key[t];
            if (pass > 0 && (kk >> shifts[pass - 1]) != prefix) continue;
            uint32_t ww = __ldg(thist + t);
            if (ww) atomicAdd(&hist[(kk >> shifts[pass]) & mask], ww);
        }
        __syncthreads();
        find_digit<NT>(hist, nbins[pass], k_rem, wsum, sh);
        k_rem -= sh[1];
        prefix = (prefix << (pass == 2 ? 10 : 11)) | sh[0];
        __syncthreads();
    }
    const uint32_t kstar = prefix;
    for (int t = tid; t < C2; t += NT) {
        uint32_t kk = key[t];
        uint8_t c = kk > kstar ? 1 : (kk == kstar ? 2 : 0);
        cls[t] = c;
        if (c == 2 && __ldg(thist + t)) eql[atomicAdd(&sh[2], 1u)] = (uint32_t)t;
        if (tkey_out) tkey_out[t] = kk;
    }
    __syncthreads();
    const int neq = (int)sh[2];
    for (int e = tid; e < neq * n_chunks; e += NT) {
        int c = e / neq, t = (int)eql[e % neq];
        uint32_t v = chist[(long long)c * C2 + t];
        if (v) atomicAdd(&ceq[c], v);
    }
    __syncthreads();
    if (tid < 32) {  // chunk holding the k_rem-th equal token (warp scan over chunks)
        const int lane = tid;
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

}  // namespace pqkv_dev
