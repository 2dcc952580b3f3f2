// attend.cu -- K/V gather + sparse softmax attention on sm_100a (hot path B).
//
// selective_attention (attention.cpp:62-91) attends over init [0,n_init) ++
// the selected middle tokens in ascending id ++ the local window: on the flat
// per-head layout that is simply the selected token ids in ascending order.
//
// Fast path (d_h = 128, g in {1,2,4}, fp32, PQKV_PREC_F32) -- the decode hot loop:
//   grid = chunks x heads, sized so every CTA is resident in one wave.  A CTA
//   owns a PQKV_TUPLE_CHUNK-multiple range of middle tokens (+ the init rows
//   for chunk 0, the local rows for the last chunk).  It first turns its
//   range into ascending row ids in shared memory -- from the selection
//   bitmap, or directly from the codes via the code-pair classes of
//   tuple_select (no bitmap round trip) -- then every 16-lane half-warp
//   gathers one 512 B K row and one V row per step with coalesced 128-bit
//   loads, double-buffered (the next row is in flight while the current one
//   is consumed), and folds it into an fp32 online softmax in the log2
//   domain with lazy rescaling.  Half-warps, warps and CTAs are merged with
//   (max, sum, acc) rescaling; the last CTA of a head to finish merges the
//   per-CTA partials (atomic arrival counter), so a layer is one launch.
//
// Exact path (PQKV_PREC_F64, any d_h) -- the C++ API drop-in:
//   exact_scores (attention.cpp:11-26) in fp64 with the same summation order
//   (bit-identical f32 scores), max-subtracted fp64 exp, the serial fp64 total
//   and the row-ordered fp64 accumulation of softmax_attention
//   (attention.cpp:35-60).  Only exp() differs in implementation from libm.
#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "internal.cuh"
#include "select_common.cuh"

namespace pqkv_dev {
namespace {

constexpr int AT_THREADS = 256;
constexpr int AT_WARPS = AT_THREADS / 32;
constexpr int DH = 128;
constexpr int LPR = 16;            // lanes per K/V row
constexpr int VPL = DH / 4 / LPR;  // float4 per lane per row (2)

enum { SRC_ROWS = 0, SRC_BITMAP = 1, SRC_TUPLE = 2, SRC_PAIRS = 3, SRC_KEYS = 4 };

struct AtArgs {
    const float* queries;  // [P][G][128]
    const float* keys;
    const float* values;
    long long kv_head_stride;
    int src;
    int n_init, n_local, total, s_mid;
    int chunk;     // middle tokens (bitmap/tuple) or list positions (rows) per CTA
    int n_chunks;  // CTAs per head
    // SRC_BITMAP
    const uint32_t* bitmap;
    int words;
    // SRC_TUPLE
    const uint16_t* codes;
    long long codes_head_stride;
    int C;
    const uint8_t* cls;  // [P][C*C]
    const int* cut;      // [P][2]
    // SRC_PAIRS (pair select fused into the prologue)
    const float* centroids;       // [P][2][C][64]
    const uint32_t* thist;        // [P][C*C]
    const uint16_t* chist;        // [P][n_tchunks][C*C]
    int n_tchunks, k, region;     // region: bytes of the aliased scratch area
    int m;                        // SRC_KEYS: subspaces (any m, b with m * 2^b * 8 <= 16 KB)
    long long tchunk_stride;      // chunks per head of chist
    // SRC_ROWS
    const int64_t* rows;
    int t;
    float scale_log2;    // log2(e) / sqrt(d_h)
    float* part;         // [P][n_chunks][G][DH + 2]
    float* part2;        // two-level merge: [P][n_groups][G][DH + 2] group partials, else null
    int n_groups;        // two-level merge: ceil(n_chunks / MERGE_GROUP)
    unsigned* arrivals;  // [P] (+ [P][n_groups] two-level) zero on entry; reset by the combining CTAs
    float* out;          // [P][G][DH]
    uint32_t* sel_dump;        // [P][words] selection words of the fused modes (test hook) or null
    int ring_off;              // g > 1: byte offset of the cp.async row ring in dynamic smem
    int ring4;                 // g > 1: ring depth 4 (else 2: large chunks keep 2 CTAs/SM)
    int win;                   // selected middle rows expanded per gather window (list modes: chunk)
    int stage;                 // pair mode: stage the CTA's codes in shared memory
    int nt;                    // threads per CTA (AT_THREADS, or 1024 for the wide g > 1 plans)
    int claim;                 // wide plans: warps claim rows dynamically (experiment: PQKV_CLAIM=1)
    uint32_t* sel_only;        // SRC_KEYS: write the selection bitmap [P][words] here and stop (split launch)
    unsigned* ready_out;       // select-only launch: [P] bumped once per CTA after its words are written, or null
    unsigned* ready_in;        // gather of a split path: [P] polled until ready_need (instead of the grid wait), or null
    unsigned ready_need;       // select CTAs per unit
    unsigned long long* prof;  // [grid][PQKV_PROF_SLOTS] phase timestamps (profiling mode) or null
};

__device__ __forceinline__ float safe_scale(float m_old, float m_new) {
    return m_old == -INFINITY ? 0.0f : exp2f(m_old - m_new);
}

// Shared memory: rows[rows_cap] | words[chunk/32] | cls[C*C] (tuple) | small.
struct AtSmem {
    int* rows;
    uint32_t* words;
    uint8_t* cls;
};

// Expands selection words (bit b of word w = middle token base + 32w + b) into
// ascending token ids at rows[off...]; every warp owns a contiguous range of
// words.  Returns the number of rows written (block-uniform).
template <int NT = AT_THREADS>
__device__ int expand_words(const uint32_t* words, int nwords, int token_base, int* rows, int off,
                            uint32_t* wtot) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int per = (nwords + (NT / 32) - 1) / (NT / 32);
    const int w0 = warp * per, w1 = min(nwords, w0 + per);
    uint32_t cnt = 0;
    for (int w = w0 + lane; w < w1; w += 32) cnt += __popc(words[w]);
    cnt = warp_sum(cnt);
    if (lane == 0) wtot[warp] = cnt;
    __syncthreads();
    uint32_t before = 0, total = 0;
#pragma unroll
    for (int w = 0; w < (NT / 32); ++w) {
        uint32_t v = wtot[w];
        before += w < warp ? v : 0;
        total += v;
    }
    __syncthreads();
    uint32_t run = off + before;
    for (int wb = w0; wb < w1; wb += 32) {
        const int w = wb + lane;
        uint32_t bits = w < w1 ? words[w] : 0u;
        uint32_t c = __popc(bits), x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(FULL, x, o);
            if (lane >= o) x += y;
        }
        uint32_t pos = run + x - c;
        while (bits) {
            int b = __ffs(bits) - 1;
            bits &= bits - 1;
            rows[pos++] = token_base + w * 32 + b;
        }
        run += __shfl_sync(FULL, x, 31);
    }
    __syncthreads();
    return (int)total;
}

// expand_words restricted to the selected bits of rank [lo, hi) (rank = the
// bit's position among all set bits of words[0..nwords) in id order); the
// row of rank j goes to rows[off + j - lo].  Returns the number written.
template <int NT = AT_THREADS>
__device__ int expand_words_range(const uint32_t* words, int nwords, int token_base, int* rows, int off, uint32_t lo,
                                  uint32_t hi, uint32_t* wtot) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int per = (nwords + (NT / 32) - 1) / (NT / 32);
    const int w0 = warp * per, w1 = min(nwords, w0 + per);
    uint32_t cnt = 0;
    for (int w = w0 + lane; w < w1; w += 32) cnt += __popc(words[w]);
    cnt = warp_sum(cnt);
    if (lane == 0) wtot[warp] = cnt;
    __syncthreads();
    uint32_t before = 0, total = 0;
#pragma unroll
    for (int w = 0; w < (NT / 32); ++w) {
        uint32_t v = wtot[w];
        before += w < warp ? v : 0;
        total += v;
    }
    __syncthreads();
    if (before < hi && before + cnt > lo) {
        uint32_t run = before;
        for (int wb = w0; wb < w1; wb += 32) {
            const int w = wb + lane;
            uint32_t bits = w < w1 ? words[w] : 0u;
            uint32_t c = __popc(bits), x = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(FULL, x, o);
                if (lane >= o) x += y;
            }
            uint32_t pos = run + x - c;
            if (pos < hi && pos + c > lo)
                while (bits) {
                    const int b = __ffs(bits) - 1;
                    bits &= bits - 1;
                    if (pos >= lo && pos < hi) rows[off + (int)(pos - lo)] = token_base + w * 32 + b;
                    ++pos;
                }
            run += __shfl_sync(FULL, x, 31);
        }
    }
    __syncthreads();
    return (int)(min(total, hi) > lo ? min(total, hi) - lo : 0u);
}

// Staged code layout: within every block of 256 16-byte chunks (1024
// tokens = 32 selection words), chunk u of word w sits at u * 32 + w, so the
// 32 lanes of a warp reading chunk u of 32 consecutive words hit 32
// consecutive 16-byte slots (no bank conflicts).
__device__ __forceinline__ int code_swz(int f) { return (f & ~255) | ((f & 7) << 5) | ((f >> 3) & 31); }

// Tuple classification of middle tokens [r0, r1) into selection words
// (pq.cpp:128-140 pair score, topk.cpp tie rule via the pair-select cut).
// r0 is a multiple of 32 (r1 too, unless it is s_mid), so a 32-token word
// never straddles a PQKV_TUPLE_CHUNK chunk.  Code pairs come from shared
// memory (`staged`: this CTA's range with the code_swz layout) or from
// global memory (cd_g, absolute rows).  Each warp owns a contiguous run of
// words; each lane builds whole words from 8 128-bit loads.
//  * FINAL: cls in {0 below / absent, 1 above, 2 equal}.  A token is
//    selected when its pair class is "above", or "equal" and it is among the
//    first `take` equal tokens of tuple chunk c* in id order (all equal
//    tokens of earlier chunks, none of later ones).  words[] = selection.
//  * PRELIM (early release): cls in {0 below, 1 above, 3 pending}.
//    words[] = above, eqw[] = pending.
template <bool PRELIM, int NT = AT_THREADS>
__device__ void classify_range(const AtArgs& a, int r0, int r1, const uint32_t* cd_g, const uint32_t* staged,
                               uint32_t* words, uint32_t* eqw, const uint8_t* cls, uint32_t* wtot, int cstar,
                               uint32_t take) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nw = (max(0, r1 - r0) + 31) >> 5;
    const int per = (nw + (NT / 32) - 1) / (NT / 32);
    const int w0 = min(nw, warp * per), w1 = min(nw, w0 + per);
    const uint32_t C = (uint32_t)a.C;
    const uint32_t eqc = PRELIM ? 3u : 2u;
    const bool gvec = (reinterpret_cast<uintptr_t>(cd_g + r0) & 15) == 0;
    // ---- step 1: above / equal (pending) words ----
    if (!staged && per <= 16) {
        // few words per warp (wide CTAs): lane l classifies token l of each
        // word (one coalesced 128-byte load per word, all issued up front)
        // instead of one word per lane on w1 - w0 lanes
        uint32_t pv[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int t = r0 + 32 * (w0 + u) + lane;
            pv[u] = (u < w1 - w0 && t < r1) ? cd_g[t] : 0u;
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            if (u >= w1 - w0) break;
            const bool ok = r0 + 32 * (w0 + u) + lane < r1;
            const uint32_t cl = ok ? cls[(pv[u] & 0xffffu) * C + (pv[u] >> 16)] : 0u;
            const uint32_t gt = __ballot_sync(FULL, cl == 1), eq = __ballot_sync(FULL, cl == eqc);
            if (lane == 0) {
                words[w0 + u] = gt;
                eqw[w0 + u] = eq;
            }
        }
    } else
    for (int wb = w0; wb < w1; wb += 32) {
        const int wi = wb + lane;
        if (wi >= w1) continue;
        const int nvalid = min(32, r1 - (r0 + 32 * wi));
        uint32_t gt = 0, eq = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            uint4 v;
            if (staged) {
                v = reinterpret_cast<const uint4*>(staged)[code_swz(wi * 8 + u)];
            } else if (gvec && nvalid == 32) {
                v = *reinterpret_cast<const uint4*>(cd_g + r0 + 32 * wi + 4 * u);
            } else {
                const uint32_t* c = cd_g + r0 + 32 * wi + 4 * u;
                v.x = 4 * u + 0 < nvalid ? c[0] : 0u;
                v.y = 4 * u + 1 < nvalid ? c[1] : 0u;
                v.z = 4 * u + 2 < nvalid ? c[2] : 0u;
                v.w = 4 * u + 3 < nvalid ? c[3] : 0u;
            }
            const uint32_t pv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int t = 4 * u + e;
                if (t < nvalid) {
                    const uint32_t cl = cls[(pv[e] & 0xffffu) * C + (pv[e] >> 16)];
                    gt |= (uint32_t)(cl == 1) << t;
                    eq |= (uint32_t)(cl == eqc) << t;
                }
            }
        }
        words[wi] = gt;
        eqw[wi] = eq;
    }
    __syncthreads();
    if constexpr (PRELIM) return;
    // ---- step 2: equal tokens: all of chunks before c*, the first `take` of
    // c* in id order, none after ----
    const int a0 = cstar * PQKV_TUPLE_CHUNK, a1 = a0 + PQKV_TUPLE_CHUNK;
    for (int w = tid; w < nw; w += NT)
        if ((r0 + 32 * w) / PQKV_TUPLE_CHUNK < cstar) words[w] |= eqw[w];
    const int b0 = max(r0, a0), b1 = min(r1, a1);
    if (b0 < b1) {  // this range holds part of chunk c* (block-uniform)
        // equal tokens of c* before this range (other CTAs' tokens)
        uint32_t pre = 0;
        for (int i = a0 + tid; i < r0; i += NT) {
            const uint32_t pr = cd_g[i];
            pre += cls[(pr & 0xffffu) * C + (pr >> 16)] == 2;
        }
        pre = warp_sum(pre);
        if (lane == 0) wtot[warp] = pre;
        __syncthreads();
        pre = 0;
#pragma unroll
        for (int w = 0; w < (NT / 32); ++w) pre += wtot[w];
        __syncthreads();
        // ordered prefix over the words of c* in this range: <= 128 words,
        // thread t owns word wb0 + t
        const int wb0 = (b0 - r0) >> 5, wb1 = (b1 - r0 + 31) >> 5;
        const int w = wb0 + tid;
        const uint32_t e = w < wb1 ? eqw[w] : 0u;
        const uint32_t before = pre + block_excl_scan<NT>((uint32_t)__popc(e), wtot, nullptr);
        if (w < wb1 && e) {
            uint32_t keep = 0;
            const uint32_t c = __popc(e);
            if (before + c <= take) keep = e;
            else if (before < take) {
                uint32_t mm = e;
                for (uint32_t k = take - before; k; --k) { keep |= mm & (0u - mm); mm &= mm - 1; }
            }
            words[w] |= keep;
        }
    }
    __syncthreads();
}

// ---- SRC_KEYS: fused exact top-k over per-token ADC scores (generic m, b) ----
// The CTAs of one head form one thread-block cluster; CTA rank r owns the
// middle tokens [r*chunk, ...), so rank order is id order.  Every CTA builds
// the fp64 ADC table (pq.cpp:113-126), computes its tokens' keys
// f32(((0.0 + T[0][c0]) + T[1][c1]) + ...) (pq.cpp:128-140) into shared
// memory and histograms them; three radix digit passes (11/11/10 bits) find
// the k-th largest key K*, each pass merging the cluster's histograms through
// DSMEM (every CTA sums the same bins, so one cluster barrier per pass; two
// histogram buffers alternate so a buffer is only cleared after everyone has
// read it).  Ties at K* go to the lowest ids (topk.cpp:17-22): a cluster-wide
// prefix of per-CTA equal counts gives each CTA its share.  Output: the
// CTA's selection words (bit = middle row selected).
__device__ __forceinline__ void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Histogram increment; bin == ~0u is a no-op.
__device__ __forceinline__ void hist_inc(uint32_t* h, uint32_t bin) {
    if (bin != 0xffffffffu) atomicAdd(&h[bin], 1u);
}

__device__ __forceinline__ double dsmem_ld64(const double* local_ptr, unsigned rank) {
    uint32_t ra;
    double v;
    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"((unsigned)__cvta_generic_to_shared(local_ptr)), "r"(rank));
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra));
    return v;
}

// ADC table entries [e0, e1) (pq.cpp:113-126 per entry; lut_entry_vec for
// d_m = 32 / 64, the generic sequential chain otherwise).
__device__ void build_lut_range(double* lut, const float* q, const float* cen, int g, int d_h, int m, int C,
                                int e0, int e1) {
    const int d_m = d_h / m;
    const bool aligned = ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(cen)) & 15) == 0 &&
                         (d_h % 4) == 0;
    for (int e = e0 + (int)threadIdx.x; e < e1; e += blockDim.x) {
        const int j = e / C;
        if (aligned && d_m == 64 && g > 1) { lut_entry_multi<64>(lut, q, cen, g, d_h, e, j); continue; }
        if (aligned && d_m == 32 && g > 1) { lut_entry_multi<32>(lut, q, cen, g, d_h, e, j); continue; }
        if (aligned && d_m == 64) { lut_entry_vec<64>(lut, q, cen, g, d_h, e, j); continue; }
        if (aligned && d_m == 32) { lut_entry_vec<32>(lut, q, cen, g, d_h, e, j); continue; }
        const float* cc = cen + (long long)e * d_m;
        double t = 0.0;
        for (int r = 0; r < g; ++r) {
            const float* qq = q + (long long)r * d_h + j * d_m;
            double acc = 0.0;
            for (int u = 0; u < d_m; ++u) acc = __fma_rn((double)qq[u], (double)__ldg(cc + u), acc);
            t = __dadd_rn(t, acc);
        }
        lut[e] = t;
    }
}

__device__ __forceinline__ uint32_t dsmem_ld(const void* local_ptr, unsigned rank) {
    uint32_t ra, v;
    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"((unsigned)__cvta_generic_to_shared(local_ptr)), "r"(rank));
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(ra));
    return v;
}

// One cluster-wide select step over a histogram pass, entered after the
// barrier that completes every CTA's histogram h[nb] (bins ascending in key
// order): CTA r sums its 1/ncl share of the bins over the cluster (DSMEM)
// into own[] -> barrier -> every CTA locates the share holding the k_rem-th
// largest participant and reads that share's merged bins.  Result: sh[0] =
// the bin, sh[1] = participants in higher bins, sh[4] = the bin's count.
template <int NT>
__device__ void cluster_locate(const uint32_t* h, uint32_t* own, int nb, uint32_t k_rem, unsigned crank,
                               unsigned ncl, uint32_t* pub, uint32_t* wtot, uint32_t* sh) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int share = (nb + (int)ncl - 1) / (int)ncl;  // bins per CTA
    {
        const int o0 = (int)crank * share, o1 = min(nb, o0 + share);
        uint32_t tot = 0;
        for (int bn = o0 + tid; bn < o1; bn += NT) {
            uint32_t v = 0;
            for (unsigned r = 0; r < ncl; ++r) v += dsmem_ld(h + bn, r);
            own[bn - o0] = v;
            tot += v;
        }
        tot = warp_sum(tot);
        if (lane == 0) wtot[warp] = tot;
        __syncthreads();
        if (tid == 0) {
            uint32_t t = 0;
            for (int w = 0; w < (NT / 32); ++w) t += wtot[w];
            pub[3] = t;
        }
        __syncthreads();
    }
    cluster_barrier();  // every share is merged
    if (tid < 32) {  // the share holding the k_rem-th largest key (shares in descending bin order)
        const unsigned r = ncl - 1 - (unsigned)lane;
        const uint32_t t = lane < (int)ncl ? dsmem_ld(pub + 3, r) : 0u;
        uint32_t x = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, x, o);
            if (lane >= o) x += y;
        }
        const unsigned hit = __ballot_sync(FULL, lane < (int)ncl && x >= k_rem && x - t < k_rem);
        const int l = __ffs(hit) - 1;
        if (lane == l) { sh[2] = r; sh[3] = x - t; }
    }
    __syncthreads();
    const unsigned rs = sh[2];
    const uint32_t above_share = sh[3];
    // digit inside share rs: thread t owns share bins [hi - per, hi), top down
    const int o0 = (int)rs * share, cnt_bins = min(nb, o0 + share) - o0;
    const int nbe = max(cnt_bins, NT);
    const int per = (nbe + NT - 1) / NT;  // 1..8
    const int hi = nbe - per * tid;
    uint32_t cnt[8];
    uint32_t local = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int bn = hi - per + e;
        cnt[e] = (e < per && bn >= 0 && bn < cnt_bins) ? dsmem_ld(own + bn, rs) : 0u;
        local += cnt[e];
    }
    const uint32_t kk = k_rem - above_share;
    const uint32_t above = block_excl_scan<NT>(local, wtot, nullptr);
    if (above < kk && kk <= above + local) {
        uint32_t acc = above;
#pragma unroll
        for (int e = 7; e >= 0; --e) {  // bins from the top
            if (e >= per) continue;
            if (kk <= acc + cnt[e]) {
                sh[0] = (uint32_t)(o0 + hi - per + e);
                sh[1] = above_share + acc;
                sh[4] = cnt[e];
                break;
            }
            acc += cnt[e];
        }
    }
    __syncthreads();
}

// Value-linear bin of score v over [lo, lo + NB / sc): monotone
// non-decreasing in v (every step rounds monotonically and the ends clamp),
// so bins are ordered like keys whatever the rounding.
__device__ __forceinline__ int vbin(float v, float lo, float sc) {
    const int b = __float2int_rz(__fmul_rn(__fsub_rn(v, lo), sc));
    return min(NB - 1, max(0, b));
}

// Last u32 key in [k0, k1] for which pred holds, pred holding on a prefix
// of the range and at k0 (k0 - 1 if it holds nowhere): a warp-wide 33-ary
// search, ~7 rounds for a full 32-bit range.
template <class Pred>
__device__ uint32_t warp_last_true(uint32_t k0, uint32_t k1, Pred pred) {
    const int lane = threadIdx.x & 31;
    // the first key where pred fails lies in [lo, hi] (hi = k1 + 1: nowhere)
    unsigned long long lo = k0, hi = (unsigned long long)k1 + 1;
    while (hi > lo) {
        const unsigned long long span = hi - lo;
        const unsigned long long pt = lo + span * (unsigned long long)(lane + 1) / 33;  // < hi
        const unsigned t = __ballot_sync(FULL, pred((uint32_t)pt));
        const int c = __popc(t);  // lanes 0..c-1 hold (probes ascend with the lane)
        const unsigned long long p_last = __shfl_sync(FULL, pt, max(c - 1, 0));
        const unsigned long long p_next = __shfl_sync(FULL, pt, min(c, 31));
        if (c > 0) lo = p_last + 1;
        if (c < 32) hi = p_next;
    }
    return (uint32_t)(lo - 1);
}

constexpr uint32_t KEYS_CAND_CAP = 512;  // final-bin keys resolved by counting (else the radix passes)

template <int G, int NT = AT_THREADS>
__device__ void keys_select_words(const AtArgs& a, const float* q, int p, int r0, int r1, unsigned char* region,
                                  uint32_t* words,
                                  uint32_t* hbuf /*[2][NB] + own[NB]*/, uint32_t* pub /*[4]*/, uint32_t* wtot,
                                  uint32_t* sh /*[8]*/, unsigned long long* tp) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = max(0, r1 - r0), C = a.C, m = a.m;
    uint32_t crank, ncl;
    asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
    asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(ncl));
    // scores as floats with -0 folded onto +0: float compares are the
    // reference's (topk.cpp:17-22)
    float* sc_s = reinterpret_cast<float*>(region);                  // [chunk]
    double* lut = reinterpret_cast<double*>(sc_s + a.chunk);          // [m][C]
    for (int e = tid; e < 2 * NB; e += NT) hbuf[e] = 0u;      // both buffers
    // ADC table split over the cluster: rank r computes its share of the
    // m*C entries, then copies the others' through DSMEM
    {
        const int ME = m * C, share = (ME + (int)ncl - 1) / (int)ncl;
        const int e0 = min(ME, (int)crank * share), e1 = min(ME, e0 + share);
        build_lut_range(lut, q, a.centroids + (long long)p * m * C * (DH / m), G, DH,
                        m, C, e0, e1);
        __syncthreads();
        cluster_barrier();
        for (int e = tid; e < ME; e += NT)
            if (e < e0 || e >= e1) lut[e] = dsmem_ld64(lut + e, (unsigned)(e / share));
    }
    __syncthreads();
    // a-priori score range: fp64 addition and the f32 rounding are monotone,
    // so f32(((min T0 + min T1) + ...)) <= every score <= the same over the
    // maxima.  Every CTA holds the same table: the same range cluster-wide.
    __shared__ double tmin_s[DH], tmax_s[DH];  // m <= d_h
    for (int j = warp; j < m; j += NT / 32) {
        double lo = INFINITY, hi = -INFINITY;
        for (int c = lane; c < C; c += 32) {
            lo = fmin(lo, lut[j * C + c]);
            hi = fmax(hi, lut[j * C + c]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = fmin(lo, __shfl_xor_sync(FULL, lo, o));
            hi = fmax(hi, __shfl_xor_sync(FULL, hi, o));
        }
        if (lane == 0) { tmin_s[j] = lo; tmax_s[j] = hi; }
    }
    __syncthreads();
    float lo0, hi0;
    {
        double slo = 0.0, shi = 0.0;
        for (int j = 0; j < m; ++j) {
            slo = __dadd_rn(slo, tmin_s[j]);
            shi = __dadd_rn(shi, tmax_s[j]);
        }
        lo0 = (float)slo;
        hi0 = (float)shi;
    }
    // first value pass fused into the score loop (w0 > 0 checked by all CTAs alike)
    const float w0 = __fsub_rn(hi0, lo0), sc0 = __fdiv_rn((float)NB, w0);
    const bool fuse0 = w0 > 0.f && sc0 > 0.f && !isinf(w0) && !isinf(sc0);
    uint32_t* h0 = hbuf;
    PQKV_T(0);
    // ---- scores (pq.cpp:128-140 in j order, one f32 rounding) ----
    // eight code rows in flight per thread and eight independent fp64 chains
    const uint16_t* cd = a.codes + p * a.codes_head_stride + (long long)r0 * m;
    const bool v4 = m == 4 && (reinterpret_cast<uintptr_t>(cd) & 7) == 0;
    constexpr int RIF = 16;  // code rows in flight per thread
    for (int i0 = 0; i0 < n; i0 += RIF * NT) {
        if (v4) {
            uint2 cv[RIF];
#pragma unroll
            for (int u = 0; u < RIF; ++u) {
                const int i = i0 + u * NT + tid;
                cv[u] = i < n ? *reinterpret_cast<const uint2*>(cd + 4LL * i) : make_uint2(0u, 0u);
            }
#pragma unroll
            for (int u = 0; u < RIF; ++u) {
                const int i = i0 + u * NT + tid;
                double acc = 0.0;
                acc = __dadd_rn(acc, lut[0 * C + (cv[u].x & 0xffffu)]);
                acc = __dadd_rn(acc, lut[1 * C + (cv[u].x >> 16)]);
                acc = __dadd_rn(acc, lut[2 * C + (cv[u].y & 0xffffu)]);
                acc = __dadd_rn(acc, lut[3 * C + (cv[u].y >> 16)]);
                float f = (float)acc;
                if (f == 0.0f) f = 0.0f;
                if (i < n) {
                    sc_s[i] = f;
                    if (fuse0) atomicAdd(&h0[vbin(f, lo0, sc0)], 1u);
                }
            }
        } else {
            for (int u = 0; u < RIF; ++u) {
                const int i = i0 + u * NT + tid;
                if (i >= n) break;
                double acc = 0.0;
                for (int j = 0; j < m; ++j) acc = __dadd_rn(acc, lut[j * C + cd[(long long)i * m + j]]);
                float f = (float)acc;
                if (f == 0.0f) f = 0.0f;
                sc_s[i] = f;
                if (fuse0) atomicAdd(&h0[vbin(f, lo0, sc0)], 1u);
            }
        }
    }
    __syncthreads();
    PQKV_T(1);
    uint32_t* own = hbuf + 2 * NB;  // [NB] merged counts of this CTA's share
    uint32_t k_rem = (uint32_t)a.k;

    // ---- value-linear passes: bins linear in the score over the current
    // interval [ylo, xhi] of scores (the a-priori range, then the chosen
    // bin's exact range), at most three, until the bin holding the k-th
    // largest has at most KEYS_CAND_CAP scores cluster-wide.  A radix digit
    // of the u32 key is exponent-major: scores spanning zero (gaussian keys)
    // leave ~5-10K of a 128K unit in the first digit's bin; value bins leave
    // ~100 (gaussian) or, after one refinement, ~20 (powerlaw, whose k-th
    // score sits in the dense low end of a long tail).  A chosen bin is a
    // score interval (vbin is monotone): its exact ends are found by two
    // warp-parallel searches over the float order, so every later scan tests
    // a score with two compares.  Every CTA derives the same numbers from
    // the same cluster-wide inputs, so the decisions are uniform.
    __shared__ float ends_s[2];
    float ylo = lo0, xhi = hi0;  // scores taking part in the current pass: [ylo, xhi]
    int nv = 0;
    bool cand_ok = false;
    if (fuse0) {
#pragma unroll 1
        for (int pass = 0; pass < 3; ++pass) {
            const float lo = ylo;
            const float w = __fsub_rn(xhi, lo);
            const float scl = __fdiv_rn((float)NB, w);
            if (!(w > 0.f) || !(scl > 0.f) || isinf(w) || isinf(scl)) break;
            uint32_t* h = hbuf + (pass & 1) * NB;
            if (pass >= 1) {
                if (pass >= 2) {  // this buffer was last read before the previous pass's barriers
                    for (int e = tid; e < NB; e += NT) h[e] = 0u;
                    __syncthreads();
                }
                for (int i = 4 * tid; i < n; i += 4 * NT) {
                    const float4 x = reinterpret_cast<const float4*>(sc_s)[i >> 2];
                    const float xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if (i + e < n && xv[e] >= ylo && xv[e] <= xhi) atomicAdd(&h[vbin(xv[e], lo, scl)], 1u);
                }
                __syncthreads();
            }
            cluster_barrier();  // every CTA's histogram of this pass is complete
            if (pass == 0) PQKV_T(2);
            cluster_locate<NT>(h, own, NB, k_rem, crank, ncl, pub, wtot, sh);
            if (pass == 0) PQKV_T(3);
            const int b = (int)sh[0];
            k_rem -= sh[1];
            const uint32_t nbin = sh[4];
            // the chosen bin's scores: [ylo', xhi'] inside [ylo, xhi]; warp 0
            // finds the last score with bin <= b, warp 1 the last with bin < b
            if (warp < 2) {
                const int bb = warp == 0 ? b : b - 1;
                const uint32_t k0 = score_key(ylo), k1 = score_key(xhi);
                const uint32_t last = warp_last_true(k0, k1, [&](uint32_t key) {
                    return vbin(key_score(key), lo, scl) <= bb;
                });
                if (lane == 0) ends_s[warp] = warp == 0 ? key_score(last) : key_score(last + 1);
            }
            __syncthreads();
            xhi = ends_s[0];
            ylo = ends_s[1];
            nv = pass + 1;
            __syncthreads();
            if (nbin <= KEYS_CAND_CAP) {
                cand_ok = true;
                break;
            }
        }
    }
    PQKV_T(4);
    if (tp && tid == 0) { tp[13] = (unsigned long long)nv | ((unsigned long long)cand_ok << 8); tp[15] = sh[4]; }
    const int seg = a.chunk / (NT / 32);
    const int s0 = warp * seg, s1 = min(n, s0 + seg);
    if (cand_ok) {
        // ---- one scan: provisional words (scores above the final bin) and
        // this CTA's candidates (scores in it: value + middle-row index), in
        // the histogram buffer the next pass would have used (nobody reads it)
        float* cand = reinterpret_cast<float*>(hbuf + (nv & 1) * NB);
        uint32_t* cidx = hbuf + (nv & 1) * NB + KEYS_CAND_CAP;
        __shared__ uint32_t coff[17];
        if (tid == 0) sh[5] = 0;
        __syncthreads();
        // thread t builds whole words t, t + NT, ...: 32 consecutive scores
        // as eight 16-byte loads, visited in a lane-rotated order so the 8
        // lanes of a load wavefront hit different banks; no ballots
        const int nwd = (n + 31) / 32;
        const float4* sc4 = reinterpret_cast<const float4*>(sc_s);
        for (int w = tid; w < nwd; w += NT) {
            uint32_t wd = 0, cb = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int jj = (j + lane) & 7;
                const float4 x = sc4[w * 8 + jj];
                const float xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int bit = 4 * jj + e;
                    const bool ok = w * 32 + bit < n;
                    wd |= (uint32_t)(ok && xv[e] > xhi) << bit;
                    cb |= (uint32_t)(ok && xv[e] >= ylo && xv[e] <= xhi) << bit;
                }
            }
            words[w] = wd;
            if (cb) {  // rare: ~100 scores of a 128K unit
                const uint32_t base = atomicAdd(&sh[5], (uint32_t)__popc(cb));
                uint32_t at = base;
                for (uint32_t r = cb; r; r &= r - 1) {
                    const int bit = __ffs(r) - 1;
                    cand[at] = sc_s[w * 32 + bit];
                    cidx[at] = (uint32_t)(w * 32 + bit);
                    ++at;
                }
            }
        }
        __syncthreads();
        PQKV_T(5);
        if (tid == 0) pub[0] = sh[5];
        cluster_barrier();  // every CTA's candidates are listed (and every locate is done)
        PQKV_T(6);
        if (tid < 32) {
            const uint32_t cr = lane < (int)ncl ? dsmem_ld(pub, (unsigned)lane) : 0u;
            uint32_t x = cr;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(FULL, x, o);
                if (lane >= o) x += y;
            }
            if (lane <= (int)ncl) coff[lane] = x - cr;  // lane ncl: the total
        }
        __syncthreads();
        const uint32_t T = coff[ncl];
        if (tp && tid == 0) tp[14] = T;
        float* all = reinterpret_cast<float*>(own);  // every CTA's candidate values, in rank (= id) order
        for (uint32_t e = tid; e < T; e += NT) {
            unsigned r = 0;
            while (e >= coff[r + 1]) ++r;
            const uint32_t o = e - coff[r];
            all[e] = r == crank ? cand[o] : __uint_as_float(dsmem_ld(cand + o, r));
        }
        // no remote reads of this CTA's buffers after this point; the
        // matching wait is at the end of the kernel (no CTA leaves early)
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        __syncthreads();
        // K* = the candidate x with #{> x} < k_rem <= #{>= x} (one thread per
        // candidate, the others read in lockstep: broadcast loads)
        for (uint32_t i = tid; i < (T + NT - 1) / NT * NT; i += NT) {
            const float x = i < T ? all[i] : 0.f;
            uint32_t gt = 0, eq = 0;
            for (uint32_t j = 0; j < T; ++j) {
                const float y = all[j];
                gt += y > x;
                eq += y == x;
            }
            if (i < T && gt < k_rem && k_rem <= gt + eq) { sh[6] = __float_as_uint(x); sh[7] = gt; }
        }
        __syncthreads();
        PQKV_T(7);
        const float kv = __uint_as_float(sh[6]);
        const uint32_t budget = k_rem - sh[7];  // ties at K* taken, lowest ranks (ids) first
        const uint32_t o0 = coff[crank];
        uint32_t eb = 0;
        for (uint32_t j = tid; j < o0; j += NT) eb += all[j] == kv;
        eb = warp_sum(eb);
        if (lane == 0) wtot[warp] = eb;
        __syncthreads();
        uint32_t eq_before = 0;
#pragma unroll
        for (int w = 0; w < (NT / 32); ++w) eq_before += wtot[w];
        const uint32_t take = budget > eq_before ? budget - eq_before : 0u;
        // this CTA's candidates: above K*, or among the `take` lowest-index ties
        const uint32_t mine = coff[crank + 1] - o0;
        for (uint32_t e = tid; e < mine; e += NT) {
            const float v = cand[e];
            bool sel = v > kv;
            if (v == kv) {
                uint32_t before = 0;
                for (uint32_t f = 0; f < mine; ++f) before += cand[f] == kv && cidx[f] < cidx[e];
                sel = before < take;
            }
            if (sel) atomicOr(&words[cidx[e] >> 5], 1u << (cidx[e] & 31));
        }
        __syncthreads();
        return;
    }
    // ---- fallback: radix digits over rel = key - kmin of the order-preserving
    // u32 keys (the first spans [kmin, kmax], later ones refine 11 bits at a
    // time), when the value passes cannot isolate the k-th largest (hundreds
    // of equal scores at K*, or a degenerate range) ----
    uint32_t kmin = 0xffffffffu, kmax = 0u;
    for (int i = tid; i < n; i += NT) {
        const uint32_t key = score_key(sc_s[i]);
        kmin = min(kmin, key);
        kmax = max(kmax, key);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(FULL, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(FULL, kmax, o));
    }
    __syncthreads();  // every warp is past the value passes' use of wtot / sh
    if (lane == 0) wtot[warp] = kmin;
    __syncthreads();
    if (tid == 0) {
        uint32_t lo = 0xffffffffu;
        for (int w = 0; w < (NT / 32); ++w) lo = min(lo, wtot[w]);
        pub[1] = lo;
    }
    __syncthreads();
    if (lane == 0) wtot[warp] = kmax;
    __syncthreads();
    if (tid == 0) {
        uint32_t hi = 0u;
        for (int w = 0; w < (NT / 32); ++w) hi = max(hi, wtot[w]);
        pub[2] = hi;
    }
    for (int e = tid; e < 2 * NB; e += NT) hbuf[e] = 0u;  // not read remotely since the last locate
    __syncthreads();
    cluster_barrier();  // every CTA's key range is published
    kmin = 0xffffffffu;
    kmax = 0u;
    for (unsigned r = 0; r < ncl; ++r) {
        kmin = min(kmin, dsmem_ld(pub + 1, r));
        kmax = max(kmax, dsmem_ld(pub + 2, r));
    }
    k_rem = (uint32_t)a.k;
    const uint32_t range = kmax - kmin;
    const int bits = 32 - __clz(range | 1u);
    int shift = max(0, bits - 11), width = bits - shift;
    uint32_t prefix = 0;
    uint32_t neq_local = 0;  // this CTA's scores equal to K* (bin count of the last pass)
    for (int pass = 0;; ++pass) {
        const int nb = 1 << width;
        uint32_t* h = hbuf + (pass & 1) * NB;
        if (pass >= 2) {
            for (int e = tid; e < NB; e += NT) h[e] = 0u;
            __syncthreads();
        }
        for (int i0 = 0; i0 < n; i0 += NT) {
            const int i = i0 + tid;
            uint32_t bin = 0xffffffffu;
            if (i < n) {
                const uint32_t rel = score_key(sc_s[i]) - kmin;
                if (pass == 0 || (rel >> (shift + width)) == prefix) bin = (rel >> shift) & (uint32_t)(nb - 1);
            }
            hist_inc(h, bin);
        }
        __syncthreads();
        cluster_barrier();  // every CTA's histogram of this pass is complete
        cluster_locate<NT>(h, own, nb, k_rem, crank, ncl, pub, wtot, sh);
        k_rem -= sh[1];
        prefix = (prefix << width) | sh[0];
        if (shift == 0) neq_local = h[sh[0]];  // local scores in the final bin == K*
        __syncthreads();
        if (shift == 0) break;
        width = min(11, shift);
        shift -= width;
    }
    const float kv = key_score(kmin + prefix);  // the k-th largest; k_rem of its ties are taken
    // ---- ties: equal scores of lower ranks come first ----
    const uint32_t cta_eq = neq_local;
    if (tid == 0) pub[0] = cta_eq;
    cluster_barrier();
    uint32_t eq_before = 0;
    for (unsigned r = 0; r < crank; ++r) eq_before += dsmem_ld(pub, r);
    // no remote reads of this CTA's histograms / pub after this point; the
    // matching wait is at the end of the kernel (no CTA leaves early)
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    const uint32_t take = k_rem > eq_before ? min(cta_eq, k_rem - eq_before) : 0u;
    PQKV_T(7);
    // ---- selection words in id order ----
    uint32_t weq = 0;
    for (int i0 = s0; i0 < s1; i0 += 32) {
        const int i = i0 + lane;
        weq += __popc(__ballot_sync(FULL, i < s1 && sc_s[i] == kv));
    }
    if (lane == 0) wtot[warp] = weq;
    __syncthreads();
    uint32_t run = 0;
    for (int v = 0; v < warp; ++v) run += wtot[v];
    for (int i0 = s0; i0 < s1; i0 += 32) {
        const int i = i0 + lane;
        const float v = i < s1 ? sc_s[i] : -INFINITY;
        const bool gt = i < s1 && v > kv, eq = i < s1 && v == kv;
        const unsigned em = __ballot_sync(FULL, eq);
        const bool sel = gt || (eq && run + __popc(em & lanemask_lt()) < take);
        const unsigned word = __ballot_sync(FULL, sel);
        if (lane == 0) words[i0 >> 5] = word;
        run += __popc(em);
    }
    __syncthreads();
}

// Row-list refill of the gather loops: called when the current rows are
// consumed; returns the next rows' count, or < 0 when the CTA is done.
// WindowRefill: windowed chunks (selected rows expanded `win` at a time from
// the CTA's selection words; the local rows follow the last window).
template <int NT = AT_THREADS>
struct WindowRefill {
    const AtArgs& a;
    int c;
    const uint32_t* words;
    uint32_t* wtot;
    int sel_total;
    int win_base;
    __device__ int operator()(int* rows) {
        if (win_base + a.win >= sel_total) return -1;
        __syncthreads();
        win_base += a.win;
        const int r0 = c * a.chunk, r1 = min(a.s_mid, r0 + a.chunk);
        const int nw = (max(0, r1 - r0) + 31) / 32;
        int nrows = expand_words_range<NT>(words, nw, a.n_init + r0, rows, 0, (uint32_t)win_base,
                                       (uint32_t)(win_base + a.win), wtot);
        if (c == a.n_chunks - 1 && win_base + a.win >= sel_total) {
            for (int e = threadIdx.x; e < a.n_local; e += NT) rows[nrows + e] = a.total - a.n_local + e;
            nrows += a.n_local;
        }
        __syncthreads();
        return nrows;
    }
};

// ---- g = 1 gather: one half-warp per K/V row ----
// 16 lanes x 2 float4 cover a 512 B row; each half-warp double-buffers its
// next row in registers (128-bit loads, L2 evict-first), fp32 online softmax
// in the log2 domain with lazy rescale; half-warps then merge into the
// per-warp area (wacc / wm / wl).  Rows: rows[0..nrows) of this CTA, and for
// windowed chunks the later windows of its selection words.
template <class Refill>
__device__ __forceinline__ void gather_rows_halfwarp(const AtArgs& a, const float* qsrc, int p, int* rows, int nrows,
                                                     Refill& refill,
                                                     unsigned char* smem_raw, float (*wm)[1], float (*wl)[1]) {
    constexpr int G = 1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int half = lane >> 4, hl = lane & 15;
    const long long cta = (long long)blockIdx.y * gridDim.x + blockIdx.x;
    // ---- 2. queries in the lane layout: dims {64j + 4hl + e} ----
    float q[G][4 * VPL];
#pragma unroll
    for (int r = 0; r < G; ++r) {
        const float4* qp = reinterpret_cast<const float4*>(qsrc + r * DH);
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
            float4 v = qp[j * LPR + hl];
            q[r][4 * j + 0] = v.x * a.scale_log2;
            q[r][4 * j + 1] = v.y * a.scale_log2;
            q[r][4 * j + 2] = v.z * a.scale_log2;
            q[r][4 * j + 3] = v.w * a.scale_log2;
        }
    }
    float m[G], l[G], acc[G][4 * VPL];
#pragma unroll
    for (int r = 0; r < G; ++r) {
        m[r] = -INFINITY;
        l[r] = 0.f;
#pragma unroll
        for (int e = 0; e < 4 * VPL; ++e) acc[r][e] = 0.f;
    }

    // ---- 3. gather (double-buffered 128-bit loads) + online softmax ----
    const float4* kb = reinterpret_cast<const float4*>(a.keys + (long long)p * a.kv_head_stride);
    const float4* vb = reinterpret_cast<const float4*>(a.values + (long long)p * a.kv_head_stride);
    const int slot = warp * 2 + half;          // 0..15
    constexpr int STEP = AT_WARPS * 2;         // rows per CTA step
    const uint64_t pol = l2_evict_first_policy();
    float4 kc[VPL], vc[VPL], kn[VPL], vn[VPL];
    // g > 1: a RING-deep cp.async pipeline per half-warp in shared memory
    // (each lane copies and later reads back only its own 16-byte chunks, so
    // no barrier is needed); g = 1: two rows in registers
    const int RING = a.ring4 ? 4 : 2;
    float4* ring = G > 1 ? reinterpret_cast<float4*>(smem_raw + a.ring_off) + (size_t)slot * RING * 64 : nullptr;
    auto issue = [&](int rr, int u) {
        if (rr < nrows) {
            const long long row = rows[rr];
#pragma unroll
            for (int j = 0; j < VPL; ++j) {
                cp_async16_hint(ring + u * 64 + j * LPR + hl, kb + row * (DH / 4) + j * LPR + hl, pol);
                cp_async16_hint(ring + u * 64 + 32 + j * LPR + hl, vb + row * (DH / 4) + j * LPR + hl, pol);
            }
        }
        cp_async_commit();
    };
    for (;;) {
    int ri = slot;
    if constexpr (G > 1) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (u < RING) issue(slot + u * STEP, u);
    } else if (ri < nrows) {
        const long long row = rows[ri];
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
            kc[j] = ldg_stream(kb + row * (DH / 4) + j * LPR + hl, pol);
            vc[j] = ldg_stream(vb + row * (DH / 4) + j * LPR + hl, pol);
        }
    }
    for (int it = 0; ri < nrows; ri += STEP, ++it) {  // half-warp uniform trip count
        if constexpr (G > 1) {
            if (a.ring4) cp_async_wait_group<3>();  // this half-warp's oldest row has landed
            else cp_async_wait_group<1>();
            const int u = it & (RING - 1);
#pragma unroll
            for (int j = 0; j < VPL; ++j) {
                kc[j] = ring[u * 64 + j * LPR + hl];
                vc[j] = ring[u * 64 + 32 + j * LPR + hl];
            }
            issue(ri + RING * STEP, u);
        } else {
            const int rn = ri + STEP;
            if (rn < nrows) {  // prefetch the next row of this half-warp
                const long long row = rows[rn];
#pragma unroll
                for (int j = 0; j < VPL; ++j) {
                    kn[j] = ldg_stream(kb + row * (DH / 4) + j * LPR + hl, pol);
                    vn[j] = ldg_stream(vb + row * (DH / 4) + j * LPR + hl, pol);
                }
            }
        }
#pragma unroll
        for (int r = 0; r < G; ++r) {
            float d = 0.f;
#pragma unroll
            for (int j = 0; j < VPL; ++j) {
                d = fmaf(q[r][4 * j + 0], kc[j].x, d);
                d = fmaf(q[r][4 * j + 1], kc[j].y, d);
                d = fmaf(q[r][4 * j + 2], kc[j].z, d);
                d = fmaf(q[r][4 * j + 3], kc[j].w, d);
            }
            d += __shfl_xor_sync(0xffffu << (half * 16), d, 1, 16);
            d += __shfl_xor_sync(0xffffu << (half * 16), d, 2, 16);
            d += __shfl_xor_sync(0xffffu << (half * 16), d, 4, 16);
            d += __shfl_xor_sync(0xffffu << (half * 16), d, 8, 16);
            if (d > m[r]) {  // lazy rescale: only when the running max grows
                const float alpha = safe_scale(m[r], d);
                l[r] *= alpha;
#pragma unroll
                for (int e = 0; e < 4 * VPL; ++e) acc[r][e] *= alpha;
                m[r] = d;
            }
            const float pw = exp2f(d - m[r]);
            l[r] += pw;
#pragma unroll
            for (int j = 0; j < VPL; ++j) {
                acc[r][4 * j + 0] = fmaf(pw, vc[j].x, acc[r][4 * j + 0]);
                acc[r][4 * j + 1] = fmaf(pw, vc[j].y, acc[r][4 * j + 1]);
                acc[r][4 * j + 2] = fmaf(pw, vc[j].z, acc[r][4 * j + 2]);
                acc[r][4 * j + 3] = fmaf(pw, vc[j].w, acc[r][4 * j + 3]);
            }
        }
        if constexpr (G == 1) {
#pragma unroll
            for (int j = 0; j < VPL; ++j) {
                kc[j] = kn[j];
                vc[j] = vn[j];
            }
        }
    }
    if constexpr (G > 1) cp_async_wait_all();
    {
        const int nn = refill(rows);  // the next window's rows, or < 0: done
        if (nn < 0) break;
        nrows = nn;
    }
    }

    if (a.prof) {
        __syncthreads();
        if (tid == 0) { a.prof[cta * PQKV_PROF_SLOTS + 3] = clock64(); a.prof[cta * PQKV_PROF_SLOTS + 6] = globaltimer_ns(); }
    }
    // ---- 4. merge the two half-warps (lanes hl and hl+16 hold the same dims) ----
#pragma unroll
    for (int r = 0; r < G; ++r) {
        float mo = __shfl_xor_sync(FULL, m[r], 16);
        float lo = __shfl_xor_sync(FULL, l[r], 16);
        float mn = fmaxf(m[r], mo);
        float sa = safe_scale(m[r], mn), sb = safe_scale(mo, mn);
        l[r] = l[r] * sa + lo * sb;
#pragma unroll
        for (int e = 0; e < 4 * VPL; ++e) {
            float ao = __shfl_xor_sync(FULL, acc[r][e], 16);
            acc[r][e] = acc[r][e] * sa + ao * sb;
        }
        m[r] = mn;
    }
    __syncthreads();  // every warp is past the gather loop: rows[] is free
    float* wacc = reinterpret_cast<float*>(smem_raw);  // [AT_WARPS][G][DH]
#pragma unroll
    for (int r = 0; r < G; ++r) {
        if (half == 0) {
#pragma unroll
            for (int j = 0; j < VPL; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) wacc[(warp * G + r) * DH + 64 * j + 4 * hl + e] = acc[r][4 * j + e];
            if (hl == 0) { wm[warp][r] = m[r]; wl[warp][r] = l[r]; }
        }
    }
    __syncthreads();

}

// ---- g > 1 gather: one warp per K/V row ----
// Each warp streams its rows (rows[warp], rows[warp + 8], ...) through a
// private ring of `depth` 1 KB slots in shared memory: every lane copies 16 B
// of the K row and 16 B of the V row with cp.async (one commit group per
// row, so cp.async.wait_group depth-1 means "the oldest row has landed"; no
// barrier -- each lane reads back only what it copied).  A lane holds dims
// 4*lane..4*lane+3 of the G query rows and accumulators (2*4*G floats: half
// the registers of the half-warp layout, so 4 CTAs fit per SM), and the G
// partial dots are reduced by a transpose-reduce: after the xor-16 (and for
// G = 4 xor-8) exchange a lane keeps a partial of one query row only, three
// (four) more shuffles complete it -- the lanes of group r then own row r's
// online-softmax state and broadcast its weight.  Measured on cfg3's shape
// (tools/microbench/gqa_probe.cu): 4.95 TB/s vs 4.2-4.35 TB/s for the
// half-warp-per-row ring.
template <int G, int NT, class Refill>
__device__ __forceinline__ void gather_rows_warp(const AtArgs& a, const float* qsrc, int p, int* rows, int nrows,
                                                 Refill& refill,
                                                 unsigned char* smem_raw, float (*wm)[G], float (*wl)[G],
                                                 unsigned* claim = nullptr) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float4* kb = reinterpret_cast<const float4*>(a.keys + (long long)p * a.kv_head_stride);
    const float4* vb = reinterpret_cast<const float4*>(a.values + (long long)p * a.kv_head_stride);
    const uint64_t pol = l2_evict_first_policy();
    const int depth = a.ring4 ? 4 : 2;
    float4* ring = reinterpret_cast<float4*>(smem_raw + a.ring_off) + (size_t)warp * depth * 64;
    float4 q[G];
#pragma unroll
    for (int r = 0; r < G; ++r) {
        const float4 v = reinterpret_cast<const float4*>(qsrc + r * DH)[lane];
        q[r] = make_float4(v.x * a.scale_log2, v.y * a.scale_log2, v.z * a.scale_log2, v.w * a.scale_log2);
    }
    const bool b4 = (lane & 16) != 0, b3 = (lane & 8) != 0;
    float m_own = -INFINITY, l_own = 0.f;  // state of query row `own` (lane group)
    float4 acc[G];
#pragma unroll
    for (int r = 0; r < G; ++r) acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (;;) {
        int mine = nrows > warp ? (nrows - warp + (NT / 32) - 1) / (NT / 32) : 0;
        // claim != null (wide CTAs): the warps take CLAIM rows at a time from
        // a shared counter, so all 32 finish within a row of each other; a
        // warp's first batch is rows [warp * CLAIM, warp * CLAIM + CLAIM)
        constexpr int CLAIM = 4;
        int q_base = warp * CLAIM, q_pos = 0, n_got = 0;
        bool dry = false;
        auto issue = [&](int it, int slot) {
            if (claim) {
                if (!dry) {
                    if (q_pos == CLAIM) {
                        int b = 0;
                        if (lane == 0) b = (int)atomicAdd(claim, (unsigned)CLAIM);
                        q_base = __shfl_sync(FULL, b, 0);
                        q_pos = 0;
                    }
                    const int i = q_base + q_pos++;
                    if (i < nrows) {
                        const long long row = rows[i];
                        cp_async16_hint(ring + slot * 64 + lane, kb + row * (DH / 4) + lane, pol);
                        cp_async16_hint(ring + slot * 64 + 32 + lane, vb + row * (DH / 4) + lane, pol);
                        ++n_got;
                    } else {
                        dry = true;
                    }
                }
            } else if (it < mine) {
                const long long row = rows[warp + (NT / 32) * it];
                cp_async16_hint(ring + slot * 64 + lane, kb + row * (DH / 4) + lane, pol);
                cp_async16_hint(ring + slot * 64 + 32 + lane, vb + row * (DH / 4) + lane, pol);
            }
            cp_async_commit();
        };
        for (int sl = 0; sl < depth; ++sl) issue(sl, sl);
        for (int it = 0; claim ? it < n_got : it < mine; ++it) {
            const int sl = it & (depth - 1);
            if (depth == 4) cp_async_wait_group<3>();
            else cp_async_wait_group<1>();
            const float4 k = ring[sl * 64 + lane], v = ring[sl * 64 + 32 + lane];
            issue(it + depth, sl);
            // packed fp32 (FFMA2 / FMUL2): half the FMA instructions of the
            // scalar form -- the g = 4 gather is close to issue-bound
            float d[G];
            const float2 kxy = make_float2(k.x, k.y), kzw = make_float2(k.z, k.w);
#pragma unroll
            for (int r = 0; r < G; ++r) {
                const float2 t2 =
                    __ffma2_rn(make_float2(q[r].z, q[r].w), kzw, __fmul2_rn(make_float2(q[r].x, q[r].y), kxy));
                d[r] = t2.x + t2.y;
            }
            float x;
            if constexpr (G == 4) {
                float a0 = b4 ? d[2] : d[0], a1 = b4 ? d[3] : d[1];
                const float s0 = b4 ? d[0] : d[2], s1 = b4 ? d[1] : d[3];
                a0 += __shfl_xor_sync(FULL, s0, 16);
                a1 += __shfl_xor_sync(FULL, s1, 16);
                x = b3 ? a1 : a0;
                x += __shfl_xor_sync(FULL, b3 ? a0 : a1, 8);
            } else {  // G == 2: own row = bit 4
                x = b4 ? d[1] : d[0];
                x += __shfl_xor_sync(FULL, b4 ? d[0] : d[1], 16);
                x += __shfl_xor_sync(FULL, x, 8);
            }
            x += __shfl_xor_sync(FULL, x, 4);
            x += __shfl_xor_sync(FULL, x, 2);
            x += __shfl_xor_sync(FULL, x, 1);
            float alpha = 1.f;
            if (x > m_own) {  // lazy rescale: only when the running max grows
                alpha = safe_scale(m_own, x);
                l_own *= alpha;
                m_own = x;
            }
            const float pw = exp2f(x - m_own);
            l_own += pw;
            const bool grew = __any_sync(FULL, alpha != 1.f);
            constexpr int GRP = 32 / G;  // lanes per query row group
#pragma unroll
            for (int r = 0; r < G; ++r) {
                const float pr = __shfl_sync(FULL, pw, GRP * r);
                float2 axy = make_float2(acc[r].x, acc[r].y), azw = make_float2(acc[r].z, acc[r].w);
                if (grew) {
                    const float ar = __shfl_sync(FULL, alpha, GRP * r);
                    axy = __fmul2_rn(axy, make_float2(ar, ar));
                    azw = __fmul2_rn(azw, make_float2(ar, ar));
                }
                axy = __ffma2_rn(make_float2(pr, pr), make_float2(v.x, v.y), axy);
                azw = __ffma2_rn(make_float2(pr, pr), make_float2(v.z, v.w), azw);
                acc[r] = make_float4(axy.x, axy.y, azw.x, azw.y);
            }
        }
        cp_async_wait_all();
        if (claim) break;  // wide plans keep whole lists (no windows)
        const int nn = refill(rows);  // the next window's rows, or < 0: done
        if (nn < 0) break;
        nrows = nn;
    }
    if (a.prof) {
        __syncthreads();
        const long long cta = (long long)blockIdx.y * gridDim.x + blockIdx.x;
        if (tid == 0) { a.prof[cta * PQKV_PROF_SLOTS + 3] = clock64(); a.prof[cta * PQKV_PROF_SLOTS + 6] = globaltimer_ns(); }
    }
    __syncthreads();  // every warp is past the gather loop: rows[] is free
    // this warp's partial (m, l, acc per query row) -> the per-warp merge area
    float* wacc = reinterpret_cast<float*>(smem_raw);  // [(NT / 32)][G][DH]
    constexpr int GRP = 32 / G;
#pragma unroll
    for (int r = 0; r < G; ++r) {
        const float mr = __shfl_sync(FULL, m_own, GRP * r), lr = __shfl_sync(FULL, l_own, GRP * r);
        reinterpret_cast<float4*>(wacc + (warp * G + r) * DH)[lane] = acc[r];
        if (lane == 0) {
            wm[warp][r] = mr;
            wl[warp][r] = lr;
        }
    }
    __syncthreads();
}

// Per-warp partials (wacc / wm / wl in shared memory) -> this CTA's partial
// part[p][c] = (M, L, O[d]) per query row.
template <int G, int NT = AT_THREADS>
__device__ __forceinline__ void write_partial(const AtArgs& a, int p, int c, unsigned char* smem_raw, float (*wm)[G],
                                              float (*wl)[G]) {
    const float* wacc = reinterpret_cast<const float*>(smem_raw);  // [(NT / 32)][G][DH]
    // per (warp, row) scale to the CTA's running max, computed once: [G][NT/32]
    __shared__ float wsc[G][NT / 32], wmax[G], wsum[G];
    if (threadIdx.x < G * 32) {
        const int r = threadIdx.x / 32, ln = threadIdx.x % 32;
        float M = -INFINITY;
        for (int w = ln; w < (NT / 32); w += 32) M = fmaxf(M, wm[w][r]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(FULL, M, o));
        float L = 0.f;
        for (int w = ln; w < (NT / 32); w += 32) {
            const float sc = M != -INFINITY ? safe_scale(wm[w][r], M) : 0.f;
            wsc[r][w] = sc;
            L += wl[w][r] * sc;
        }
        L = warp_sum(L);
        if (ln == 0) { wmax[r] = M; wsum[r] = L; }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < G * DH; e += NT) {
        const int r = e / DH, d = e % DH;
        float O = 0.f;
#pragma unroll 8
        for (int w = 0; w < (NT / 32); ++w) O = fmaf(wacc[(w * G + r) * DH + d], wsc[r][w], O);
        float* o = a.part + (((long long)p * a.n_chunks + c) * G + r) * (DH + 2);
        o[2 + d] = O;
        if (d == 0) { o[0] = wmax[r]; o[1] = wsum[r]; }
    }
}

// Merges n partial results (pb: [n][G][DH + 2] = running max, sum of
// weights, unnormalised output) into dst_out [G][DH] (normalised) or, when
// dst_part is set, into one partial [G][DH + 2].  m and l of every partial
// are read in one pass; the output sums read 2 x 16 partial values in flight
// per thread (the merge sits on the kernel's critical tail, so its cost is
// the number of dependent L2 round trips).
constexpr int MERGE_GROUP = 8;

template <int G, int NT = AT_THREADS>
__device__ __forceinline__ void merge_parts(const float* pb, int n, float* dst_part, float* dst_out,
                                            unsigned char* smem_raw) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    float* sm = reinterpret_cast<float*>(smem_raw) + (NT / 32) * G * DH;  // [G][n]: m, then the scale
    float* sl = sm + G * n;                                                // [G][n]: l
    float* sml = sl + G * n;                                               // [G][2]: M, L
    const long long cstr = (long long)G * (DH + 2);
    // this thread's outputs (one, or two when G * DH > NT): their first PF
    // partial values are loaded before m and l, so both round trips overlap
    constexpr bool TWO = G * DH > NT;
    constexpr int PF = TWO ? 16 : 32;
    const int e0 = tid, e1 = tid + NT;
    const bool has0 = e0 < G * DH, has1 = TWO && e1 < G * DH;
    const int r0 = has0 ? e0 / DH : 0, d0 = has0 ? e0 % DH : 0, r1 = has1 ? e1 / DH : 0, d1 = has1 ? e1 % DH : 0;
    const float* p0 = pb + (long long)r0 * (DH + 2) + 2 + d0;
    const float* p1 = pb + (long long)r1 * (DH + 2) + 2 + d1;
    float v0[PF], v1[TWO ? PF : 1];
#pragma unroll
    for (int u = 0; u < PF; ++u) {
        v0[u] = has0 && u < n ? __ldcg(p0 + u * cstr) : 0.f;
        if constexpr (TWO) v1[u] = has1 && u < n ? __ldcg(p1 + u * cstr) : 0.f;
    }
    for (int i = tid; i < n * G; i += NT) {  // i = cc * G + r
        const float* pc = pb + (long long)i * (DH + 2);
        const int cc = i / G, r = i - cc * G;
        sm[r * n + cc] = __ldcg(pc);
        sl[r * n + cc] = __ldcg(pc + 1);
    }
    __syncthreads();
    for (int r = warp; r < G; r += (NT / 32)) {
        float M = -INFINITY;
        for (int cc = lane; cc < n; cc += 32) M = fmaxf(M, sm[r * n + cc]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(FULL, M, o));
        float L = 0.f;
        for (int cc = lane; cc < n; cc += 32) {
            const float f = safe_scale(sm[r * n + cc], M);
            sm[r * n + cc] = f;
            L += sl[r * n + cc] * f;
        }
        L = warp_sum(L);
        if (lane == 0) { sml[2 * r] = M; sml[2 * r + 1] = L; }
    }
    __syncthreads();
    {
        const float* f0 = sm + r0 * n;
        const float* f1 = sm + r1 * n;
        float O0 = 0.f, O1 = 0.f;
#pragma unroll
        for (int u = 0; u < PF; ++u)
            if (u < n) {
                O0 = fmaf(v0[u], f0[u], O0);
                if constexpr (TWO) O1 = fmaf(v1[u], f1[u], O1);
            }
        for (int cc = PF; cc < n; cc += PF) {
#pragma unroll
            for (int u = 0; u < PF; ++u) {
                v0[u] = has0 && cc + u < n ? __ldcg(p0 + (cc + u) * cstr) : 0.f;
                if constexpr (TWO) v1[u] = has1 && cc + u < n ? __ldcg(p1 + (cc + u) * cstr) : 0.f;
            }
#pragma unroll
            for (int u = 0; u < PF; ++u)
                if (cc + u < n) {
                    O0 = fmaf(v0[u], f0[cc + u], O0);
                    if constexpr (TWO) O1 = fmaf(v1[u], f1[cc + u], O1);
                }
        }
        if (dst_out) {
            if (has0) dst_out[e0] = O0 / sml[2 * r0 + 1];
            if (has1) dst_out[e1] = O1 / sml[2 * r1 + 1];
        } else {
            if (has0) dst_part[r0 * (DH + 2) + 2 + d0] = O0;
            if (has1) dst_part[r1 * (DH + 2) + 2 + d1] = O1;
        }
    }
    for (int e = tid + 2 * NT; e < G * DH; e += NT) {  // G * DH > 2 NT (not instantiated today)
        const int r = e / DH, d = e % DH;
        const float* pe = pb + (long long)r * (DH + 2) + 2 + d;
        float O = 0.f;
        for (int cc = 0; cc < n; ++cc) O = fmaf(__ldcg(pe + cc * cstr), sm[r * n + cc], O);
        if (dst_out) dst_out[e] = O / sml[2 * r + 1];
        else dst_part[r * (DH + 2) + 2 + d] = O;
    }
    if (dst_part && tid < G) {
        dst_part[tid * (DH + 2)] = sml[2 * tid];
        dst_part[tid * (DH + 2) + 1] = sml[2 * tid + 1];
    }
}

// MODE: 0 = the list modes (rows / bitmap / tuple classes, a.src at run
// time), SRC_PAIRS or SRC_KEYS -- the fused single-launch modes get their own
// instantiation so their prologues do not perturb the others' code.
template <int G, int MODE, int NT = AT_THREADS>
__global__ void __launch_bounds__(NT, NT == 2 * AT_THREADS ? 2 : NT > AT_THREADS ? 1 : ((MODE == SRC_KEYS && G > 1) ? 2 : 4)) attend_kernel(AtArgs a) {
    const int src = MODE == 0 ? a.src : MODE;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ uint32_t wtot[(NT / 32)];
    __shared__ int nrows_s;
    __shared__ float wm[(NT / 32)][G], wl[(NT / 32)][G];

    const int p = blockIdx.y, c = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nwords = a.chunk / 32;
    int* rows = reinterpret_cast<int*>(smem_raw);
    uint32_t* words = reinterpret_cast<uint32_t*>(smem_raw + a.region);
    uint32_t* eqw = words + nwords;
    uint8_t* cls = reinterpret_cast<uint8_t*>(eqw + nwords);

    const long long cta = (long long)blockIdx.y * gridDim.x + blockIdx.x;
    if (a.prof && tid == 0) {
        a.prof[cta * PQKV_PROF_SLOTS + 0] = clock64();
        a.prof[cta * PQKV_PROF_SLOTS + 4] = globaltimer_ns();
        unsigned smid, crk;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crk));
        a.prof[cta * PQKV_PROF_SLOTS + 16] = smid;
        a.prof[cta * PQKV_PROF_SLOTS + 17] = crk;
        a.prof[cta * PQKV_PROF_SLOTS + 18] = (MODE == SRC_PAIRS) && crk == (cta / 8) % 8;
    }
    // ---- 0. programmatic dependent launch ----
    // Launched with programmatic stream serialization, this grid may start
    // while the previous kernel on the stream is still draining.  Until
    // griddepcontrol.wait returns it only warms L2 and the TLBs with
    // prefetches of what its prologue reads (no loads: the previous kernel
    // may still be writing them); it then lets the next decode launch early.
    if (MODE == SRC_PAIRS) {
        const int C2 = a.C * a.C;
        const int r0 = c * a.chunk, r1 = min(a.s_mid, r0 + a.chunk);
        const char* cd = reinterpret_cast<const char*>(a.codes + p * a.codes_head_stride + 2 * (long long)r0);
        for (int o = tid * 128; o < 4 * (r1 - r0); o += NT * 128) prefetch_l2(cd + o);
        if ((c & 7) == 0 || NT > AT_THREADS) {  // the selecting CTAs: the head's select tables
            const char* ce = reinterpret_cast<const char*>(a.centroids + (long long)p * 2 * a.C * (DH / 2));
            for (int o = tid * 128; o < 4 * a.C * DH; o += NT * 128) prefetch_l2(ce + o);
            const char* th = reinterpret_cast<const char*>(a.thist + (long long)p * C2);
            for (int o = tid * 128; o < 4 * C2; o += NT * 128) prefetch_l2(th + o);
        }
    }
    // wide pair CTAs (each its own selector, nothing else in shared memory
    // yet) stage the centroid table of their pair select before the wait: no
    // kernel that lets this grid launch early writes centroids
    bool cen_pre = false;
    if (MODE == SRC_PAIRS && NT > AT_THREADS) {
        PairScratch ps0(smem_raw, a.C, a.n_tchunks);
        const float* cen = a.centroids + (long long)p * 2 * a.C * (DH / 2);
        float4* stage = pair_lut_stage(a.C, DH, ps0.hist);
        // = build_lut's staging predicate: the queries come from q_sh (16-byte aligned), d_m = 64
        cen_pre = stage && (reinterpret_cast<uintptr_t>(cen) & 15) == 0;
        if (cen_pre) stage_centroids(cen, DH, 2, a.C, stage);
    }
    if (MODE == SRC_KEYS) {  // this CTA's code rows and its share of the centroids (ADC table)
        const int r0 = c * a.chunk, r1 = min(a.s_mid, r0 + a.chunk);
        const char* cd = reinterpret_cast<const char*>(a.codes + p * a.codes_head_stride + (long long)r0 * a.m);
        const uint32_t bytes = 2u * a.m * (uint32_t)max(0, r1 - r0);
        if ((reinterpret_cast<uintptr_t>(cd) & 15) == 0) {  // one bulk (TMA) prefetch of the rows
            if (tid == 0 && bytes >= 16)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(cd), "r"(bytes & ~15u) : "memory");
        } else {
            for (int o = tid * 128; o < (int)bytes; o += NT * 128) prefetch_l2(cd + o);
        }
        unsigned crk, ncl;
        asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(crk));
        asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(ncl));
        const int me = a.m * a.C, share = (me + (int)ncl - 1) / (int)ncl;
        const int e0 = min(me, (int)crk * share), e1 = min(me, e0 + share);
        const char* ce = reinterpret_cast<const char*>(a.centroids + (long long)p * a.C * DH) + (long long)e0 * (DH / a.m) * 4;
        for (int o = tid * 128; o < (e1 - e0) * (DH / a.m) * 4; o += NT * 128) prefetch_l2(ce + o);
    }
    // split pair path (SRC_TUPLE): stage this CTA's code pairs while the
    // select grid (the previous kernel) runs -- the codes are not written by
    // it, and it waited for their producer before letting this grid launch
    const uint32_t* tup_staged = nullptr;
    if (MODE == 0 && a.src == SRC_TUPLE && a.stage) {
        const int r0 = c * a.chunk, r1 = min(a.s_mid, r0 + a.chunk), n = max(0, r1 - r0);
        const uint32_t* src = reinterpret_cast<const uint32_t*>(a.codes + p * a.codes_head_stride) + r0;
        uint32_t* dst = reinterpret_cast<uint32_t*>(smem_raw);
        int head = 0;
        if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
            head = n & ~3;
            for (int f = tid; f < head / 4; f += NT) cp_async16(dst + 4 * code_swz(f), src + 4 * f);
        }
        for (int e = head + tid; e < n; e += NT) cp_async4(dst + 4 * code_swz(e >> 2) + (e & 3), src + e);
        cp_async_commit();
        tup_staged = dst;
    }
    if (a.ready_in) {
        // split key / pair paths: the bitmap of this unit is complete once its select
        // CTAs have counted in (the select grid waited for everything before
        // it, and its release publishes that too), so the gather does not
        // wait for the slowest unit's select
        if (tid == 0) {
            unsigned v;
            for (;;) {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.ready_in + p) : "memory");
                if (v >= a.ready_need) break;
                __nanosleep(64);
            }
        }
        __syncthreads();
    } else {
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    asm volatile("griddepcontrol.launch_dependents;");
    // g > 1: this head's G query rows, read once into shared memory (they
    // may sit in page-locked host memory: pqkv_decode_host passes mapped
    // queries straight through).  g = 1 reads them from global memory (the
    // shared copy cost the north star's gather ~9 us: bimodal CTA spans).
    __shared__ __align__(16) float q_sh[G > 1 ? G * DH : 4];
    const float* q_s = a.queries + (long long)p * G * DH;
    if constexpr (G > 1) {
        for (int i = tid; i < G * DH / 4; i += NT)
            reinterpret_cast<float4*>(q_sh)[i] = reinterpret_cast<const float4*>(q_s)[i];
        __syncthreads();
        q_s = q_sh;
    }
    // ---- 1. this CTA's row list (ascending token ids) ----
    int nrows = 0;
    int sel_total = 0;  // windowed list: selected middle rows of this CTA (0: one window)
    if (src == SRC_ROWS) {
        const int b0 = c * a.chunk, cnt = max(0, min(a.chunk, a.t - b0));
        for (int e = tid; e < cnt; e += NT) rows[e] = (int)a.rows[(long long)p * a.t + b0 + e];
        nrows = cnt;
    } else {
        if (c == 0 && (MODE != SRC_PAIRS) && (MODE != SRC_KEYS) && !tup_staged)  // written after the select (shared region)
            for (int e = tid; e < a.n_init; e += NT) rows[e] = e;
        nrows = c == 0 ? a.n_init : 0;
        const int r0 = c * a.chunk, r1 = min(a.s_mid, r0 + a.chunk);
        const int nw = (max(0, r1 - r0) + 31) / 32;
        if (src == SRC_BITMAP) {
            for (int w = tid; w < nw; w += NT) words[w] = a.bitmap[(long long)p * a.words + r0 / 32 + w];
        } else if ((MODE == SRC_KEYS)) {
            __shared__ uint32_t pub_s[4], sh_s[8];
            keys_select_words<G>(a, q_s, p, r0, r1, smem_raw, words, eqw /* [2][NB/2] in keys mode */, pub_s, wtot, sh_s,
                                 a.prof ? a.prof + cta * PQKV_PROF_SLOTS + 8 : nullptr);
            if (a.prof && tid == 0) a.prof[cta * PQKV_PROF_SLOTS + 1] = clock64();
            if (a.sel_only) {  // select-only launch: the bitmap-mode attention follows
                for (int w = tid; w < nw; w += NT) {
                    a.sel_only[(long long)p * a.words + r0 / 32 + w] = words[w];
                    if (a.sel_dump) a.sel_dump[(long long)p * a.words + r0 / 32 + w] = words[w];
                }
                // this unit's gather CTAs start as soon as its 8 select CTAs are done
                __syncthreads();
                if (a.ready_out && tid == 0) {
                    __threadfence();
                    atomicAdd(&a.ready_out[p], 1u);
                }
                asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
                return;
            }
            if (c == 0)
                for (int e = tid; e < a.n_init; e += NT) rows[e] = e;
        } else if ((MODE == SRC_PAIRS)) {
            // per-head pair-level top-k: computed by one CTA of each thread-block
            // cluster and shared with the others through DSMEM.  The selecting
            // rank rotates with the cluster index: the scheduler places equal
            // ranks of neighbouring clusters on the same SM, so a fixed rank
            // would stack up to four latency-bound selects on one SM.
            namespace cg = cooperative_groups;
            cg::cluster_group cluster = cg::this_cluster();
            const unsigned crank = cluster.block_rank();
            const unsigned ncl = cluster.num_blocks();
            const unsigned sel = (unsigned)(cta / ncl) % ncl;
            // this CTA's code pairs (4 B per token): the other CTAs stage them
            // in shared memory (cp.async, rows[] region) while the selector
            // works; the selector reads them from L2 (prefetched)
            const uint32_t* cd_g = reinterpret_cast<const uint32_t*>(a.codes + p * a.codes_head_stride);
            const uint32_t* staged = nullptr;
            auto stage_codes = [&](uint32_t* dst) {
                const int n = max(0, r1 - r0);
                const uint32_t* src = cd_g + r0;
                int head = 0;
                if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
                    head = n & ~3;
                    for (int f = tid; f < head / 4; f += NT) cp_async16(dst + 4 * code_swz(f), src + 4 * f);
                }
                for (int e = head + tid; e < n; e += NT) cp_async4(dst + 4 * code_swz(e >> 2) + (e & 3), src + e);
                cp_async_commit();
            };
            {
                const int n = max(0, r1 - r0);
                const uint32_t* src = cd_g + r0;
                if (crank == sel || !a.stage) {
                    for (int o = tid * 32; o < n; o += NT * 32) prefetch_l2(src + o);
                } else {
                    stage_codes(reinterpret_cast<uint32_t*>(smem_raw));
                    staged = reinterpret_cast<const uint32_t*>(smem_raw);
                }
            }
            __shared__ uint32_t cut_s[2];
            const int C = a.C, C2 = C * C;
            if (crank == sel) {
                PairScratch ps(smem_raw, C, a.n_tchunks);  // aliases rows[]: free until expansion
                pair_select<NT, (4096 + NT - 1) / NT>(q_s, G, DH,
                                            a.centroids + (long long)p * 2 * C * (DH / 2), C,
                                            a.thist + (long long)p * C2, a.chist + (long long)p * a.tchunk_stride * C2,
                                            a.n_tchunks, a.k, ps.lut, ps.hist, ps.cnt, ps.lst, ps.ceq, ps.wsum, ps.sh, cls,
                                            nullptr, a.prof ? a.prof + cta * PQKV_PROF_SLOTS + 8 : nullptr, cen_pre);
                const uint32_t* sh = ps.sh;
                if (tid == 0) { cut_s[0] = sh[3]; cut_s[1] = sh[4]; }
            }
            cluster.sync();
            if (a.prof && tid == 0) a.prof[cta * PQKV_PROF_SLOTS + 15] = clock64();
            if (crank != sel) {
                const uint32_t* rc = cluster.map_shared_rank(reinterpret_cast<const uint32_t*>(cls), sel);
                for (int e = tid; e < (C2 + 3) / 4; e += NT) reinterpret_cast<uint32_t*>(cls)[e] = rc[e];
                if (tid < 2) cut_s[tid] = cluster.map_shared_rank(cut_s, sel)[tid];
            }
            // the selector's cls[]/cut_s are never written again; its exit is
            // held back by the matching cluster wait at the end of the kernel
            asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
            __syncthreads();
            if (a.prof && tid == 0) a.prof[cta * PQKV_PROF_SLOTS + 1] = clock64();
            const int cstar = (int)cut_s[0];
            const uint32_t take = cut_s[1];
            cp_async_wait_all();
            __syncthreads();
            if (a.prof && tid == 0) a.prof[cta * PQKV_PROF_SLOTS + 19] = clock64();
            classify_range<false, NT>(a, r0, r1, cd_g, staged, words, eqw, cls, wtot, cstar, take);
            if (a.prof && tid == 0) a.prof[cta * PQKV_PROF_SLOTS + 20] = clock64();
            if (c == 0)  // after the staged codes are consumed (they share rows[])
                for (int e = tid; e < a.n_init; e += NT) rows[e] = e;
        } else {
            const int C2 = a.C * a.C;
            if ((C2 & 3) == 0) {
                const uint32_t* src = reinterpret_cast<const uint32_t*>(a.cls + (long long)p * C2);
                for (int e = tid; e < C2 / 4; e += NT) reinterpret_cast<uint32_t*>(cls)[e] = src[e];
            } else {
                for (int e = tid; e < C2; e += NT) cls[e] = a.cls[(long long)p * C2 + e];
            }
            if (tup_staged) cp_async_wait_all();
            __syncthreads();
            classify_range<false, NT>(a, r0, r1, reinterpret_cast<const uint32_t*>(a.codes + p * a.codes_head_stride),
                                      tup_staged, words, eqw, cls, wtot, a.cut[2 * p], (uint32_t)a.cut[2 * p + 1]);
            if (c == 0 && tup_staged)  // after the staged codes are consumed (they share rows[])
                for (int e = tid; e < a.n_init; e += NT) rows[e] = e;
        }
        __syncthreads();
        if (a.sel_dump && ((MODE == SRC_PAIRS) || (MODE == SRC_KEYS) || src == SRC_TUPLE))
            for (int w = tid; w < nw; w += NT) a.sel_dump[(long long)p * a.words + r0 / 32 + w] = words[w];
        if (a.win >= a.chunk) {
            nrows += expand_words<NT>(words, nw, a.n_init + r0, rows, nrows, wtot);
            sel_total = 0;
        } else {  // windowed: the first a.win selected middle rows now, the rest after each gather window
            uint32_t t = 0;
            for (int w = tid; w < nw; w += NT) t += __popc(words[w]);
            t = warp_sum(t);
            if (lane == 0) wtot[warp] = t;
            __syncthreads();
            t = 0;
#pragma unroll
            for (int w = 0; w < (NT / 32); ++w) t += wtot[w];
            __syncthreads();
            sel_total = (int)t;
            nrows += expand_words_range<NT>(words, nw, a.n_init + r0, rows, nrows, 0u, (uint32_t)a.win, wtot);
        }
        if (c == a.n_chunks - 1 && sel_total <= a.win) {
            for (int e = tid; e < a.n_local; e += NT) rows[nrows + e] = a.total - a.n_local + e;
            nrows += a.n_local;
        }
    }
    if (tid == 0) nrows_s = nrows;
    __syncthreads();
    nrows = nrows_s;
    if (a.prof && tid == 0) { a.prof[cta * PQKV_PROF_SLOTS + 2] = clock64(); a.prof[cta * PQKV_PROF_SLOTS + 5] = globaltimer_ns(); }

    WindowRefill<NT> refill{a, c, words, wtot, sel_total, 0};
    if constexpr (G == 1) {
        gather_rows_halfwarp(a, q_s, p, rows, nrows, refill, smem_raw, wm, wl);
    } else if (NT > AT_THREADS && a.claim) {
        __shared__ unsigned claim_ctr;
        if (tid == 0) claim_ctr = (unsigned)(NT / 32) * 4u;  // the warps' first batches are static
        __syncthreads();
        gather_rows_warp<G, NT>(a, q_s, p, rows, nrows, refill, smem_raw, wm, wl, &claim_ctr);
    } else {
        gather_rows_warp<G, NT>(a, q_s, p, rows, nrows, refill, smem_raw, wm, wl);
    }
    // ---- 5. merge warps, write this CTA's partial ----
    write_partial<G, NT>(a, p, c, smem_raw, wm, wl);

    // ---- 6. the last CTA of this head merges all partials (no extra launch);
    // many chunks: the last CTA of each group of MERGE_GROUP merges the
    // group's partials, the last group's merger merges the group partials ----
    __shared__ unsigned ticket;
    __threadfence();
    __syncthreads();
    unsigned* grp_ctr = a.part2 ? a.arrivals + gridDim.y + (long long)p * a.n_groups + c / MERGE_GROUP : nullptr;
    if (tid == 0) ticket = atomicAdd(a.part2 ? grp_ctr : &a.arrivals[p], 1u);
    // pair mode: pairs with the cluster arrive after the DSMEM reads (no CTA
    // of the cluster exits while another may still read its shared memory)
    if ((MODE == SRC_PAIRS) || (MODE == SRC_KEYS)) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    __syncthreads();
    if (a.prof && tid == 0) a.prof[cta * PQKV_PROF_SLOTS + 7] = globaltimer_ns();
    const float* pb = a.part + (long long)p * a.n_chunks * G * (DH + 2);
    if (a.part2) {
        const int g0 = c / MERGE_GROUP * MERGE_GROUP, gn = min(MERGE_GROUP, a.n_chunks - g0);
        if (ticket != (unsigned)gn - 1) return;
        __threadfence();
        float* gp = a.part2 + ((long long)p * a.n_groups + c / MERGE_GROUP) * G * (DH + 2);
        merge_parts<G, NT>(pb + (long long)g0 * G * (DH + 2), gn, gp, nullptr, smem_raw);
        if (tid == 0) *grp_ctr = 0;
        __threadfence();
        __syncthreads();
        if (tid == 0) ticket = atomicAdd(&a.arrivals[p], 1u);
        __syncthreads();
        if (ticket != (unsigned)a.n_groups - 1) return;
        __threadfence();
        merge_parts<G, NT>(a.part2 + (long long)p * a.n_groups * G * (DH + 2), a.n_groups, nullptr,
                       a.out + (long long)p * G * DH, smem_raw);
    } else {
        if (ticket != (unsigned)a.n_chunks - 1) return;
        __threadfence();
        merge_parts<G, NT>(pb, a.n_chunks, nullptr, a.out + (long long)p * G * DH, smem_raw);
    }
    if (tid == 0) {
        a.arrivals[p] = 0;  // ready for the next launch on this stream
        if (a.ready_in) a.ready_in[p] = 0;
    }
    if (a.prof && tid == 0) a.prof[cta * PQKV_PROF_SLOTS + 7] = globaltimer_ns();
}

// ---- exact (fp64) path ------------------------------------------------------

// exact_scores (attention.cpp:11-26) for every (head, query row, list row).
__global__ void exact_scores_kernel(const float* queries, int G, int d_h, const float* keys,
                                    long long kv_head_stride, const int64_t* rows, int t,
                                    double scale, float* scores) {
    const int pr = blockIdx.y, p = pr / G;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= t) return;
    const float* q = queries + (long long)pr * d_h;
    const float* k = keys + p * kv_head_stride + rows[(long long)p * t + i] * d_h;
    double acc = 0.0;
    for (int j = 0; j < d_h; ++j) acc = __fma_rn((double)__ldg(q + j), (double)__ldg(k + j), acc);
    scores[(long long)pr * t + i] = (float)__dmul_rn(acc, scale);
}

// softmax_attention (attention.cpp:35-60) given the f32 scores:
// softmax_weights_kernel (max_element, exp of max-subtracted scores, the
// serial fp64 total in row order, w / total), then weighted_products_kernel +
// sum_chain_kernel (acc[j] += w_i * v_ij in row order per output dim).  Same operations and
// order as the reference; the serial chains read their operands from shared
// memory / registers filled ahead of them, so they run at add latency.
constexpr int SW_THREADS = 1024, SW_CHUNK = 4096;

__global__ void __launch_bounds__(SW_THREADS) softmax_weights_kernel(const float* scores, int t, double* w) {
    const int pr = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float* sc = scores + (long long)pr * t;
    double* wr = w + (long long)pr * t;
    __shared__ float smax[32];
    __shared__ double buf[SW_CHUNK];
    __shared__ double stotal;
    float mx = -INFINITY;
    for (int i = tid; i < t; i += SW_THREADS) mx = fmaxf(mx, sc[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, o));
    if (lane == 0) smax[warp] = mx;
    __syncthreads();
    if (tid == 0) {
        float v = smax[0];
        for (int e = 1; e < SW_THREADS / 32; ++e) v = fmaxf(v, smax[e]);
        smax[0] = v;
    }
    __syncthreads();
    const double max_score = (double)smax[0];
    double total = 0.0;  // thread 0's serial running total
    for (int c0 = 0; c0 < t; c0 += SW_CHUNK) {
        const int cnt = min(SW_CHUNK, t - c0);
        for (int i = tid; i < cnt; i += SW_THREADS) {
            const double e = exp(__dsub_rn((double)sc[c0 + i], max_score));
            buf[i] = e;
            wr[c0 + i] = e;
        }
        __syncthreads();
        if (tid == 0) {
            int i = 0;
            for (; i + 8 <= cnt; i += 8) {
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = buf[i + u];
#pragma unroll
                for (int u = 0; u < 8; ++u) total = __dadd_rn(total, v[u]);
            }
            for (; i < cnt; ++i) total = __dadd_rn(total, buf[i]);
        }
        __syncthreads();
    }
    if (tid == 0) stotal = total;
    __syncthreads();
    const double tot = stotal;
    for (int i = tid; i < t; i += SW_THREADS) wr[i] = __ddiv_rn(wr[i], tot);
}

// The output sum is one serial fp64 chain per (query row, dim): acc +=
// w_i * v_ij in row order.  The products are independent, so
// weighted_products_kernel forms them with the whole GPU (the row gather)
// into a [dim group][rows][32] fp64 block, and sum_chain_kernel runs the
// chains: one warp per 32 dims, lane = dim, the group's contiguous rows
// streamed through a shared-memory ring by bulk copies (one lane issues one
// cp.async.bulk per 32-row stage, completion on an mbarrier) SC_STAGES
// stages ahead of the adds, so each add waits only on the previous one.
constexpr int SC_DIMS = 32, SC_STAGE = 32, SC_STAGES = 16;  // 16 x 32 rows x 256 B = 128 KB ring
constexpr size_t SC_SMEM = (size_t)SC_STAGES * SC_STAGE * SC_DIMS * sizeof(double) + SC_STAGES * 8;

__global__ void weighted_products_kernel(int G, int d_h, int ldp, const float* values, long long kv_head_stride,
                                         const int64_t* rows, int t, const double* w, int pr0, double* prod) {
    const int pr = pr0 + blockIdx.y, p = pr / G;
    const long long n = (long long)t * ldp;
    const float* vb = values + p * kv_head_stride;
    const int64_t* rr = rows + (long long)p * t;
    const double* wr = w + (long long)pr * t;
    double* out = prod + (long long)blockIdx.y * n;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(e / ldp), j = (int)(e - (long long)i * ldp);
        const double v = j < d_h ? __dmul_rn(wr[i], (double)__ldg(vb + rr[i] * d_h + j)) : 0.0;
        out[((long long)(j / SC_DIMS) * t + i) * SC_DIMS + (j % SC_DIMS)] = v;
    }
}

__global__ void __launch_bounds__(SC_DIMS) sum_chain_kernel(int d_h, int ldp, int t, const double* prod, int pr0,
                                                            float* out) {
    extern __shared__ __align__(128) double ring[];  // [SC_STAGES][SC_STAGE][SC_DIMS], then the mbarriers
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)SC_STAGES * SC_STAGE * SC_DIMS);
    const int lane = threadIdx.x, j0 = blockIdx.x * SC_DIMS;
    const double* src = prod + ((long long)blockIdx.y * ldp / SC_DIMS + blockIdx.x) * (long long)t * SC_DIMS;
    const int n_stages = (t + SC_STAGE - 1) / SC_STAGE;
    const unsigned ring_s = (unsigned)__cvta_generic_to_shared(ring), full_s = (unsigned)__cvta_generic_to_shared(full);
    if (lane == 0) {
        for (int b = 0; b < SC_STAGES; ++b)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(full_s + b * 8) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    auto issue = [&](int s) {  // lane 0: stage s into slot s % SC_STAGES
        if (s >= n_stages) return;
        const int slot = s % SC_STAGES;
        const unsigned bytes = (unsigned)(min(SC_STAGE, t - s * SC_STAGE) * SC_DIMS * sizeof(double));
        const unsigned bar = full_s + slot * 8, dst = ring_s + slot * (SC_STAGE * SC_DIMS * 8);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(dst), "l"(src + (long long)s * SC_STAGE * SC_DIMS), "r"(bytes), "r"(bar) : "memory");
    };
    if (lane == 0)
        for (int s = 0; s < SC_STAGES; ++s) issue(s);
    double acc = 0.0;
#pragma unroll 1
    for (int s = 0; s < n_stages; ++s) {
        const int slot = s % SC_STAGES;
        const unsigned parity = (unsigned)(s / SC_STAGES) & 1u;
        unsigned done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(full_s + slot * 8), "r"(parity) : "memory");
        const double* cur = ring + (size_t)slot * SC_STAGE * SC_DIMS + lane;
        const int cnt = min(SC_STAGE, t - s * SC_STAGE);
        if (cnt == SC_STAGE) {
            double v[SC_STAGE];
#pragma unroll
            for (int u = 0; u < SC_STAGE; ++u) v[u] = cur[u * SC_DIMS];
#pragma unroll
            for (int u = 0; u < SC_STAGE; ++u) acc = __dadd_rn(acc, v[u]);
        } else {
            for (int u = 0; u < cnt; ++u) acc = __dadd_rn(acc, cur[u * SC_DIMS]);
        }
        __syncwarp();  // every lane is done with slot s % SC_STAGES ...
        if (lane == 0) issue(s + SC_STAGES);  // ... before it is refilled
    }
    if (j0 + lane < d_h) out[(long long)(pr0 + blockIdx.y) * d_h + j0 + lane] = (float)acc;
}

// bitmap -> ascending row list (init ++ selected ++ local), one CTA per head
__global__ void bitmap_rows_kernel(const uint32_t* bitmap, int words, int n_init, int n_local,
                                   int total, int T, int64_t* rows) {
    const int p = blockIdx.x, tid = threadIdx.x;
    int64_t* out = rows + (long long)p * T;
    __shared__ uint32_t run;
    __shared__ uint32_t cnts[256];
    if (tid == 0) run = 0;
    for (int e = tid; e < n_init; e += blockDim.x) out[e] = e;
    for (int e = tid; e < n_local; e += blockDim.x) out[T - n_local + e] = total - n_local + e;
    __syncthreads();
    for (int w0 = 0; w0 < words; w0 += 256) {
        int w = w0 + tid;
        uint32_t bits = (tid < 256 && w < words) ? bitmap[(long long)p * words + w] : 0u;
        if (tid < 256) cnts[tid] = __popc(bits);
        __syncthreads();
        if (tid == 0) {
            uint32_t r = run;
            for (int e = 0; e < 256; ++e) { uint32_t v = cnts[e]; cnts[e] = r; r += v; }
            run = r;
        }
        __syncthreads();
        if (tid < 256) {
            uint32_t off = cnts[tid] + n_init;
            while (bits) {
                int b = __ffs(bits) - 1;
                bits &= bits - 1;
                out[off++] = n_init + (long long)w * 32 + b;
            }
        }
        __syncthreads();
    }
}

}  // namespace

void launch_exact(pqkv_ctx* ctx, const float* queries, size_t P, size_t G, size_t d_h,
                  const float* keys, const float* values, size_t kv_head_stride,
                  const int64_t* rows, size_t t, float* out, cudaStream_t st) {
    // the product block of up to `batch` (head, query row) pairs at a time
    const size_t ldp = round_up(d_h, (size_t)SC_DIMS), per_pr = t * ldp;
    const size_t batch = std::max<size_t>(1, std::min(P * G, (size_t(256) << 20) / (per_pr * sizeof(double))));
    Scratch sc(ctx);
    size_t h_s = sc.plan<float>(P * G * t), h_w = sc.plan<double>(P * G * t), h_p = sc.plan<double>(batch * per_pr);
    sc.commit();
    float* scores = sc.get<float>(h_s);
    double* w = sc.get<double>(h_w);
    double* prod = sc.get<double>(h_p);
    double scale = 1.0 / std::sqrt(static_cast<double>(d_h));
    dim3 g1((unsigned)ceil_div(t, 128), (unsigned)(P * G));
    exact_scores_kernel<<<g1, 128, 0, st>>>(queries, (int)G, (int)d_h, keys, (long long)kv_head_stride,
                                           rows, (int)t, scale, scores);
    PQKV_LAUNCHED("exact_scores_kernel");
    softmax_weights_kernel<<<(unsigned)(P * G), SW_THREADS, 0, st>>>(scores, (int)t, w);
    PQKV_LAUNCHED("softmax_weights_kernel");
    for (size_t pr0 = 0; pr0 < P * G; pr0 += batch) {
        const size_t nb = std::min(batch, P * G - pr0);
        const unsigned gx = (unsigned)std::min<size_t>(ceil_div(per_pr, 256), 4 * (size_t)ctx->sm_count);
        weighted_products_kernel<<<dim3(gx, (unsigned)nb), 256, 0, st>>>((int)G, (int)d_h, (int)ldp, values,
                                                                         (long long)kv_head_stride, rows, (int)t, w,
                                                                         (int)pr0, prod);
        PQKV_LAUNCHED("weighted_products_kernel");
        PQKV_CUDA(cudaFuncSetAttribute(sum_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SC_SMEM));
        sum_chain_kernel<<<dim3((unsigned)(ldp / SC_DIMS), (unsigned)nb), SC_DIMS, SC_SMEM, st>>>(
            (int)d_h, (int)ldp, (int)t, prod, (int)pr0, out);
        PQKV_LAUNCHED("sum_chain_kernel");
    }
}

// Chunk geometry: all CTAs resident in one wave where possible (the gather
// reaches streaming bandwidth with ~1.6K rows per CTA, tools/microbench/
// gather_probe.cu); middle chunks are multiples of PQKV_TUPLE_CHUNK so the
// code-pair classification never splits a tuple chunk.
static int plan_chunk_tokens(pqkv_ctx* ctx, size_t P, size_t G, size_t s_mid, bool fill) {
    static const int forced = [] {  // experiments only: PQKV_CHUNK_TOKENS=1024|2048|4096k
        const char* e = std::getenv("PQKV_CHUNK_TOKENS");
        return e ? std::atoi(e) : 0;
    }();
    if (forced > 0) return forced;
    const size_t occ = 4;
    const size_t target = (size_t)ctx->sm_count * occ;
    const size_t per_head = std::max<size_t>(1, target / std::max<size_t>(P, 1));
    const size_t tcs = std::max<size_t>(1, ceil_div(s_mid, PQKV_TUPLE_CHUNK));
    if (per_head >= 2 * tcs) {  // few heads: 1/2 or 1/4 code-pair chunks per CTA
        const size_t sub = per_head >= 4 * tcs ? 4 : 2;
        return (int)(PQKV_TUPLE_CHUNK / sub);
    }
    // split pair path (no clusters): chunks of any 32-token multiple, sized
    // so the grid fills every CTA slot of the wave (north star: 18 chunks of
    // 7296 tokens = 576 CTAs, 4 per SM on all but 16 SMs, instead of 16 of
    // 8192 = 512 CTAs with 68 SMs at 4 and 80 at 3): 156.0 / 151.7 ->
    // 154.2 / 150.6 us
    if (fill) {
        const size_t ch = round_up(ceil_div(s_mid, per_head), (size_t)32);
        if (ch <= 8192) return (int)ch;
    }
    size_t q = std::min<size_t>(8, std::max<size_t>(1, ceil_div(tcs, per_head)));
    return (int)(q * PQKV_TUPLE_CHUNK);
}


// Shared memory: region (rows[] / merge partials / pair-select scratch)
// followed by words[] and the pair classes.
static size_t attend_smem(AtArgs& a, int G) {
    const size_t nw = (size_t)(a.nt > 0 ? a.nt : AT_THREADS) / 32;  // warps per CTA
    const bool wide = a.nt > AT_THREADS;
    // Chunks whose full row list + staged codes would cost CTAs per SM (many
    // heads: one wave of CTAs needs few, large chunks) expand and gather their
    // rows in windows of 4096 and, in pair mode, classify codes straight from
    // L2 instead of staging them, so the shared memory stays at the
    // 8192-token footprint.  Measured: g = 1, 64 units x 128K (16K chunks):
    // windowed 285 us vs 468; g = 2, 32 heads (16K chunks, 2 CTAs/SM either
    // way): staged 156 us vs windowed 194.
    {
        const size_t full_rows = ((size_t)a.chunk + a.n_init + a.n_local) * 4;
        const size_t tail_est = (size_t)a.chunk / 32 * 8 + ((a.src == SRC_TUPLE || a.src == SRC_PAIRS) ? (size_t)a.C * a.C : 0);
        const size_t ring2 = (G > 1 && a.src != SRC_KEYS) ? nw * 2 * 2 * DH * 4 : 0;
        const size_t budget = 55 * 1024;
        const bool full = wide || a.src == SRC_ROWS || a.chunk <= 8192 || full_rows + tail_est + ring2 <= budget;
        a.win = full ? a.chunk : 4096;
        // wide pair CTAs are their own selectors and classify from L2 (staging
        // their codes behind the select's scratch: select +1.5 us, classify
        // -0.6 us)
        a.stage = full && !(wide && a.src == SRC_PAIRS);
    }
    size_t rows_cap = a.src == SRC_ROWS ? (size_t)a.chunk : (size_t)a.win + a.n_init + a.n_local;
    const size_t rows_bytes = round_up(rows_cap * 4, 16);
    const size_t merge = nw * G * DH * 4 + ((size_t)2 * G * a.n_chunks + 2 * G) * 4;
    // g > 1: the per-warp cp.async row ring (8 warps x depth rows x K + V)
    // sits right after rows[]; the pair select's scratch (selector CTA, before
    // the gather) and the per-warp merge (after it) alias it.  Not for the
    // key path, whose g > 1 launch only selects.
    const bool ring = G > 1 && a.src != SRC_KEYS;
    const size_t ring4 = nw * 4 * 2 * DH * 4;
    auto region_for = [&](size_t ring_bytes) {
        size_t r = std::max(rows_bytes + ring_bytes, merge);
        if (a.src == SRC_PAIRS) r = std::max(r, pair_select_scratch(a.C, a.n_tchunks));
        // staged code pairs: the code_swz layout fills whole 1024-token blocks
        if ((a.src == SRC_PAIRS || a.src == SRC_TUPLE) && a.stage) r = std::max(r, round_up((size_t)a.chunk, 1024) * 4);
        if (a.src == SRC_KEYS) r = std::max(r, (size_t)a.chunk * 4 + (size_t)a.m * a.C * 8);
        return round_up(r, 16);
    };
    const size_t tail = (size_t)a.chunk / 32 * 4 + (a.src == SRC_KEYS ? (size_t)NB * 12 : (size_t)a.chunk / 32 * 4) +
                        ((a.src == SRC_TUPLE || a.src == SRC_PAIRS) ? (size_t)a.C * a.C : 0);
    // depth 4 unless only depth 2 keeps 4 CTAs per SM (227 KB / 4 less the
    // 1 KB per-CTA reservation)
    const size_t per4 = 55 * 1024;
    a.ring4 = wide || !ring || region_for(ring4) + tail <= per4 || region_for(ring4 / 2) + tail > per4;
    const size_t region = region_for(ring ? (a.ring4 ? ring4 : ring4 / 2) : 0);
    a.region = (int)region;
    a.ring_off = (int)rows_bytes;
    return region + round_up(tail, 16);
}

template <int G, int MODE, int NT = AT_THREADS>
static void launch_attend_gm(const AtArgs& a, dim3 grid, size_t smem, int cl, cudaStream_t st) {
    auto kern = attend_kernel<G, MODE, NT>;
    // attributes only grow: set once per (instantiation, device, thread) and
    // new size instead of on every decode
    static thread_local int smem_set[64], np_set[64];
    static thread_local bool init = false;
    if (!init) {
        for (int d = 0; d < 64; ++d) { smem_set[d] = -1; np_set[d] = 0; }
        init = true;
    }
    int dev = 0;
    PQKV_CUDA(cudaGetDevice(&dev));
    dev &= 63;
    if ((int)smem > smem_set[dev]) {
        PQKV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        smem_set[dev] = (int)smem;
    }
    if (cl > 8 && !np_set[dev]) {
        PQKV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        np_set[dev] = 1;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    // programmatic dependent launch (see the kernel's step 0).  Not for
    // clustered g > 1 grids (2 heavy CTAs per SM): placed early, while the
    // previous grid drains, their 8-CTA clusters pack onto the SMs that free
    // first (cfg3 73.5 -> 84 us, 32 heads g = 2 155 -> 193 us with it on)
    static const bool pdl_env = std::getenv("PQKV_NO_PDL") == nullptr;
    const bool pdl = pdl_env && !(G > 1 && cl > 1);
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 2 : 1;
    if (std::getenv("PQKV_DEBUG_CLUSTERS")) {
        int nc = -1;
        cudaOccupancyMaxActiveClusters(&nc, kern, &cfg);
        std::fprintf(stderr, "attend_kernel<%d>: grid %u x %u, cluster %d, smem %zu -> max active clusters %d\n", G,
                     grid.x, grid.y, cl, smem, nc);
    }
    PQKV_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
}

template <int G>
static void launch_attend_g(const AtArgs& a, dim3 grid, size_t smem, int cl, cudaStream_t st) {
    if constexpr (G > 1) {
        if (a.nt > AT_THREADS) {  // wide g > 1 plans (1024 threads, no key path)
            if (a.src == SRC_PAIRS) launch_attend_gm<G, SRC_PAIRS, 1024>(a, grid, smem, cl, st);
            else if (a.nt == 2 * AT_THREADS) launch_attend_gm<G, 0, 2 * AT_THREADS>(a, grid, smem, cl, st);
            else launch_attend_gm<G, 0, 1024>(a, grid, smem, cl, st);
            return;
        }
    }
    if (a.src == SRC_PAIRS) launch_attend_gm<G, SRC_PAIRS>(a, grid, smem, cl, st);
    else if (a.src == SRC_KEYS) launch_attend_gm<G, SRC_KEYS>(a, grid, smem, cl, st);
    else launch_attend_gm<G, 0>(a, grid, smem, cl, st);
}

// Cluster size and dynamic shared memory of an attention launch; pads
// a.n_chunks to a multiple of the cluster.
static int plan_attend_launch(AtArgs& a, int G, size_t* smem) {
    // pair-select mode: 8-CTA clusters share one pair select (pad the chunk
    // count to a multiple of the cluster; padded CTAs own empty ranges)
    int cl = 1;
    static const int forced_cl = [] {  // experiments only: PQKV_CLUSTER=4|8
        const char* e = std::getenv("PQKV_CLUSTER");
        return e ? std::atoi(e) : 0;
    }();
    if (a.src == SRC_PAIRS && a.n_chunks >= 4 && a.nt <= AT_THREADS) {  // wide CTAs select on their own
        cl = a.n_chunks >= 8 ? 8 : 4;  // 4 chunks per head (many heads): no empty padded CTAs
        if (forced_cl == 4 || forced_cl == 8) cl = forced_cl;
        a.n_chunks = (int)round_up((size_t)a.n_chunks, (size_t)cl);
    }
    if (a.src == SRC_KEYS) cl = a.n_chunks;  // one cluster per head (<= 16 CTAs)
    *smem = attend_smem(a, G);
    return cl;
}

static void launch_attend_kernel(pqkv_ctx* ctx, AtArgs& a, size_t P, int G, cudaStream_t st) {
    size_t smem = 0;
    const int cl = plan_attend_launch(a, G, &smem);
    // two-level merge from 32 chunks per head (a one-level merge of n
    // partials costs n / 16 dependent L2 round trips on the kernel's tail)
    a.n_groups = a.n_chunks >= 32 ? (a.n_chunks + MERGE_GROUP - 1) / MERGE_GROUP : 0;
    Scratch sc(ctx);
    size_t h_part = sc.plan<float>(P * a.n_chunks * G * (DH + 2));
    size_t h_part2 = sc.plan<float>(std::max<size_t>(1, P * a.n_groups * G * (DH + 2)));
    sc.commit();
    a.part = sc.get<float>(h_part);
    a.part2 = a.n_groups ? sc.get<float>(h_part2) : nullptr;
    a.arrivals = arrival_counters(ctx, P * (1 + a.n_groups), st);
    a.prof = nullptr;
    a.sel_dump = ctx->sel_dump;
    // PQKV_PROF_SELECT=1: profile only the key path's select launch (the
    // bitmap gather that follows would otherwise overwrite its stamps)
    static const bool prof_select_only = std::getenv("PQKV_PROF_SELECT") != nullptr;
    if (ctx->profiling && (!prof_select_only || a.sel_only)) {
        if (ctx->d_prof) cudaFree(ctx->d_prof);
        ctx->n_prof = (size_t)a.n_chunks * P;
        PQKV_CUDA(cudaMalloc(&ctx->d_prof, ctx->n_prof * PQKV_PROF_SLOTS * sizeof(unsigned long long)));
        PQKV_CUDA(cudaMemsetAsync(ctx->d_prof, 0, ctx->n_prof * PQKV_PROF_SLOTS * sizeof(unsigned long long), st));
        a.prof = ctx->d_prof;
    }
    dim3 grid((unsigned)a.n_chunks, (unsigned)P);
    switch (G) {
        case 1: launch_attend_g<1>(a, grid, smem, cl, st); break;
        case 2: launch_attend_g<2>(a, grid, smem, cl, st); break;
        case 4: launch_attend_g<4>(a, grid, smem, cl, st); break;
        default: fail(PQKV_EINVAL, "attend: g must be 1, 2 or 4 on the fast path");
    }
    PQKV_LAUNCHED("attend_kernel");
}

void launch_attend_rows(pqkv_ctx* ctx, const float* queries, size_t P, size_t G, size_t d_h,
                        const float* keys, const float* values, size_t kv_head_stride,
                        const int64_t* rows, size_t t, int precision, float* out,
                        cudaStream_t st) {
    bind_device(ctx);
    if (P == 0 || G == 0) return;
    if (t == 0) fail(PQKV_EINVAL, "attention: need at least one token");
    bool fast = precision == PQKV_PREC_F32 && d_h == DH && (G == 1 || G == 2 || G == 4) &&
                kv_head_stride % 4 == 0;
    if (!fast) {
        launch_exact(ctx, queries, P, G, d_h, keys, values, kv_head_stride, rows, t, out, st);
        return;
    }
    AtArgs a{};
    a.queries = queries;
    a.keys = keys;
    a.values = values;
    a.kv_head_stride = (long long)kv_head_stride;
    a.src = SRC_ROWS;
    a.rows = rows;
    a.t = (int)t;
    const size_t target = (size_t)ctx->sm_count * 4;
    const size_t per_head = std::max<size_t>(1, target / P);
    a.chunk = (int)std::min<size_t>(8192, round_up(std::max<size_t>(32, ceil_div(t, per_head)), 32));
    a.n_chunks = (int)ceil_div(t, (size_t)a.chunk);
    a.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)d_h));
    a.out = out;
    launch_attend_kernel(ctx, a, P, (int)G, st);
}

bool decode_fast_path(const pqkv_layer& L, size_t G) {
    return L.d_h == DH && (G == 1 || G == 2 || G == 4) && L.kv_head_stride % 4 == 0;
}

bool decode_pairs_fused(const pqkv_layer& L, size_t G) {
    return decode_fast_path(L, G) && L.m == 2 && L.b <= 6 && L.tuple_hist && L.tuple_chunk_hist;
}

// SRC_KEYS geometry: one portable cluster of n_chunks <= 8 CTAs per head
// (16-CTA clusters do not all fit one wave), chunks of 1024-token multiples
// up to 16K tokens, keys + ADC table in the shared region.
static bool keys_geometry(const pqkv_layer& L, size_t G, int* chunk, int* n_chunks) {
    (void)G;
    const size_t s_mid = L.total - L.n_init - L.n_local;
    const size_t C = size_t{1} << L.b;
    if (L.m * C * 8 > 16 * 1024 || s_mid == 0) return false;
    const size_t nc = std::min<size_t>(8, ceil_div(s_mid, 1024));
    const size_t ch = round_up(ceil_div(s_mid, nc), 1024);
    if (ch > 16384) return false;
    if (chunk) *chunk = (int)ch;
    if (n_chunks) *n_chunks = (int)ceil_div(s_mid, ch);
    return true;
}

bool decode_keys_fused(const pqkv_layer& L, size_t G) {
    return decode_fast_path(L, G) && keys_geometry(L, G, nullptr, nullptr);
}

// Key path in two launches (cluster select -> bitmap, then a finer bitmap-mode
// gather): always for g > 1 (one 8-CTA cluster per head leaves 1 CTA/SM for
// a gather that needs 2); for g = 1 unless the cluster grid fills the GPU in
// one wave with at least two CTAs per SM (16 units x 128K: fused 127 us,
// split 99.5 us; 64 units: the 98 KB key CTAs need two waves fused).
bool decode_keys_split(const pqkv_layer& L, size_t G) {
    if (G > 1) return true;
    int chunk = 0, n_chunks = 0;
    if (!keys_geometry(L, G, &chunk, &n_chunks)) return false;
    const int sms = current_sm_count();
    const size_t ctas = L.n_heads * (size_t)n_chunks;
    const size_t C = (size_t)1 << L.b;
    const size_t smem = (size_t)chunk * 4 + L.m * C * 8 + (size_t)chunk / 32 * 4 + (size_t)NB * 12 + 3072;
    const size_t per_sm = std::min<size_t>(4, (size_t)227 * 1024 / smem);
    return ctas < 2 * (size_t)sms || ctas > per_sm * (size_t)sms;
}

// Wide plans (1024-thread CTAs) for the g > 1 gathers: on unless
// PQKV_WIDE=0; needs the whole row list of a chunk in shared memory next to
// the 128 KB row ring.
static bool wide_plan(pqkv_ctx* ctx, const pqkv_layer& L, size_t G) {
    static const bool on = [] {
        const char* e = std::getenv("PQKV_WIDE");
        return !(e && *e == '0');
    }();
    if (!on || G < 2 || L.n_heads == 0) return false;
    const size_t s_mid = L.total - L.n_init - L.n_local;
    const size_t per_head = std::max<size_t>(1, (size_t)ctx->sm_count / L.n_heads);
    const size_t chunk = round_up(ceil_div(s_mid, per_head), (size_t)32);
    return (chunk + L.n_init + L.n_local) * 4 + chunk / 8 + 128 * 1024 + 8192 <= 200 * 1024;
}

// AtArgs of a decode attention launch (everything but queries, out and the
// selection inputs).
static void decode_args(pqkv_ctx* ctx, const pqkv_layer& L, size_t G, size_t k_pairs, size_t k_keys, bool bitmap,
                        bool tuple_cls, AtArgs& a) {
    const size_t s_mid = L.total - L.n_init - L.n_local;
    a.keys = L.keys;
    a.values = L.values;
    a.kv_head_stride = (long long)L.kv_head_stride;
    a.src = k_keys ? SRC_KEYS : (k_pairs ? SRC_PAIRS : (tuple_cls ? SRC_TUPLE : SRC_BITMAP));
    a.n_init = (int)L.n_init;
    a.n_local = (int)L.n_local;
    a.total = (int)L.total;
    a.s_mid = (int)s_mid;
    a.chunk = plan_chunk_tokens(ctx, L.n_heads, G, s_mid, tuple_cls || (bitmap && !k_pairs && !k_keys));
    a.n_chunks = (int)std::max<size_t>(1, ceil_div(s_mid, (size_t)a.chunk));
    a.words = (int)ceil_div(s_mid, 32);
    a.codes = L.codes;
    a.codes_head_stride = (long long)L.codes_head_stride;
    a.C = 1 << L.b;
    a.centroids = L.centroids;
    a.thist = L.tuple_hist;
    a.chist = L.tuple_chunk_hist;
    a.n_tchunks = (int)ceil_div(s_mid, PQKV_TUPLE_CHUNK);
    a.tchunk_stride = L.tuple_chunks ? (long long)L.tuple_chunks : a.n_tchunks;
    a.k = (int)(k_keys ? k_keys : k_pairs);
    a.m = (int)L.m;
    a.sel_only = nullptr;
    a.nt = AT_THREADS;
    if (k_keys) {
        keys_geometry(L, G, &a.chunk, &a.n_chunks);
    } else if (wide_plan(ctx, L, G)) {
        // g > 1: one 1024-thread CTA per SM whose 32 warps claim rows
        // dynamically (every SM gets the same share of rows and no warp idles
        // at the end); pair mode selects in every CTA (no clusters)
        // bitmap-mode gathers (the key path's second launch) run two
        // 512-thread CTAs per SM: a CTA (~100 KB, 32K registers) fits beside
        // a select CTA still running on its SM, so units whose select is done
        // start gathering there (cfg5 86.7 / 90.9 -> 83.1 / 87.6 us);
        // PQKV_WIDE_NT=1024 restores one 1024-thread CTA per SM
        static const int wide_nt = [] {
            const char* e = std::getenv("PQKV_WIDE_NT");
            return e && std::atoi(e) == 1024 ? 1024 : 2 * AT_THREADS;
        }();
        a.nt = bitmap ? wide_nt : 1024;
        const size_t per_head = std::max<size_t>(1, (size_t)ctx->sm_count * (1024 / a.nt) / L.n_heads);
        static const bool claim = std::getenv("PQKV_CLAIM") != nullptr;
        a.claim = claim;
        a.chunk = (int)round_up(ceil_div(s_mid, per_head), (size_t)32);
        a.n_chunks = (int)std::max<size_t>(1, ceil_div(s_mid, (size_t)a.chunk));
    }
    a.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)L.d_h));
}

void plan_decode_attend(pqkv_ctx* ctx, const pqkv_layer& L, size_t G, size_t k_pairs, size_t k_keys,
                        bool tuple_cls, pqkv_decode_plan_t* out) {
    AtArgs a{};
    decode_args(ctx, L, G, k_pairs, k_keys, !k_pairs && !tuple_cls, tuple_cls, a);
    size_t smem = 0;
    const int cl = plan_attend_launch(a, (int)G, &smem);
    out->chunk_tokens = a.chunk;
    out->ctas_per_head = a.n_chunks;
    out->cluster = cl;
    out->staged = (a.src == SRC_PAIRS || a.src == SRC_TUPLE) ? a.stage : 0;
    out->window = a.win;
    out->ring_depth = (G > 1 && a.src != SRC_KEYS) ? (a.ring4 ? 4 : 2) : 0;
    out->smem_bytes = smem;
}

void launch_decode_attend(pqkv_ctx* ctx, const pqkv_layer& L, const float* queries, size_t G,
                          const uint32_t* bitmap, const uint8_t* cls, const int* cut, float* out,
                          cudaStream_t st, size_t k_pairs, size_t k_keys, unsigned* ready) {
    bind_device(ctx);
    AtArgs a{};
    decode_args(ctx, L, G, k_pairs, k_keys, bitmap != nullptr, cls != nullptr, a);
    a.ready_in = ready;  // split pair path: one select CTA per head
    a.ready_need = 1;
    a.queries = queries;
    a.bitmap = bitmap;
    a.cls = cls;
    a.cut = cut;
    // g > 1 (1 CTA/SM per key cluster): select in one launch, gather in a
    // second bitmap-mode launch with its own (finer) chunking
    if (k_keys && bitmap && decode_keys_split(L, G)) {
        a.sel_only = const_cast<uint32_t*>(bitmap);
        a.ready_in = nullptr;
        a.ready_out = ready_counters(ctx, L.n_heads, st);
        launch_attend_kernel(ctx, a, L.n_heads, (int)G, st);
        AtArgs b{};
        decode_args(ctx, L, G, 0, 0, true, false, b);
        b.queries = queries;
        b.bitmap = bitmap;
        b.out = out;
        b.ready_in = a.ready_out;
        b.ready_need = (unsigned)a.n_chunks;
        launch_attend_kernel(ctx, b, L.n_heads, (int)G, st);
        return;
    }
    a.out = out;
    launch_attend_kernel(ctx, a, L.n_heads, (int)G, st);
}

void launch_exact_scores(pqkv_ctx* ctx, const float* queries, size_t P, size_t G, size_t d_h,
                         const float* keys, size_t kv_head_stride, const int64_t* rows, size_t t,
                         float* scores, cudaStream_t st) {
    bind_device(ctx);
    if (t == 0 || P == 0 || G == 0) return;
    double scale = 1.0 / std::sqrt(static_cast<double>(d_h));
    dim3 g1((unsigned)ceil_div(t, 128), (unsigned)(P * G));
    exact_scores_kernel<<<g1, 128, 0, st>>>(queries, (int)G, (int)d_h, keys, (long long)kv_head_stride,
                                           rows, (int)t, scale, scores);
    PQKV_LAUNCHED("exact_scores_kernel");
}

void launch_bitmap_rows(pqkv_ctx* ctx, const uint32_t* bitmap, size_t P, size_t words,
                        size_t n_init, size_t n_local, size_t total, size_t T, int64_t* rows,
                        cudaStream_t st) {
    bind_device(ctx);
    bitmap_rows_kernel<<<(unsigned)P, 256, 0, st>>>(bitmap, (int)words, (int)n_init, (int)n_local,
                                                   (int)total, (int)T, rows);
    PQKV_LAUNCHED("bitmap_rows_kernel");
}

}  // namespace pqkv_dev
