// select.cu -- ADC scoring and exact top-k selection on sm_100a (hot path B).
//
// pq_score_gqa (pq.cpp:113-161) + approx_topk/top_k_desc (pq.cpp:174-177,
// topk.cpp:8-25) as one fused kernel per head, run by a thread-block CLUSTER
// of SEL_CL CTAs that split the head's middle tokens:
//
//  1. every CTA builds the fp64 ADC table T[j][c] in shared memory
//     (sequential-t dot per (j,c), query rows summed in order -- the
//     products are exact in fp64 so FMA is harmless, pq.cpp:118-124);
//  2. scans its slice of codes, score_i = f32(((0.0 + T[0][c_i0]) + ...)),
//     bit-identical to gather_scores (pq.cpp:128-140), and keeps the
//     order-preserving 32-bit keys in shared memory;
//  3. radix-selects the k-th largest key in three digit passes
//     (11/11/10 bits); per-CTA histograms are merged through distributed
//     shared memory (DSMEM), so no global atomics and no extra launches;
//  4. resolves the tie at the threshold exactly like partial_sort with the
//     (score desc, id asc) comparator: all keys above the threshold are
//     selected, plus the lowest-id keys equal to it -- a cluster-wide
//     exclusive prefix of per-CTA equal counts tells each CTA how many of
//     its own equal keys it takes;
//  5. writes the selection bitmap (one ballot per 32 tokens) and optionally
//     the selected (key, id) pairs compacted in id order, which the
//     stable radix sort kernel below orders into approx_topk's output.
//
// The same kernel serves top_k_desc over explicit scores (with the
// reference's optional exclusion set, topk.cpp:10-15).
#include <cooperative_groups.h>

#include <algorithm>
#include <vector>

#include "internal.cuh"
#include "select_common.cuh"

namespace cg = cooperative_groups;

namespace pqkv_dev {
namespace {

constexpr int SEL_CL = 8;         // CTAs per head (portable cluster size)
constexpr int SEL_THREADS = 512;  // 16 warps
constexpr int SEL_WARPS = SEL_THREADS / 32;

struct SelArgs {
    // ADC source
    const float* queries;
    int g, d_h, m, C;
    const float* centroids;
    const uint16_t* codes;
    long long codes_head_stride;
    // score source
    const float* scores;
    long long scores_stride;
    const uint8_t* excluded;
    // geometry
    int n, k, slice, keys_smem;
    uint32_t* gkeys;  // [rows][n] when !keys_smem
    // outputs
    uint32_t* bitmap;  // [rows][words] or null
    int words;
    uint32_t* sel_key;  // [rows][k] compacted in id order, or null
    uint32_t* sel_id;
    int* status;  // [rows]
};

__device__ __forceinline__ uint32_t adc_key(const double* lut, const uint16_t* code, int m, int C) {
    double acc = 0.0;
    for (int j = 0; j < m; ++j) acc = __dadd_rn(acc, lut[j * C + code[j]]);
    return score_key((float)acc);
}

// Warp-aggregated shared-memory histogram increment; bin == ~0u is a no-op.
__device__ __forceinline__ void hist_add(uint32_t* hist, uint32_t bin) {
    unsigned peers = __match_any_sync(FULL, bin);
    int leader = __ffs(peers) - 1;
    if ((threadIdx.x & 31) == leader && bin != 0xffffffffu) atomicAdd(&hist[bin], __popc(peers));
}

__global__ void __launch_bounds__(SEL_THREADS, 1) select_kernel(SelArgs a) {
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int row = blockIdx.x / SEL_CL;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int lo = rank * a.slice;
    const int hi = min(a.n, lo + a.slice);
    const int cnt = max(0, hi - lo);

    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* hist0 = reinterpret_cast<uint32_t*>(smem);  // 3 digit passes
    uint32_t* hist1 = hist0 + NB;
    uint32_t* hist2 = hist1 + NB;
    uint32_t* tot = hist2 + NB;             // merged histogram [NB]
    uint32_t* pub = tot + NB;               // published per-CTA counts [8]
    uint32_t* wsum = pub + 8;               // [32]
    uint32_t* sh = wsum + 32;               // misc [8]
    double* lut = reinterpret_cast<double*>(sh + 8);
    const int lut_elems = a.codes ? a.m * a.C : 0;
    uint32_t* skeys = reinterpret_cast<uint32_t*>(lut + lut_elems);
    uint32_t* keys = a.keys_smem ? skeys : a.gkeys + (long long)row * a.n + lo;

    for (int b = tid; b < 4 * NB; b += SEL_THREADS) hist0[b] = 0;
    if (a.codes) {
        build_lut(lut, a.queries + (long long)row * a.g * a.d_h,
                  a.centroids + (long long)row * a.m * a.C * (a.d_h / a.m), a.g, a.d_h, a.m, a.C);
    }
    __syncthreads();

    // ---- keys + first digit histogram ----
    for (int i0 = 0; i0 < cnt + SEL_THREADS - 1; i0 += SEL_THREADS) {
        int li = i0 + tid;
        uint32_t bin = 0xffffffffu;
        if (li < cnt) {
            int i = lo + li;
            uint32_t key;
            if (a.codes) {
                key = adc_key(lut, a.codes + (long long)row * a.codes_head_stride + (long long)i * a.m, a.m, a.C);
            } else {
                bool ex = a.excluded && a.excluded[(long long)row * a.n + i];
                key = ex ? 0u : score_key(a.scores[(long long)row * a.scores_stride + i]);
            }
            keys[li] = key;
            if (key) bin = key >> 21;
        }
        hist_add(hist0, bin);
    }
    cluster.sync();

    // ---- three digit passes ----
    uint32_t k_rem = (uint32_t)a.k, prefix = 0;
    const int shifts[3] = {21, 10, 0};
    const int nbins[3] = {2048, 2048, 1024};
    uint32_t* hists[3] = {hist0, hist1, hist2};
    for (int p = 0; p < 3; ++p) {
        if (p > 0) {
            // local histogram of the next digit among keys matching the prefix
            const int sh_hi = shifts[p - 1];
            const uint32_t mask = (uint32_t)(nbins[p] - 1);
            for (int i0 = 0; i0 < cnt + SEL_THREADS - 1; i0 += SEL_THREADS) {
                int li = i0 + tid;
                uint32_t bin = 0xffffffffu;
                if (li < cnt) {
                    uint32_t key = keys[li];
                    if (key && (key >> sh_hi) == prefix) bin = (key >> shifts[p]) & mask;
                }
                hist_add(hists[p], bin);
            }
            cluster.sync();
        }
        // merge through DSMEM
        for (int b = tid; b < nbins[p]; b += SEL_THREADS) {
            uint32_t s = 0;
#pragma unroll
            for (int r = 0; r < SEL_CL; ++r) s += cluster.map_shared_rank(hists[p], r)[b];
            tot[b] = s;
        }
        __syncthreads();
        if (p == 0) {
            // candidate count check (exclusions can leave fewer than k)
            uint32_t local = 0;
            for (int b = tid; b < NB; b += SEL_THREADS) local += tot[b];
            uint32_t total;
            block_excl_scan<SEL_THREADS>(local, wsum, &total);
            if (total < k_rem) {
                if (tid == 0 && rank == 0) a.status[row] = 1;
                cluster.sync();
                return;  // uniform across the cluster
            }
        }
        find_digit<SEL_THREADS>(tot, nbins[p], k_rem, wsum, sh);
        uint32_t digit = sh[0];
        k_rem -= sh[1];
        prefix = (prefix << (p == 0 ? 11 : (p == 1 ? 11 : 10))) | digit;
        __syncthreads();
    }
    const uint32_t kstar = prefix;  // the k-th largest key; take k_rem of the ties

    // ---- per-CTA counts of keys above / equal to the threshold ----
    uint32_t ngt = 0, neq = 0;
    for (int li = tid; li < cnt; li += SEL_THREADS) {
        uint32_t key = keys[li];
        ngt += key > kstar;
        neq += key == kstar;
    }
    uint32_t cta_gt, cta_eq;
    block_excl_scan<SEL_THREADS>(ngt, wsum, &cta_gt);
    block_excl_scan<SEL_THREADS>(neq, wsum, &cta_eq);
    if (tid == 0) { pub[0] = cta_gt; pub[1] = cta_eq; }
    cluster.sync();
    // how many equal keys this CTA takes, and where its selections start
    uint32_t eq_before = 0, sel_before = 0;
    for (int r = 0; r < rank; ++r) {
        const uint32_t* rp = cluster.map_shared_rank(pub, r);
        uint32_t rgt = rp[0], req = rp[1];
        uint32_t take_r = k_rem > eq_before ? min(req, k_rem - eq_before) : 0;
        sel_before += rgt + take_r;
        eq_before += req;
    }
    const uint32_t take = k_rem > eq_before ? min(cta_eq, k_rem - eq_before) : 0;

    // ---- ordered pass: bitmap words + compacted (key, id) ----
    uint32_t eq_run = 0, sel_run = 0;
    uint32_t* bm = a.bitmap ? a.bitmap + (long long)row * a.words : nullptr;
    for (int i0 = 0; i0 < cnt; i0 += SEL_THREADS) {
        int li = i0 + tid;
        uint32_t key = li < cnt ? keys[li] : 0u;
        bool gt = li < cnt && key > kstar;
        bool eq = li < cnt && key == kstar;
        unsigned eqm = __ballot_sync(FULL, eq);
        // eq rank within the CTA's slice, in id order
        if (lane == 0) wsum[warp] = __popc(eqm);
        __syncthreads();
        uint32_t wbefore = 0, tile_eq = 0;
        for (int w = 0; w < SEL_WARPS; ++w) {
            uint32_t c = wsum[w];
            if (w < warp) wbefore += c;
            tile_eq += c;
        }
        __syncthreads();
        uint32_t my_eq_rank = eq_run + wbefore + __popc(eqm & lanemask_lt());
        bool sel = gt || (eq && my_eq_rank < take);
        unsigned selm = __ballot_sync(FULL, sel);
        if (bm && lane == 0) {
            int word = (lo + i0) / 32 + warp;
            if ((lo + i0 + warp * 32) < hi) bm[word] = selm;
        }
        if (a.sel_key) {
            if (lane == 0) wsum[warp] = __popc(selm);
            __syncthreads();
            uint32_t sbefore = 0, tile_sel = 0;
            for (int w = 0; w < SEL_WARPS; ++w) {
                uint32_t c = wsum[w];
                if (w < warp) sbefore += c;
                tile_sel += c;
            }
            __syncthreads();
            if (sel) {
                uint32_t pos = sel_before + sel_run + sbefore + __popc(selm & lanemask_lt());
                a.sel_key[(long long)row * a.k + pos] = key;
                a.sel_id[(long long)row * a.k + pos] = (uint32_t)(lo + li);
            }
            sel_run += tile_sel;
        }
        eq_run += tile_eq;
    }
    cluster.sync();  // keep this CTA's smem alive for remote readers
}

// ---- stable LSD radix sort of k (key, id) pairs by key, descending --------
// One CTA per row; ids arrive in ascending order so stability yields the
// reference's (score desc, id asc) order (topk.cpp:17-22).
constexpr int SORT_THREADS = 1024;
constexpr int SORT_WARPS = SORT_THREADS / 32;

__global__ void __launch_bounds__(SORT_THREADS, 1)
    sort_desc_kernel(const uint32_t* key_in, const uint32_t* id_in, uint32_t* key_tmp,
                     uint32_t* id_tmp, int k, int64_t* ids_out) {
    __shared__ uint32_t base[256];
    __shared__ uint32_t cnt[SORT_WARPS][256];
    __shared__ uint32_t tile_tot[256];
    const int row = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t* kin = key_in + (long long)row * k;
    const uint32_t* iin = id_in + (long long)row * k;
    uint32_t* kout = key_tmp + (long long)row * k;
    uint32_t* iout = id_tmp + (long long)row * k;
    // Ping-pong: pass 0 in->tmp, 1 tmp->in(copy area), ... we use the input
    // buffers as the second half (they are scratch owned by the launcher).
    uint32_t* ka = const_cast<uint32_t*>(kin);
    uint32_t* ia = const_cast<uint32_t*>(iin);
    uint32_t* kb = kout;
    uint32_t* ib = iout;
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = 8 * pass;
        for (int d = tid; d < 256; d += SORT_THREADS) base[d] = 0;
        __syncthreads();
        for (int i = tid; i < k; i += SORT_THREADS) atomicAdd(&base[255 - ((ka[i] >> shift) & 255)], 1u);
        __syncthreads();
        if (tid < 32) {  // exclusive scan of 256 counters by one warp
            uint32_t v[8], s = 0;
#pragma unroll
            for (int e = 0; e < 8; ++e) { v[e] = base[lane * 8 + e]; s += v[e]; }
            uint32_t x = s;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(FULL, x, o);
                if (lane >= o) x += y;
            }
            uint32_t run = x - s;
#pragma unroll
            for (int e = 0; e < 8; ++e) { base[lane * 8 + e] = run; run += v[e]; }
        }
        __syncthreads();
        for (int t0 = 0; t0 < k; t0 += SORT_THREADS) {
            for (int e = tid; e < SORT_WARPS * 256; e += SORT_THREADS) (&cnt[0][0])[e] = 0;
            __syncthreads();
            int i = t0 + tid;
            uint32_t d = 0xffffffffu, key = 0, id = 0;
            if (i < k) { key = ka[i]; id = ia[i]; d = 255 - ((key >> shift) & 255); }
            unsigned peers = __match_any_sync(FULL, d);
            uint32_t rank = __popc(peers & lanemask_lt());
            if (d != 0xffffffffu && rank == 0) cnt[warp][d] = __popc(peers);
            __syncthreads();
            if (tid < 256) {
                uint32_t run = 0;
                for (int w = 0; w < SORT_WARPS; ++w) {
                    uint32_t c = cnt[w][tid];
                    cnt[w][tid] = run;
                    run += c;
                }
                tile_tot[tid] = run;
            }
            __syncthreads();
            if (d != 0xffffffffu) {
                uint32_t pos = base[d] + cnt[warp][d] + rank;
                kb[pos] = key;
                ib[pos] = id;
            }
            __syncthreads();
            if (tid < 256) base[tid] += tile_tot[tid];
            __syncthreads();
        }
        uint32_t* t;
        t = ka; ka = kb; kb = t;
        t = ia; ia = ib; ib = t;
    }
    // after 4 passes the sorted data is back in the input buffers
    for (int i = tid; i < k; i += SORT_THREADS) ids_out[(long long)row * k + i] = (int64_t)ia[i];
}

// ---- pq_score (materialised scores): LUT kernel + gather kernel ----------
__global__ void lut_kernel(const float* queries, int g, int d_h, int m, int C,
                           const float* centroids, double* lut_out) {
    int p = blockIdx.x;
    build_lut(lut_out + (long long)p * m * C, queries + (long long)p * g * d_h,
              centroids + (long long)p * m * C * (d_h / m), g, d_h, m, C);
}

__global__ void gather_scores_kernel(const double* lut_g, int m, int C, const uint16_t* codes,
                                     long long codes_head_stride, int s, float* scores,
                                     long long scores_stride, int lut_smem) {
    extern __shared__ double lut_s[];
    int p = blockIdx.y;
    const double* lut = lut_g + (long long)p * m * C;
    if (lut_smem) {
        for (int e = threadIdx.x; e < m * C; e += blockDim.x) lut_s[e] = lut[e];
        __syncthreads();
        lut = lut_s;
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < s; i += gridDim.x * blockDim.x) {
        const uint16_t* code = codes + p * codes_head_stride + (long long)i * m;
        double acc = 0.0;
        for (int j = 0; j < m; ++j) acc = __dadd_rn(acc, lut[j * C + code[j]]);
        scores[p * scores_stride + i] = (float)acc;
    }
}


// ===========================================================================
// Tuple path (m == 2, C^2 <= 16384): the ADC score of a token is a function
// of its code pair only, f32((0.0 + T[0][c0]) + T[1][c1]) (pq.cpp:128-140),
// so the radix select runs over the C^2 pair keys weighted by how many middle
// tokens carry each pair.  Per head the index keeps
//   thist[p][t]        tokens with pair t                (u32)
//   chist[p][c][t]     same, per TCHUNK-row chunk c      (u16)
// maintained by tuple_tables_kernel at build and on append.  tuple_select
// (one CTA per head) finds the threshold key K*, classifies every pair
// (above / equal / below) and -- from chist -- the chunk c* that holds the
// lowest-id boundary of the equal keys and how many of c*'s equal tokens are
// taken.  tuple_bitmap then streams the codes once per chunk.
// ===========================================================================
// 512 threads (128 registers, 8 pairs per thread) for up to 4096 pairs
// (b <= 6): powerlaw select 11.3 -> 9.6 us against 256 threads
// (tools/microbench/pair_select_probe.cu); 1024 threads for b = 7's 16384
constexpr int TUP_THREADS = 512, TUP_THREADS_B7 = 1024;

__global__ void tuple_tables_kernel(const uint16_t* codes, long long codes_head_stride, int C,
                                    int row_begin, int row_end, uint32_t* thist, uint16_t* chist,
                                    int n_chunks) {
    extern __shared__ uint32_t cnt[];  // [C*C]
    const int p = blockIdx.y, c = blockIdx.x, C2 = C * C;
    const int r0 = max(row_begin, c * PQKV_TUPLE_CHUNK), r1 = min(row_end, (c + 1) * PQKV_TUPLE_CHUNK);
    if (r0 >= r1) return;
    for (int t = threadIdx.x; t < C2; t += blockDim.x) cnt[t] = 0;
    __syncthreads();
    const uint16_t* cd = codes + p * codes_head_stride;
    for (int i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
        uint32_t t = (uint32_t)cd[2LL * i] * C + cd[2LL * i + 1];
        atomicAdd(&cnt[t], 1u);
    }
    __syncthreads();
    uint16_t* ch = chist + ((long long)p * n_chunks + c) * C2;
    uint32_t* th = thist + (long long)p * C2;
    for (int t = threadIdx.x; t < C2; t += blockDim.x) {
        uint32_t v = cnt[t];
        if (v) {
            ch[t] = (uint16_t)(ch[t] + v);
            atomicAdd(&th[t], v);
        }
    }
}

struct TupArgs {
    const float* queries;
    int g, d_h, C;
    const float* centroids;
    const uint32_t* thist;
    const uint16_t* chist;
    int n, k, n_chunks;
    uint8_t* cls;           // [P][C2]: 0 below, 1 above, 2 equal
    uint32_t* tkey;         // [P][C2] pair keys (ids mode) or null
    int* cut;               // [P][2]: c*, take
    uint32_t* sel_before;   // [P][n_chunks] exclusive prefix of selected rows (ids mode) or null
    long long chunk_stride;  // chunks per head of chist
    unsigned* ready;        // [P] bumped once a head's classes are written (the attention polls it), or null
    float* q_copy;          // [P][g][d_h] device copy of the queries for the attention (host-mapped input), or null
};

template <int NT>
__global__ void __launch_bounds__(NT, 1) tuple_select_kernel(TupArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int p = blockIdx.x, tid = threadIdx.x, C = a.C, C2 = C * C;
    PairScratch ps(smem, C, a.n_chunks);
    uint32_t* sh = ps.sh;
    uint32_t* ceq = ps.ceq;
    uint32_t* hist = ps.hist;  // per-chunk counts below (dead radix bins, 2*NB entries with cnt)
    uint8_t* cls = a.cls + (long long)p * C2;
    const uint16_t* ch = a.chist + (long long)p * a.chunk_stride * C2;
    // the centroid table is staged before the wait (no kernel that lets this
    // grid launch early writes centroids: only the attention and select
    // kernels trigger programmatic launches)
    const float* cen = a.centroids + (long long)p * 2 * C * (a.d_h / 2);
    float4* stage = pair_lut_stage(C, a.d_h, ps.hist);
    const bool prestaged =
        lut_staged((a.q_copy ? a.q_copy : a.queries) + (long long)p * a.g * a.d_h, cen, a.d_h, 2, stage);
    if (prestaged) stage_centroids(cen, a.d_h, 2, C, stage);
    // launched with programmatic stream serialization: wait for the queries'
    // producer, then let the attention grid launch and stage its codes
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    // host-mapped queries: read once, into the device copy the attention
    // uses (published with the classes by the ready flag below) and which
    // the select then reads
    const float* qp = a.queries + (long long)p * a.g * a.d_h;
    if (a.q_copy) {
        float* qc = a.q_copy + (long long)p * a.g * a.d_h;
        for (int e = tid; e < a.g * a.d_h; e += NT) qc[e] = qp[e];
        __syncthreads();
        qp = qc;
    }
    pair_select<NT, NT >= 1024 ? 16 : 4096 / NT>(qp, a.g, a.d_h,
                                 a.centroids + (long long)p * 2 * C * (a.d_h / 2), C, a.thist + (long long)p * C2,
                                 ch, a.n_chunks, a.k, ps.lut, ps.hist, ps.cnt, ps.lst, ps.ceq, ps.wsum, ps.sh, cls,
                                 a.tkey ? a.tkey + (long long)p * C2 : nullptr, nullptr, prestaged);
    if (tid == 0) {
        a.cut[2 * p] = (int)sh[3];
        a.cut[2 * p + 1] = (int)sh[4];
    }
    if (a.sel_before) {  // selected rows per chunk -> exclusive prefix (ordered ids)
        const int cstar = (int)sh[3];
        const uint32_t take = sh[4];
        for (int c = tid >> 5; c < a.n_chunks; c += NT / 32) {
            uint32_t gt = 0;
            for (int t = tid & 31; t < C2; t += 32)
                if (cls[t] == 1) gt += ch[(long long)c * C2 + t];
            gt = warp_sum(gt);
            if ((tid & 31) == 0) {
                uint32_t eqc = c < cstar ? ceq[c] : (c == cstar ? take : 0);
                hist[c] = gt + eqc;  // hist reused as per-chunk counts
            }
        }
        __syncthreads();
        if (tid == 0) {
            uint32_t run = 0;
            for (int c = 0; c < a.n_chunks; ++c) {
                a.sel_before[(long long)p * a.n_chunks + c] = run;
                run += hist[c];
            }
        }
    }
    // this head's attention CTAs start now, not after the slowest head's select
    __syncthreads();
    if (a.ready && tid == 0) {
        __threadfence();
        atomicAdd(&a.ready[p], 1u);
    }
}

constexpr int TB_THREADS = 256;
constexpr int TB_WARPS = TB_THREADS / 32;

__global__ void __launch_bounds__(TB_THREADS) tuple_bitmap_kernel(
    const uint16_t* codes, long long codes_head_stride, int n, int C, const uint8_t* cls_g,
    const int* cut, uint32_t* bitmap, int words, const uint32_t* tkey_g,
    const uint32_t* sel_before, uint32_t* sel_key, uint32_t* sel_id, int k, int n_chunks) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int c = blockIdx.x, p = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int C2 = C * C;
    uint8_t* cls = smem;
    uint32_t* tkey = reinterpret_cast<uint32_t*>(smem + ((C2 + 15) / 16) * 16);
    __shared__ uint32_t wc[TB_WARPS], ws[TB_WARPS];
    const bool ids = sel_key != nullptr;
    if ((C2 & 3) == 0) {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(cls_g + (long long)p * C2);
        for (int t = tid; t < C2 / 4; t += TB_THREADS) reinterpret_cast<uint32_t*>(cls)[t] = src[t];
    } else {
        for (int t = tid; t < C2; t += TB_THREADS) cls[t] = cls_g[(long long)p * C2 + t];
    }
    if (ids)
        for (int t = tid; t < C2; t += TB_THREADS) tkey[t] = tkey_g[(long long)p * C2 + t];
    __syncthreads();
    const int cstar = cut[2 * p];
    const uint32_t take = (uint32_t)cut[2 * p + 1];
    const int r0 = c * PQKV_TUPLE_CHUNK, r1 = min(n, r0 + PQKV_TUPLE_CHUNK);
    const uint32_t* cd = reinterpret_cast<const uint32_t*>(codes + p * codes_head_stride);
    uint32_t eq_run = 0, sel_run = ids ? sel_before[(long long)p * n_chunks + c] : 0;
    constexpr int U = 4;
    for (int base0 = r0; base0 < r1; base0 += U * TB_THREADS) {
        uint32_t prs[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = base0 + u * TB_THREADS + tid;
            prs[u] = i < r1 ? cd[i] : 0u;  // (c0, c1) little-endian u16 pair
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int base = base0 + u * TB_THREADS;
            if (base >= r1) break;  // uniform
            const int i = base + tid;
            uint32_t t = 0;
            uint8_t cl = 0;
            if (i < r1) {
                t = (prs[u] & 0xffffu) * (uint32_t)C + (prs[u] >> 16);
                cl = cls[t];
            }
            bool gt = cl == 1, eq = cl == 2;
            bool sel;
            if (c < cstar) sel = gt || eq;
            else if (c > cstar) sel = gt;
            else {  // the boundary chunk: equal pairs in id order, first `take`
                unsigned em = __ballot_sync(FULL, eq);
                if (lane == 0) wc[warp] = __popc(em);
                __syncthreads();
                uint32_t before = 0, tile = 0;
#pragma unroll
                for (int w = 0; w < TB_WARPS; ++w) {
                    uint32_t v = wc[w];
                    before += w < warp ? v : 0;
                    tile += v;
                }
                __syncthreads();
                sel = gt || (eq && eq_run + before + __popc(em & lanemask_lt()) < take);
                eq_run += tile;
            }
            unsigned sm = __ballot_sync(FULL, sel);
            if (lane == 0 && base + warp * 32 < r1) bitmap[(long long)p * words + (base >> 5) + warp] = sm;
            if (ids) {
                if (lane == 0) ws[warp] = __popc(sm);
                __syncthreads();
                uint32_t before = 0, tile = 0;
#pragma unroll
                for (int w = 0; w < TB_WARPS; ++w) {
                    uint32_t v = ws[w];
                    before += w < warp ? v : 0;
                    tile += v;
                }
                __syncthreads();
                if (sel) {
                    uint32_t pos = sel_run + before + __popc(sm & lanemask_lt());
                    sel_key[(long long)p * k + pos] = tkey[t];
                    sel_id[(long long)p * k + pos] = (uint32_t)i;
                }
                sel_run += tile;
            }
        }
    }
}

}  // namespace

void launch_score(pqkv_ctx* ctx, const float* queries, size_t n_heads, size_t g, size_t d_h,
                  size_t m, size_t C, const float* centroids, const uint16_t* codes,
                  size_t codes_head_stride, size_t s, float* scores, size_t scores_stride,
                  cudaStream_t st) {
    bind_device(ctx);
    Scratch sc(ctx);
    size_t h_lut = sc.plan<double>(n_heads * m * C);
    sc.commit();
    double* lut = sc.get<double>(h_lut);
    lut_kernel<<<(unsigned)n_heads, 256, 0, st>>>(queries, (int)g, (int)d_h, (int)m, (int)C,
                                                  centroids, lut);
    PQKV_LAUNCHED("lut_kernel");
    if (s == 0) return;
    size_t lut_bytes = m * C * sizeof(double);
    int lut_smem = lut_bytes <= 96 * 1024;
    if (lut_smem)
        PQKV_CUDA(cudaFuncSetAttribute(gather_scores_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lut_bytes));
    unsigned bx = (unsigned)std::min<size_t>(ceil_div(s, 256), std::max(1, 2 * ctx->sm_count / (int)std::max<size_t>(1, n_heads)) + 1);
    dim3 grid(bx, (unsigned)n_heads);
    gather_scores_kernel<<<grid, 256, lut_smem ? lut_bytes : 0, st>>>(
        lut, (int)m, (int)C, codes, (long long)codes_head_stride, (int)s, scores,
        (long long)scores_stride, lut_smem);
    PQKV_LAUNCHED("gather_scores_kernel");
}

bool launch_select(pqkv_ctx* ctx, const SelectSource& src, size_t rows, size_t n, size_t k,
                   uint32_t* bitmap, int64_t* ids, cudaStream_t st, int* launches) {
    bind_device(ctx);
    int nl = 0;
    const size_t words = ceil_div(n, 32);
    if (rows == 0) return true;
    if (k == 0 || n == 0) {
        if (bitmap) PQKV_CUDA(cudaMemsetAsync(bitmap, 0, rows * words * 4, st)), ++nl;
        if (launches) *launches = nl;
        return true;
    }
    if (n > 0x7fffffff) fail(PQKV_EINVAL, "select: too many tokens");
    const bool adc = src.codes != nullptr;
    if (adc && src.m * src.C * 8 > 64 * 1024) {
        // ADC table beyond shared memory (b >= 13 at m = 1..2, PqConfig allows
        // b <= 16): materialize the scores (gather_scores_kernel reads the
        // table from global memory), then select over them -- same keys, same
        // tie rule, two launches more.
        float* scores = nullptr;
        PQKV_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&scores), rows * n * sizeof(float), st));
        launch_score(ctx, src.queries, rows, src.g, src.d_h, src.m, src.C, src.centroids, src.codes,
                     src.codes_head_stride, n, scores, n, st);
        SelectSource ss;
        ss.scores = scores;
        ss.scores_stride = n;
        bool ok = launch_select(ctx, ss, rows, n, k, bitmap, ids, st, launches);
        PQKV_CUDA(cudaFreeAsync(scores, st));
        if (launches) *launches += 2;
        return ok;
    }
    const size_t slice = round_up(ceil_div(n, SEL_CL), 32);
    const size_t fixed = (4 * NB + 8 + 32 + 8) * 4 + (adc ? src.m * src.C * 8 : 0);
    int keys_smem = fixed + slice * 4 <= 200 * 1024;
    size_t smem = fixed + (keys_smem ? slice * 4 : 0);

    Scratch sc(ctx);
    size_t h_keys = sc.plan<uint32_t>(keys_smem ? 1 : rows * n);
    size_t h_sk = sc.plan<uint32_t>(ids ? rows * k : 1), h_si = sc.plan<uint32_t>(ids ? rows * k : 1);
    size_t h_tk = sc.plan<uint32_t>(ids ? rows * k : 1), h_ti = sc.plan<uint32_t>(ids ? rows * k : 1);
    size_t h_status = sc.plan<int>(rows);
    sc.commit();

    SelArgs a{};
    a.queries = src.queries;
    a.g = (int)src.g;
    a.d_h = (int)src.d_h;
    a.m = (int)src.m;
    a.C = (int)src.C;
    a.centroids = src.centroids;
    a.codes = src.codes;
    a.codes_head_stride = (long long)src.codes_head_stride;
    a.scores = src.scores;
    a.scores_stride = (long long)src.scores_stride;
    a.excluded = src.excluded;
    a.n = (int)n;
    a.k = (int)k;
    a.slice = (int)slice;
    a.keys_smem = keys_smem;
    a.gkeys = sc.get<uint32_t>(h_keys);
    a.bitmap = bitmap;
    a.words = (int)words;
    a.sel_key = ids ? sc.get<uint32_t>(h_sk) : nullptr;
    a.sel_id = ids ? sc.get<uint32_t>(h_si) : nullptr;
    a.status = sc.get<int>(h_status);
    if (src.excluded) PQKV_CUDA(cudaMemsetAsync(a.status, 0, rows * sizeof(int), st)), ++nl;

    PQKV_CUDA(cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(rows * SEL_CL));
    cfg.blockDim = dim3(SEL_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = SEL_CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    PQKV_CUDA(cudaLaunchKernelEx(&cfg, select_kernel, a));
    ++nl;
    bool ok = true;
    if (src.excluded) {
        std::vector<int> status(rows);
        PQKV_CUDA(cudaMemcpyAsync(status.data(), a.status, rows * sizeof(int), cudaMemcpyDeviceToHost, st));
        PQKV_CUDA(cudaStreamSynchronize(st));
        for (int s : status) ok = ok && s == 0;
        if (!ok) {
            if (launches) *launches = nl;
            return false;
        }
    }
    if (ids) {
        sort_desc_kernel<<<(unsigned)rows, SORT_THREADS, 0, st>>>(a.sel_key, a.sel_id,
                                                                 sc.get<uint32_t>(h_tk),
                                                                 sc.get<uint32_t>(h_ti), (int)k, ids);
        PQKV_LAUNCHED("sort_desc_kernel");
        ++nl;
    }
    if (launches) *launches = nl;
    return ok;
}


void launch_tuple_tables(pqkv_ctx* ctx, const uint16_t* codes, size_t P, size_t codes_head_stride,
                         size_t C, size_t row_begin, size_t row_end, uint32_t* thist, uint16_t* chist,
                         size_t n_chunks, cudaStream_t st) {
    bind_device(ctx);
    if (row_end <= row_begin || P == 0) return;
    const size_t c1 = ceil_div(row_end, PQKV_TUPLE_CHUNK);
    if (c1 > n_chunks) fail(PQKV_EINVAL, "tuple tables: row range exceeds the chunk table");
    size_t smem = C * C * 4;
    PQKV_CUDA(cudaFuncSetAttribute(tuple_tables_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // blockIdx.x indexes absolute chunks; chunks before c0 exit at once
    tuple_tables_kernel<<<dim3((unsigned)c1, (unsigned)P), 512, smem, st>>>(
        codes, (long long)codes_head_stride, (int)C, (int)row_begin, (int)row_end, thist, chist, (int)n_chunks);
    PQKV_LAUNCHED("tuple_tables_kernel");
}

void launch_tuple_select(pqkv_ctx* ctx, const SelectSource& src, const uint32_t* thist,
                         const uint16_t* chist, size_t rows, size_t n, size_t k, uint8_t* cls, int* cut,
                         uint32_t* tkey, uint32_t* sel_before, cudaStream_t st, unsigned* ready) {
    bind_device(ctx);
    const size_t C = src.C, n_chunks = ceil_div(n, PQKV_TUPLE_CHUNK);
    TupArgs a{};
    a.ready = ready;
    a.q_copy = ready ? src.queries_copy : nullptr;
    a.queries = src.queries;
    a.g = (int)src.g;
    a.d_h = (int)src.d_h;
    a.C = (int)C;
    a.centroids = src.centroids;
    a.thist = thist;
    a.chist = chist;
    a.n = (int)n;
    a.k = (int)k;
    a.n_chunks = (int)n_chunks;
    a.cls = cls;
    a.tkey = tkey;
    a.cut = cut;
    a.sel_before = sel_before;
    a.chunk_stride = (long long)(src.tuple_chunk_stride ? src.tuple_chunk_stride : n_chunks);
    if (a.chunk_stride < (long long)n_chunks) fail(PQKV_EINVAL, "tuple select: chunk table smaller than the rows");
    size_t smem = pair_select_scratch((int)C, (int)n_chunks);
    if (smem > 220 * 1024 || n_chunks > 2 * (size_t)NB) fail(PQKV_EINVAL, "tuple select: table too large");
    const bool wide = C * C > (size_t)4096;
    auto kern = wide ? tuple_select_kernel<TUP_THREADS_B7> : tuple_select_kernel<TUP_THREADS>;
    PQKV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)rows);
    cfg.blockDim = dim3(wide ? TUP_THREADS_B7 : TUP_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    PQKV_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
    PQKV_LAUNCHED("tuple_select_kernel");
}

void launch_select_tuple(pqkv_ctx* ctx, const SelectSource& src, const uint32_t* thist,
                         const uint16_t* chist, size_t rows, size_t n, size_t k, uint32_t* bitmap,
                         int64_t* ids, cudaStream_t st, int* launches) {
    bind_device(ctx);
    const size_t words = ceil_div(n, 32), C = src.C, C2 = C * C;
    const size_t n_chunks = ceil_div(n, PQKV_TUPLE_CHUNK);
    int nl = 0;
    if (rows == 0) return;
    if (k == 0) {
        if (bitmap) PQKV_CUDA(cudaMemsetAsync(bitmap, 0, rows * words * 4, st)), ++nl;
        if (launches) *launches = nl;
        return;
    }
    Scratch sc(ctx);
    size_t h_cls = sc.plan<uint8_t>(rows * C2), h_cut = sc.plan<int>(rows * 2);
    size_t h_tk = sc.plan<uint32_t>(ids ? rows * C2 : 1), h_sb = sc.plan<uint32_t>(ids ? rows * n_chunks : 1);
    size_t h_bm = sc.plan<uint32_t>(bitmap ? 1 : rows * words);
    size_t h_sk = sc.plan<uint32_t>(ids ? rows * k : 1), h_si = sc.plan<uint32_t>(ids ? rows * k : 1);
    size_t h_xk = sc.plan<uint32_t>(ids ? rows * k : 1), h_xi = sc.plan<uint32_t>(ids ? rows * k : 1);
    sc.commit();
    uint8_t* cls = sc.get<uint8_t>(h_cls);
    int* cut = sc.get<int>(h_cut);
    uint32_t* tkey = ids ? sc.get<uint32_t>(h_tk) : nullptr;
    uint32_t* sel_before = ids ? sc.get<uint32_t>(h_sb) : nullptr;
    launch_tuple_select(ctx, src, thist, chist, rows, n, k, cls, cut, tkey, sel_before, st);
    ++nl;
    uint32_t* bm = bitmap ? bitmap : sc.get<uint32_t>(h_bm);
    size_t smem2 = round_up(C2, 16) + (ids ? C2 * 4 : 0);
    PQKV_CUDA(cudaFuncSetAttribute(tuple_bitmap_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
    tuple_bitmap_kernel<<<dim3((unsigned)n_chunks, (unsigned)rows), TB_THREADS, smem2, st>>>(
        src.codes, (long long)src.codes_head_stride, (int)n, (int)C, cls, cut, bm, (int)words, tkey,
        sel_before, ids ? sc.get<uint32_t>(h_sk) : nullptr, ids ? sc.get<uint32_t>(h_si) : nullptr, (int)k,
        (int)n_chunks);
    PQKV_LAUNCHED("tuple_bitmap_kernel");
    ++nl;
    if (ids) {
        sort_desc_kernel<<<(unsigned)rows, SORT_THREADS, 0, st>>>(sc.get<uint32_t>(h_sk), sc.get<uint32_t>(h_si),
                                                                 sc.get<uint32_t>(h_xk), sc.get<uint32_t>(h_xi),
                                                                 (int)k, ids);
        PQKV_LAUNCHED("sort_desc_kernel");
        ++nl;
    }
    if (launches) *launches = nl;
}

}  // namespace pqkv_dev
