// kmeans.cu -- prefill PQ codebook build on sm_100a (hot path A).
//
// Re-implements kmeans_fit (kmeans.cpp:159-190) and pq_construct
// (pq.cpp:42-72) with bit-identical results: every quantity the reference
// computes in fp64 is computed here in fp64 in the same order, with the
// same tie rules.  One CTA owns one (head, subspace) k-means problem for its
// whole life (seed -> assign -> [update -> assign]* -> emit), so a batch of
// P heads x m subspaces is one launch with P*m independent CTAs and no host
// round trips between iterations.
//
// Assign step (kmeans.cpp:86-130).  Two interchangeable evaluators:
//  * EXACT: dist2 (kmeans.cpp:14-21) in fp64 with separate DSUB/DMUL/DADD
//    (no contraction) for every (point, centroid).
//  * FILTERED (default): fp32 distances from the f32-rounded centroids plus a
//    rigorous bound E on |fp32 - fp64| (see certify()).  A point whose
//    best fp32 candidate beats the runner-up by more than both bounds has the
//    same fp64 argmin; every other point is queued and re-evaluated with the
//    exact fp64 scan.  Assignments are therefore identical to EXACT.
// The k-means++ seed (kmeans.cpp:59-84) keeps its two serial fp64 running
// sums (a warp-wide serial scan, prefix stored for the binary search) and
// uses the same filter to skip fp64 distance work that cannot lower min_d2.
// update_means (kmeans.cpp:133-147) accumulates in ascending point order per
// (cluster, dim): warp w owns clusters c = w (mod W) and walks the assignment
// array in order.
#include <cooperative_groups.h>

#include <cfloat>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "internal.cuh"

namespace pqkv_dev {
namespace {

constexpr int KM_THREADS = 256;
constexpr int KM_WARPS = KM_THREADS / 32;

struct KmArgs {
    const float* points;
    long long problem_stride, row_stride;
    int m_sub, n, dim, K, T;
    const unsigned long long* draws;  // [q][K]
    float* centroids_out;             // [q][K][dim]
    uint32_t* assign_out;             // [q][n] or null
    uint16_t* codes;                  // head row-major codes or null
    long long codes_head_stride;
    uint32_t* iterations;
    double* inertia;
    // scratch, per-problem strides in elements
    uint32_t* asg0;
    uint32_t* asg1;
    double* aux0;
    double* aux1;
    double* cen64;   // [q][K*dim]
    double* gsums;   // [q][K*dim] when sums not in smem
    uint32_t* gcounts;
    uint32_t* queue;  // [q][n]
    unsigned long long* stats;
    int counts_smem, sums_smem, cen64_smem, cenf_smem;
    int vec4;  // point rows are 16-byte aligned
    unsigned long long* timers;  // [q][8] per-phase SM cycles (thread 0's view)
    uint16_t* nearseed;          // [q][n] v2: seed index achieving min_d2 (pruning only)
    float* ubound;               // [q][n] v2 Hamerly upper bound (distance to own centroid)
    float* lbound;               // [q][n] v2 Hamerly lower bound (distance to any other)
    float* glb;                  // [q][n][KG] v2 group lower bounds (Yinyang) or null
    uint32_t* lmem;              // [q][n] v2: each CTA's points in assigned-centroid order
};

// Group lower bounds (Yinyang): after seeding the K centroids are grouped
// into KG groups (a few Lloyd steps over the centroids; the grouping only
// affects speed).  Per point: an upper bound on its distance to its own
// centroid and, per group, a lower bound on its distance to every other
// centroid of the group, moved by the largest centroid drift of the group
// after each update (rounded outward).  The assign pass evaluates only the
// groups whose bound does not exceed the point's upper bound (plus its own
// centroid's group); the skipped groups' bounds join the certification of the
// fp32 filter, so the result is still the reference's exact argmin.
constexpr int KG = 8;

struct Smem {
    double* gbuf;      // KM_THREADS*4 doubles (exact_running_sum replay buffer)
    long long* lscr;   // 32 long longs
    uint32_t* counts;
    double* sums;
    double* cen64;   // authoritative fp64 centroids (smem copy or global)
    float* cenf;     // f32-rounded centroids (filter)
    float* cnorm;    // ||cenf_c|| * (1 + 2^-20)
    int* iscratch;   // small block-reduction scratch (64 ints)
    double* dscratch;  // 64 doubles
};

__device__ __forceinline__ const float* point_ptr(const KmArgs& a, int q, int i) {
    return a.points + (long long)(q / a.m_sub) * a.problem_stride +
           (long long)(q % a.m_sub) * a.dim + (long long)i * a.row_stride;
}

// dist2 (kmeans.cpp:14-21) with x read from global, fp64, no contraction.
__device__ __forceinline__ double dist2_g(const float* x, const double* c, int dim) {
    double acc = 0.0;
    for (int t = 0; t < dim; ++t) {
        double diff = __dsub_rn((double)__ldg(x + t), c[t]);
        acc = __dadd_rn(acc, __dmul_rn(diff, diff));
    }
    return acc;
}

template <int D>
__device__ __forceinline__ double dist2_r(const double (&x)[D], const double* c) {
    double acc = 0.0;
#pragma unroll
    for (int t = 0; t < D; ++t) {
        double diff = __dsub_rn(x[t], c[t]);
        acc = __dadd_rn(acc, __dmul_rn(diff, diff));
    }
    return acc;
}

// Exact nearest (kmeans.cpp:86-97): strict <, lowest index on ties.
__device__ uint32_t nearest_g(const float* x, const double* cen, int K, int dim) {
    uint32_t best = 0;
    double best_d = dist2_g(x, cen, dim);
    for (int c = 1; c < K; ++c) {
        double d = dist2_g(x, cen + (long long)c * dim, dim);
        if (d < best_d) {
            best_d = d;
            best = c;
        }
    }
    return best;
}

template <int D>
__device__ uint32_t nearest_r(const double (&x)[D], const double* __restrict__ cen, int K) {
    uint32_t best = 0;
    double best_d = dist2_r<D>(x, cen);
    int c = 1;
    for (; c + 4 <= K; c += 4) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        const double* c0 = cen + c * D;
#pragma unroll
        for (int t = 0; t < D; ++t) {
            double d0 = __dsub_rn(x[t], c0[t]);
            double d1 = __dsub_rn(x[t], c0[D + t]);
            double d2 = __dsub_rn(x[t], c0[2 * D + t]);
            double d3 = __dsub_rn(x[t], c0[3 * D + t]);
            a0 = __dadd_rn(a0, __dmul_rn(d0, d0));
            a1 = __dadd_rn(a1, __dmul_rn(d1, d1));
            a2 = __dadd_rn(a2, __dmul_rn(d2, d2));
            a3 = __dadd_rn(a3, __dmul_rn(d3, d3));
        }
        if (a0 < best_d) { best_d = a0; best = c; }
        if (a1 < best_d) { best_d = a1; best = c + 1; }
        if (a2 < best_d) { best_d = a2; best = c + 2; }
        if (a3 < best_d) { best_d = a3; best = c + 3; }
    }
    for (; c < K; ++c) {
        double d = dist2_r<D>(x, cen + c * D);
        if (d < best_d) { best_d = d; best = c; }
    }
    return best;
}

// ---- fp32 filter ----------------------------------------------------------
//
// For one (point, centroid): S_f = fl32 sum_t fma(d_t, d_t, .) with
// d_t = fl32(x_t - cf_t), cf = f32(c).  With u = 2^-24, S = exact real
// sum (x - c)^2 and S64 the reference's fp64 value:
//   |S_f - S64| <= (D+2)u(1+o(u)) sum(x-cf)^2 + 2u sqrt(S)||c|| + u^2||c||^2
//                  + (D+2) 2^-53 S + subnormal slack,
// and sum(x-cf)^2 <= S + 2u sqrt(S)||c|| + u^2||c||^2.  E() below doubles a
// looser closed form of this (so the rounding of E itself and of the final
// comparison are covered) and adds D*2^-140 for fp32 subnormal underflow.
__device__ __forceinline__ float err_bound(float s, float cnorm, int D) {
    const float u = 5.9604645e-8f;  // 2^-24
    float su = sqrtf(fmaxf(s, 0.0f));
    return 2.0f * ((D + 6) * u * s + 2.0f * u * su * cnorm + (D + 3) * u * u * cnorm * cnorm) +
           D * 7.2e-43f;
}

template <int D>
__device__ __forceinline__ float dist_f(const float (&x)[D], const float* c) {
    float acc = 0.0f;
#pragma unroll
    for (int t = 0; t < D; ++t) {
        float d = x[t] - c[t];
        acc = fmaf(d, d, acc);
    }
    return acc;
}

// Filtered nearest: returns the certified index or -1 (needs fp64 re-check).
template <int D>
__device__ int nearest_filtered(const float (&x)[D], const float* __restrict__ cenf,
                                const float* __restrict__ cnorm, float cnorm_max, int K) {
    float b1 = FLT_MAX, b2 = FLT_MAX;
    int i1 = 0;
    int c = 0;
    for (; c + 4 <= K; c += 4) {
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
        const float* c0 = cenf + c * D;
        if constexpr (D % 4 == 0) {  // 128-bit broadcast reads of the 4 centroid rows
            const float4* q0 = reinterpret_cast<const float4*>(c0);
#pragma unroll
            for (int t4 = 0; t4 < D / 4; ++t4) {
                const float4 v[4] = {q0[t4], q0[D / 4 + t4], q0[D / 2 + t4], q0[3 * D / 4 + t4]};
                float* acc4[4] = {&a0, &a1, &a2, &a3};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    float d;
                    d = x[4 * t4 + 0] - v[e].x; *acc4[e] = fmaf(d, d, *acc4[e]);
                    d = x[4 * t4 + 1] - v[e].y; *acc4[e] = fmaf(d, d, *acc4[e]);
                    d = x[4 * t4 + 2] - v[e].z; *acc4[e] = fmaf(d, d, *acc4[e]);
                    d = x[4 * t4 + 3] - v[e].w; *acc4[e] = fmaf(d, d, *acc4[e]);
                }
            }
        } else {
#pragma unroll
            for (int t = 0; t < D; ++t) {
                float d0 = x[t] - c0[t];
                float d1 = x[t] - c0[D + t];
                float d2 = x[t] - c0[2 * D + t];
                float d3 = x[t] - c0[3 * D + t];
                a0 = fmaf(d0, d0, a0);
                a1 = fmaf(d1, d1, a1);
                a2 = fmaf(d2, d2, a2);
                a3 = fmaf(d3, d3, a3);
            }
        }
        float av[4] = {a0, a1, a2, a3};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            float v = av[e];
            if (v < b1) { b2 = b1; b1 = v; i1 = c + e; }
            else if (v < b2) { b2 = v; }
        }
    }
    for (; c < K; ++c) {
        float v = dist_f<D>(x, cenf + c * D);
        if (v < b1) { b2 = b1; b1 = v; i1 = c; }
        else if (v < b2) { b2 = v; }
    }
    if (K == 1) return 0;
    if (!(b1 < 1e37f) || !(b2 < 1e37f)) return -1;
    // b2 must lie where v - E(v) is increasing (v > ~u^2 ||c||max^2) so that
    // the runner-up bound also covers every farther centroid.
    const float u = 5.9604645e-8f;
    if (!(b2 > 8.0f * u * u * cnorm_max * cnorm_max)) return -1;
    float e1 = err_bound(b1, cnorm[i1], D);
    float e2 = err_bound(b2, cnorm_max, D);
    return (b2 - e2 > b1 + e1) ? i1 : -1;
}

// Point row -> registers, 128-bit loads when the row is 16-byte aligned.
template <int D>
__device__ __forceinline__ void load_point(const float* xp, float (&x)[D], bool vec4) {
    if constexpr (D % 4 == 0) {
        if (vec4) {
            const float4* x4 = reinterpret_cast<const float4*>(xp);
#pragma unroll
            for (int t = 0; t < D / 4; ++t) {
                float4 v = __ldg(x4 + t);
                x[4 * t] = v.x;
                x[4 * t + 1] = v.y;
                x[4 * t + 2] = v.z;
                x[4 * t + 3] = v.w;
            }
            return;
        }
    }
#pragma unroll
    for (int t = 0; t < D; ++t) x[t] = __ldg(xp + t);
}

// Filtered nearest that also returns Hamerly bounds for a certified point:
// ub >= true distance to the returned centroid, lb <= true distance to every
// other centroid (both rounded outward).  Returns -1 when not certified.
template <int D>
__device__ int nearest_filtered_b(const float (&x)[D], const float* __restrict__ cenf,
                                  const float* __restrict__ cnorm, float cnorm_max, int K, float& ub,
                                  float& lb) {
    float b1 = FLT_MAX, b2 = FLT_MAX;
    int i1 = 0;
    int c = 0;
    for (; c + 4 <= K; c += 4) {
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
        const float* c0 = cenf + c * D;
        if constexpr (D % 4 == 0) {  // 128-bit broadcast reads of the 4 centroid rows
            const float4* q0 = reinterpret_cast<const float4*>(c0);
#pragma unroll
            for (int t4 = 0; t4 < D / 4; ++t4) {
                const float4 v[4] = {q0[t4], q0[D / 4 + t4], q0[D / 2 + t4], q0[3 * D / 4 + t4]};
                float* acc4[4] = {&a0, &a1, &a2, &a3};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    float d;
                    d = x[4 * t4 + 0] - v[e].x; *acc4[e] = fmaf(d, d, *acc4[e]);
                    d = x[4 * t4 + 1] - v[e].y; *acc4[e] = fmaf(d, d, *acc4[e]);
                    d = x[4 * t4 + 2] - v[e].z; *acc4[e] = fmaf(d, d, *acc4[e]);
                    d = x[4 * t4 + 3] - v[e].w; *acc4[e] = fmaf(d, d, *acc4[e]);
                }
            }
        } else {
#pragma unroll
            for (int t = 0; t < D; ++t) {
                float d0 = x[t] - c0[t];
                float d1 = x[t] - c0[D + t];
                float d2 = x[t] - c0[2 * D + t];
                float d3 = x[t] - c0[3 * D + t];
                a0 = fmaf(d0, d0, a0);
                a1 = fmaf(d1, d1, a1);
                a2 = fmaf(d2, d2, a2);
                a3 = fmaf(d3, d3, a3);
            }
        }
        float av[4] = {a0, a1, a2, a3};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            float v = av[e];
            if (v < b1) { b2 = b1; b1 = v; i1 = c + e; }
            else if (v < b2) { b2 = v; }
        }
    }
    for (; c < K; ++c) {
        float v = dist_f<D>(x, cenf + c * D);
        if (v < b1) { b2 = b1; b1 = v; i1 = c; }
        else if (v < b2) { b2 = v; }
    }
    if (!(b1 < 1e37f)) return -1;
    const float e1 = err_bound(b1, cnorm[i1], D);
    ub = __fsqrt_ru(__fmul_ru(__fadd_ru(b1, e1), 1.000001f));
    if (K == 1) { lb = INFINITY; return 0; }
    const float u = 5.9604645e-8f;
    if (!(b2 < 1e37f) || !(b2 > 8.0f * u * u * cnorm_max * cnorm_max)) return -1;
    const float e2 = err_bound(b2, cnorm_max, D);
    if (!(b2 - e2 > b1 + e1)) return -1;
    lb = __fsqrt_rd(fmaxf(0.f, __fmul_rd(__fsub_rd(b2, e2), 0.999999f)));
    return i1;
}

// ---- block helpers --------------------------------------------------------

__device__ __forceinline__ void block_sync() { __syncthreads(); }

// Serial fp64 running sum over v[0..n) in index order (kmeans.cpp:64-65,
// 149-154), run by one warp; every lane carries the identical sum.  If
// `prefix` is non-null the running value after element i is stored there.
__device__ double warp_serial_sum(const double* v, int n, double* prefix) {
    int lane = threadIdx.x & 31;
    double total = 0.0;
    double cur = (lane < n) ? v[lane] : 0.0;
    for (int i0 = 0; i0 < n; i0 += 32) {
        int nxt = i0 + 32 + lane;
        double pre = (nxt < n) ? v[nxt] : 0.0;  // prefetch next tile
        double mine = 0.0;
        int cnt = min(32, n - i0);
        if (cnt == 32) {
#pragma unroll
            for (int l = 0; l < 32; ++l) {
                double e = __shfl_sync(FULL, cur, l);
                total = __dadd_rn(total, e);
                if (lane == l) mine = total;
            }
        } else {
            for (int l = 0; l < cnt; ++l) {
                double e = __shfl_sync(FULL, cur, l);
                total = __dadd_rn(total, e);
                if (lane == l) mine = total;
            }
        }
        if (prefix && lane < cnt) prefix[i0 + lane] = mine;
        cur = pre;
    }
    return total;
}

// Exact, block-parallel reproduction of the serial fp64 running sum
//   S_{-1} = +0.0,  S_i = fl(S_{i-1} + v_i),  v_i >= 0
// of k-means++ (kmeans.cpp:64-65 total, 70-71 cum); S_i is stored in pre[i]
// and S_{n-1} is returned to every thread.  While S stays inside one binade
// [2^e, 2^(e+1)) every step is S + round_u(v_i) with u = ulp(S) (S is a
// multiple of u, so round-to-nearest of S + v_i only rounds v_i), so a run
// of such steps is exact as S + u * (integer prefix of round_u(v_i)).  The
// first element that would leave the binade, that is a tie (v_i mod u ==
// u/2, where round-half-even depends on S), or that meets S == 0 /
// subnormal, is done serially by one thread; the parallel pass then resumes
// after it.  No approximation is ever accepted.
__device__ double exact_running_sum(const double* v, int n, double* pre, double* gbuf,
                                    long long* iscr, double* dsh, double S_init = 0.0) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int E = 4, GROUP = KM_THREADS * E;
    int* ish = reinterpret_cast<int*>(iscr + 2 * KM_WARPS);
    double S = S_init;
    double nx[E];  // next group's values, prefetched while this group runs
#pragma unroll
    for (int e = 0; e < E; ++e) nx[e] = tid * E + e < n ? v[tid * E + e] : 0.0;
    for (int g0 = 0; g0 < n; g0 += GROUP) {
        const int cnt = min(GROUP, n - g0);
        double a[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int li = tid * E + e;
            a[e] = nx[e];
            gbuf[li] = a[e];
            nx[e] = g0 + GROUP + li < n ? v[g0 + GROUP + li] : 0.0;
        }
        __syncthreads();
        int j = 0;  // first element of the group not yet summed (block uniform)
        while (j < cnt) {
            const long long sb = __double_as_longlong(S);
            const int expo = (int)((sb >> 52) & 0x7ff);
            const bool normal = S > 0.0 && expo > 52 && expo < 2046;
            double u = 0.0, inv_u = 0.0, top = 0.0;
            long long d[E];
            bool bad[E];
            long long dsum = 0;
            if (normal) {
                u = __longlong_as_double((long long)(expo - 52) << 52);
                inv_u = __longlong_as_double((long long)(2098 - expo) << 52);  // 1/u, exact
                top = __longlong_as_double((long long)(expo + 1) << 52);        // 2^(e+1)
            }
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int li = tid * E + e;
                d[e] = 0;
                bad[e] = false;
                if (li >= j && li < cnt) {
                    if (!normal) {
                        bad[e] = true;
                    } else {
                        const double qv = a[e] * inv_u;  // exact power-of-two scaling
                        const double fl = floor(qv), fr = qv - fl;
                        bad[e] = !(qv < 4503599627370496.0) || fr == 0.5;
                        d[e] = bad[e] ? 0 : (long long)fl + (fr > 0.5 ? 1 : 0);
                    }
                }
                dsum += d[e];
            }
            long long x = dsum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                long long y = __shfl_up_sync(FULL, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) iscr[warp] = x;
            if (tid == 0) ish[0] = cnt;  // first stop index
            __syncthreads();
            long long run = x - dsum;
            for (int w = 0; w < warp; ++w) run += iscr[w];
            // first element that is bad or whose exact-in-binade sum reaches top
            int stop = cnt;
            long long r2 = run;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int li = tid * E + e;
                if (li >= j && li < cnt && stop == cnt) {
                    r2 += d[e];
                    if (bad[e] || !(S + (double)r2 * u < top)) stop = li;
                }
            }
            if (stop < cnt) atomicMin(&ish[0], stop);
            __syncthreads();
            const int xs = ish[0];
            // accept [j, xs)
            r2 = run;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int li = tid * E + e;
                if (li >= j && li < xs) {
                    r2 += d[e];
                    pre[g0 + li] = S + (double)r2 * u;
                }
            }
            // new S = value at xs - 1 (held by the thread owning xs - 1)
            if (xs > j && (xs - 1) / E == tid) {
                long long r3 = run;
                for (int e = 0; e <= (xs - 1) % E; ++e) r3 += d[e];
                dsh[0] = S + (double)r3 * u;
            }
            __syncthreads();
            if (xs > j) S = dsh[0];
            if (xs < cnt) {  // the stop element, serially
                if (tid == 0) {
                    const double s2 = __dadd_rn(S, gbuf[xs]);
                    pre[g0 + xs] = s2;
                    dsh[1] = s2;
                }
                __syncthreads();
                S = dsh[1];
                j = xs + 1;
            } else {
                j = cnt;
            }
            __syncthreads();  // iscr / ish / dsh reuse
        }
    }
    return S;
}

// Speculative part of a cluster-split running sum: the slice v[0..m) will be
// entered with an exact S that is only known later, but within 1e-9
// relative of P (the fp64 sum of the earlier slices; the serial sum differs
// from it by << 1e-9 relative for any realistic n).  When P is safely inside
// one binade [2^e, 2^(e+1)) the exact S is a multiple of u = ulp(2^e), every
// step is S + round_u(v_j), and the slice is an integer prefix sum: the
// inclusive prefix I_j (as a double, exact) goes to pre[j].  Returns false
// when P is near a binade edge, an element is a rounding tie / out of range,
// or the slice could leave the binade (the caller then runs the serial
// exact sum for the slice).  *u_out, *iend_out on success.
__device__ bool slice_increments(const double* v, int m, double P, double* pre, long long* iscr, double* u_out,
                                 long long* iend_out) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int E = 4, GROUP = KM_THREADS * E;
    __shared__ int bad_s;
    const long long pb = __double_as_longlong(P);
    const int expo = (int)((pb >> 52) & 0x7ff);
    if (!(P > 0.0) || expo <= 52 || expo >= 2045) return false;  // uniform
    const double lo_edge = __longlong_as_double((long long)expo << 52);
    const double top = __longlong_as_double((long long)(expo + 1) << 52);
    if (!(P * (1.0 - 1e-9) >= lo_edge) || !(P * (1.0 + 1e-9) < top)) return false;
    const double u = __longlong_as_double((long long)(expo - 52) << 52);
    const double inv_u = __longlong_as_double((long long)(2098 - expo) << 52);
    if (tid == 0) bad_s = 0;
    __syncthreads();
    long long carry = 0;
    for (int g0 = 0; g0 < m; g0 += GROUP) {
        long long d[E], dsum = 0;
        int bad = 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int j = g0 + tid * E + e;
            d[e] = 0;
            if (j < m) {
                const double qv = v[j] * inv_u;
                const double fl = floor(qv), fr = qv - fl;
                if (!(qv < 4503599627370496.0) || fr == 0.5 || !(qv >= 0.0)) bad = 1;
                else d[e] = (long long)fl + (fr > 0.5 ? 1 : 0);
            }
            dsum += d[e];
        }
        if (bad) bad_s = 1;
        long long x = dsum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(FULL, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) iscr[warp] = x;
        __syncthreads();
        long long run = carry + x - dsum, tile = 0;
        for (int w = 0; w < KM_WARPS; ++w) {
            if (w < warp) run += iscr[w];
            tile += iscr[w];
        }
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int j = g0 + tid * E + e;
            run += d[e];
            if (j < m) pre[j] = (double)run;
        }
        carry += tile;
        __syncthreads();
    }
    const bool ok = !bad_s && carry < (1ll << 53) && P * (1.0 + 1e-9) + (double)carry * u < top;
    *u_out = u;
    *iend_out = carry;
    return ok;
}

// First i in [0, n) with pre[i] >= target (pre non-decreasing; n-1 if none),
// by one warp with 32-ary probing.
__device__ int warp_lower_bound(const double* pre, int n, double target) {
    const int lane = threadIdx.x & 31;
    int lo = 0, hi = n - 1;  // answer in [lo, hi]
    while (hi - lo >= 32) {
        const int span = hi - lo + 1;
        const int step = (span + 31) / 32;
        const int pidx = min(lo + lane * step + step - 1, hi);  // last index of lane's bucket
        const bool ge = pre[pidx] >= target;
        const unsigned m = __ballot_sync(FULL, ge);
        const int f = m ? __ffs(m) - 1 : 31;
        const int nlo = lo + f * step;
        hi = m ? min(lo + f * step + step - 1, hi) : hi;
        lo = nlo;
    }
    const int idx = lo + lane;
    const bool ge = idx <= hi && pre[idx] >= target;
    const unsigned m = __ballot_sync(FULL, ge);
    return m ? lo + __ffs(m) - 1 : n - 1;
}

// ---- the per-problem kernel -------------------------------------------------

// D > 0: compile-time subspace dim, point held in registers (fp32 for the
// filter, fp64 for EXACT).  D == 0: runtime dim, exact, global centroids.
template <int D, bool FILTER>
__global__ void __launch_bounds__(KM_THREADS, 1) kmeans_problem_kernel(KmArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int q = blockIdx.x;
    const int n = a.n, K = a.K, dim = (D > 0 ? D : a.dim), T = a.T;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long KD = (long long)K * dim;

    // ---- carve shared memory (layout planned on the host, same order) ----
    Smem s;
    {
        unsigned char* p = smem_raw;
        s.gbuf = reinterpret_cast<double*>(p);
        p += KM_THREADS * 4 * sizeof(double);
        s.lscr = reinterpret_cast<long long*>(p);
        p += 32 * sizeof(long long);
        s.iscratch = reinterpret_cast<int*>(p);
        p += 64 * sizeof(int);
        s.dscratch = reinterpret_cast<double*>(p);
        p += 64 * sizeof(double);
        if (a.counts_smem) { s.counts = reinterpret_cast<uint32_t*>(p); p += ((K * 4 + 15) / 16) * 16; }
        else s.counts = a.gcounts + (long long)q * K;
        if (a.sums_smem) { s.sums = reinterpret_cast<double*>(p); p += KD * 8; }
        else s.sums = a.gsums + q * KD;
        if (a.cen64_smem) { s.cen64 = reinterpret_cast<double*>(p); p += KD * 8; }
        else s.cen64 = a.cen64 + q * KD;
        if (a.cenf_smem) {
            s.cenf = reinterpret_cast<float*>(p); p += ((KD * 4 + 15) / 16) * 16;
            s.cnorm = reinterpret_cast<float*>(p); p += ((K * 4 + 15) / 16) * 16;
        } else { s.cenf = nullptr; s.cnorm = nullptr; }
    }
    uint32_t* asg = a.asg0 + (long long)q * n;
    uint32_t* nxt = a.asg1 + (long long)q * n;
    double* aux0 = a.aux0 + (long long)q * n;
    double* aux1 = a.aux1 + (long long)q * n;
    uint32_t* queue = a.queue + (long long)q * n;
    __shared__ int sh_int[4];
    __shared__ float sh_cmax;
    // phase timers: 0 seed chain, 1 seed distances, 2 assign+repair, 3 -, 4 update, 5 other
    unsigned long long t_acc[6] = {0, 0, 0, 0, 0, 0};
    unsigned long long t_last = clock64();
    auto tick = [&](int ph) {
        if (tid == 0) {
            unsigned long long now = clock64();
            t_acc[ph] += now - t_last;
            t_last = now;
        }
    };

    // refresh the f32 copy + norms after the fp64 centroids change
    auto refresh_f32 = [&]() {
        if (!FILTER) return;
        for (long long e = tid; e < KD; e += KM_THREADS) s.cenf[e] = (float)s.cen64[e];
        block_sync();
        if (tid == 0) sh_cmax = 0.f;
        block_sync();
        for (int c = tid; c < K; c += KM_THREADS) {
            float acc = 0.f;
            for (int t = 0; t < dim; ++t) acc = fmaf(s.cenf[c * dim + t], s.cenf[c * dim + t], acc);
            float nrm = sqrtf(acc) * (1.0f + 9.6e-7f) + 1e-30f;
            s.cnorm[c] = nrm;
            atomicMax(reinterpret_cast<int*>(&sh_cmax), __float_as_int(nrm));  // nrm >= 0
        }
        block_sync();
    };
    auto set_centroid_from_point = [&](int c, int i) {
        const float* x = point_ptr(a, q, i);
        for (int t = tid; t < dim; t += KM_THREADS) s.cen64[(long long)c * dim + t] = (double)x[t];
    };

    // exact nearest for one point, x from global
    auto exact_nearest_g = [&](int i) -> uint32_t {
        return nearest_g(point_ptr(a, q, i), s.cen64, K, dim);
    };

    // ---- one assignment pass with repair (kmeans.cpp:103-130) ----
    // writes out[], s.counts; returns after the block has synchronised.
    auto assign_with_repair = [&](uint32_t* out) {
        for (int c = tid; c < K; c += KM_THREADS) s.counts[c] = 0;
        if (tid == 0) sh_int[0] = 0;  // queue length
        block_sync();
        if constexpr (FILTER) {
            float cmax = sh_cmax;
            for (int i = tid; i < n; i += KM_THREADS) {
                float x[D > 0 ? D : 1];
                load_point<(D > 0 ? D : 1)>(point_ptr(a, q, i), x, a.vec4);
                int c = nearest_filtered<(D > 0 ? D : 1)>(x, s.cenf, s.cnorm, cmax, K);
                if (c >= 0) {
                    out[i] = (uint32_t)c;
                    atomicAdd(&s.counts[c], 1u);
                } else {
                    int slot = atomicAdd(&sh_int[0], 1);
                    queue[slot] = (uint32_t)i;
                }
            }
            block_sync();
            int qn = sh_int[0];
            for (int e = tid; e < qn; e += KM_THREADS) {
                int i = (int)queue[e];
                uint32_t c = exact_nearest_g(i);
                out[i] = c;
                atomicAdd(&s.counts[c], 1u);
            }
            if (tid == 0 && a.stats) {
                atomicAdd(&a.stats[0], (unsigned long long)qn);
                atomicAdd(&a.stats[1], (unsigned long long)n);
            }
        } else {
            for (int i = tid; i < n; i += KM_THREADS) {
                uint32_t c;
                if constexpr (D > 0) {
                    float xf[D];
                    load_point<D>(point_ptr(a, q, i), xf, a.vec4);
                    double x[D];
#pragma unroll
                    for (int t = 0; t < D; ++t) x[t] = (double)xf[t];
                    c = nearest_r<D>(x, s.cen64, K);
                } else {
                    c = exact_nearest_g(i);
                }
                out[i] = c;
                atomicAdd(&s.counts[c], 1u);
            }
        }
        block_sync();
        if (n < K) return;
        // any empty cluster?
        int empty = 0;
        for (int c = tid; c < K; c += KM_THREADS) empty |= (s.counts[c] == 0);
        if (!__syncthreads_or(empty)) return;
        // Rare path: donor repair.  d_i = dist2(p_i, mu_assign[i]) is fixed for
        // every point that stays put; a moved donor becomes ineligible.
        for (int i = tid; i < n; i += KM_THREADS)
            aux0[i] = dist2_g(point_ptr(a, q, i), s.cen64 + (long long)out[i] * dim, dim);
        block_sync();
        for (int c = 0; c < K; ++c) {
            if (s.counts[c] != 0) continue;  // uniform: counts read after a sync
            double best = -1.0;
            int bi = n;
            for (int i = tid; i < n; i += KM_THREADS) {
                if (s.counts[out[i]] < 2) continue;
                double d = aux0[i];
                if (d > best) { best = d; bi = i; }  // ascending i per thread: first max kept
            }
            // block arg-max: larger d wins, then lower index
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                double ob = __shfl_xor_sync(FULL, best, o);
                int oi = __shfl_xor_sync(FULL, bi, o);
                if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
            }
            if (lane == 0) { s.dscratch[warp] = best; s.iscratch[warp] = bi; }
            block_sync();
            if (tid == 0) {
                double b = s.dscratch[0];
                int ii = s.iscratch[0];
                for (int w = 1; w < KM_WARPS; ++w) {
                    double ob = s.dscratch[w];
                    int oi = s.iscratch[w];
                    if (ob > b || (ob == b && oi < ii)) { b = ob; ii = oi; }
                }
                sh_int[1] = ii;
            }
            block_sync();
            int donor = sh_int[1];
            if (donor >= n) break;  // fewer distinct points than clusters
            if (tid == 0) {
                s.counts[out[donor]] -= 1;
                out[donor] = (uint32_t)c;
                s.counts[c] += 1;
            }
            block_sync();
        }
        block_sync();
    };

    // ---- update_means (kmeans.cpp:133-147), ordered per (cluster, dim) ----
    // Warp w owns clusters c = w (mod KM_WARPS) and walks the assignment array
    // in index order; member rows are fetched 8 at a time before the ordered
    // fp64 accumulation so the chain does not wait on L2 per member.
    auto update_means = [&](const uint32_t* as) {
        for (long long e = tid; e < KD; e += KM_THREADS) s.sums[e] = 0.0;
        block_sync();
        constexpr int MB = 8;   // members prefetched per batch
        constexpr int DPL = 4;  // dims per lane handled by the prefetch path (dim <= 128)
        const bool pre = dim <= 32 * DPL;
        for (int i0 = 0; i0 < n; i0 += 32) {
            int i = i0 + lane;
            uint32_t c = (i < n) ? as[i] : 0xffffffffu;
            unsigned mine = __ballot_sync(FULL, i < n && (int)(c % KM_WARPS) == warp);
            while (mine) {
                int ml[MB];
                int cnt = 0;
#pragma unroll
                for (int u = 0; u < MB; ++u) {
                    ml[u] = mine ? __ffs(mine) - 1 : -1;
                    if (mine) { mine &= mine - 1; ++cnt; }
                }
                if (pre) {
                    float xv[MB][DPL];
#pragma unroll
                    for (int u = 0; u < MB; ++u) {
                        const float* xp = ml[u] >= 0 ? point_ptr(a, q, i0 + ml[u]) : nullptr;
#pragma unroll
                        for (int e = 0; e < DPL; ++e) {
                            const int t = lane + 32 * e;
                            xv[u][e] = (xp && t < dim) ? __ldg(xp + t) : 0.f;
                        }
                    }
#pragma unroll
                    for (int u = 0; u < MB; ++u) {
                        if (u >= cnt) break;
                        uint32_t cc = __shfl_sync(FULL, c, ml[u]);
                        double* srow = s.sums + (long long)cc * dim;
#pragma unroll
                        for (int e = 0; e < DPL; ++e) {
                            const int t = lane + 32 * e;
                            if (t < dim) srow[t] = __dadd_rn(srow[t], (double)xv[u][e]);
                        }
                    }
                } else {
                    for (int u = 0; u < cnt; ++u) {
                        uint32_t cc = __shfl_sync(FULL, c, ml[u]);
                        const float* xp = point_ptr(a, q, i0 + ml[u]);
                        double* srow = s.sums + (long long)cc * dim;
                        for (int t = lane; t < dim; t += 32) srow[t] = __dadd_rn(srow[t], (double)__ldg(xp + t));
                    }
                }
            }
        }
        block_sync();
        for (long long e = tid; e < KD; e += KM_THREADS) {
            uint32_t cnt = s.counts[e / dim];
            if (cnt != 0) s.cen64[e] = __ddiv_rn(s.sums[e], (double)cnt);
        }
        block_sync();
    };

    // =====================================================================
    // 1. seeding
    // =====================================================================
    const unsigned long long* draws = a.draws + (long long)q * K;
    if (n <= K) {
        // seed_from_distinct (kmeans.cpp:44-57): first appearance, memcmp
        for (int i = tid; i < n; i += KM_THREADS) {
            const uint32_t* xi = reinterpret_cast<const uint32_t*>(point_ptr(a, q, i));
            int seen = 0;
            for (int j = 0; j < i && !seen; ++j) {
                const uint32_t* xj = reinterpret_cast<const uint32_t*>(point_ptr(a, q, j));
                int eq = 1;
                for (int t = 0; t < dim && eq; ++t) eq = (xi[t] == xj[t]);
                seen = eq;
            }
            asg[i] = seen ? 0u : 1u;  // distinct flag (asg reused as scratch)
        }
        block_sync();
        if (tid == 0) {  // n <= K is small; ordered compaction by one thread
            int nd = 0;
            for (int i = 0; i < n; ++i)
                if (asg[i]) nxt[nd++] = (uint32_t)i;
            sh_int[2] = nd;
        }
        block_sync();
        int nd = sh_int[2];
        for (long long e = tid; e < KD; e += KM_THREADS) {
            int c = (int)(e / dim), t = (int)(e % dim);
            int src = (int)nxt[c < nd - 1 ? c : nd - 1];
            s.cen64[e] = (double)point_ptr(a, q, src)[t];
        }
        block_sync();
    } else {
        // seed_plus_plus (kmeans.cpp:59-84) with the pre-drawn mt19937_64 stream
        int c0 = (int)(draws[0] % (unsigned long long)n);
        set_centroid_from_point(0, c0);
        block_sync();
        for (int i = tid; i < n; i += KM_THREADS)
            aux0[i] = dist2_g(point_ptr(a, q, i), s.cen64, dim);
        for (int c = 1; c < K; ++c) {
            block_sync();
            tick(1);
            {
                double total = exact_running_sum(aux0, n, aux1, s.gbuf, s.lscr, s.dscratch);
                __syncthreads();  // aux1 (prefix) visible to warp 0's search
                if (warp == 0) {
                    int chosen;
                    if (total > 0.0) {
                        double u = (double)(draws[c] >> 11) * 0x1.0p-53;
                        double target = __dmul_rn(u, total);
                        // first i with cum >= target (kmeans.cpp:70-74): prefix is non-decreasing
                        chosen = warp_lower_bound(aux1, n, target);
                    } else {
                        chosen = (int)(draws[c] % (unsigned long long)n);
                    }
                    if (lane == 0) sh_int[3] = chosen;
                }
            }
            block_sync();
            tick(0);
            set_centroid_from_point(c, sh_int[3]);
            block_sync();
            const double* cc = s.cen64 + (long long)c * dim;
            if constexpr (FILTER) {
                // fp32 screen: skip the fp64 distance when it cannot be < min_d2
                float cf[D > 0 ? D : 1];
                float cn = 0.f;
#pragma unroll
                for (int t = 0; t < (D > 0 ? D : 1); ++t) { cf[t] = (float)cc[t]; cn = fmaf(cf[t], cf[t], cn); }
                cn = sqrtf(cn) * (1.0f + 9.6e-7f) + 1e-30f;
                for (int i = tid; i < n; i += KM_THREADS) {
                    const float* xp = point_ptr(a, q, i);
                    float xr[D > 0 ? D : 1];
                    load_point<(D > 0 ? D : 1)>(xp, xr, a.vec4);
                    float acc = 0.f;
#pragma unroll
                    for (int t = 0; t < (D > 0 ? D : 1); ++t) {
                        float d = xr[t] - cf[t];
                        acc = fmaf(d, d, acc);
                    }
                    double old = aux0[i];
                    if (acc < 1e37f && (double)(acc - err_bound(acc, cn, D)) > old) continue;
                    double d = dist2_g(xp, cc, dim);
                    if (d < old) aux0[i] = d;
                }
            } else {
                for (int i = tid; i < n; i += KM_THREADS) {
                    double d = dist2_g(point_ptr(a, q, i), cc, dim);
                    if (d < aux0[i]) aux0[i] = d;
                }
            }
        }
        block_sync();
        tick(1);
    }
    refresh_f32();
    tick(5);

    // =====================================================================
    // 2. Lloyd iterations (kmeans.cpp:174-183)
    // =====================================================================
    assign_with_repair(asg);
    tick(2);
    int iters = 0;
    for (int iter = 1; iter <= T; ++iter) {
        update_means(asg);
        tick(4);
        if (a.inertia) {
            for (int i = tid; i < n; i += KM_THREADS)
                aux0[i] = dist2_g(point_ptr(a, q, i), s.cen64 + (long long)asg[i] * dim, dim);
            block_sync();
            if (warp == 0) {
                double tot = warp_serial_sum(aux0, n, nullptr);
                if (lane == 0) a.inertia[(long long)q * T + iter - 1] = tot;
            }
            block_sync();
        }
        iters = iter;
        refresh_f32();
        tick(5);
        assign_with_repair(nxt);
        tick(2);
        int changed = 0;
        for (int i = tid; i < n; i += KM_THREADS) changed |= (nxt[i] != asg[i]);
        if (!__syncthreads_or(changed)) break;
        uint32_t* t = asg;
        asg = nxt;
        nxt = t;
    }

    // =====================================================================
    // 3. emit: f32 centroids (kmeans.cpp:186-188), codes (pq.cpp:68-69)
    // =====================================================================
    for (long long e = tid; e < KD; e += KM_THREADS) a.centroids_out[q * KD + e] = (float)s.cen64[e];
    if (a.assign_out)
        for (int i = tid; i < n; i += KM_THREADS) a.assign_out[(long long)q * n + i] = asg[i];
    if (a.codes) {
        int head = q / a.m_sub, j = q % a.m_sub;
        uint16_t* cd = a.codes + (long long)head * a.codes_head_stride + j;
        for (int i = tid; i < n; i += KM_THREADS) cd[(long long)i * a.m_sub] = (uint16_t)asg[i];
    }
    if (a.iterations && tid == 0) a.iterations[q] = (uint32_t)iters;
    tick(5);
    if (tid == 0 && a.timers)
        for (int ph = 0; ph < 6; ++ph) a.timers[(long long)q * 8 + ph] = t_acc[ph];
}

// ---- pq_encode_one (pq.cpp:74-99): one CTA per head, one warp per subspace
__global__ void encode_kernel(const float* keys, long long key_stride, int d_h, int m, int C,
                              const float* centroids, uint16_t* codes,
                              long long codes_head_stride, long long row) {
    int p = blockIdx.x;
    int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int d_m = d_h / m;
    const float* key = keys + p * key_stride;
    const float* cen = centroids + (long long)p * m * C * d_m;
    for (int j = warp; j < m; j += nw) {
        double best = INFINITY;
        int bi = 0x7fffffff;
        for (int c = lane; c < C; c += 32) {
            const float* cc = cen + ((long long)j * C + c) * d_m;
            double acc = 0.0;
            for (int t = 0; t < d_m; ++t) {
                double diff = __dsub_rn((double)key[j * d_m + t], (double)cc[t]);
                acc = __dadd_rn(acc, __dmul_rn(diff, diff));
            }
            if (acc < best) { best = acc; bi = c; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            double ob = __shfl_xor_sync(FULL, best, o);
            int oi = __shfl_xor_sync(FULL, bi, o);
            if (ob < best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        if (lane == 0) codes[p * codes_head_stride + row * m + j] = (uint16_t)(bi == 0x7fffffff ? 0 : bi);
    }
}

// ---- assign_nearest (kmeans.cpp:192-220): thread per point ----------------
__global__ void assign_nearest_kernel(const float* points, int n, int dim, const float* cen,
                                      int K, uint32_t* out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float* x = points + (long long)i * dim;
    uint32_t best = 0;
    double best_d = INFINITY;
    for (int c = 0; c < K; ++c) {
        const float* cc = cen + (long long)c * dim;
        double acc = 0.0;
        for (int t = 0; t < dim; ++t) {
            double diff = __dsub_rn((double)x[t], (double)cc[t]);
            acc = __dadd_rn(acc, __dmul_rn(diff, diff));
        }
        if (acc < best_d) { best_d = acc; best = c; }
    }
    out[i] = best;
}

// =============================================================================
// v2: one thread-block CLUSTER of R CTAs per problem (R = 1..8, so a batch of
// few problems still fills the GPU).  CTA r owns the point slice
// [r*ceil(n/R), ...).  Cluster-wide state: counts merged through DSMEM, the
// k-means++ running sum and the rare repair run on rank 0, centroids
// broadcast through global memory after each update.
//
// update_means (kmeans.cpp:133-147) without the sequential walk: the sum of
// a (cluster, dim) chain of f32 values in fp64 never rounds -- in ANY order --
// when sum|x| < 2^52 * ulp_min, ulp_min the smallest f32 ulp among its nonzero
// members (every partial sum is then a multiple of ulp_min below 2^53 ulp_min,
// hence representable).  Such chains are reduced in parallel over a stable
// member list (counting sort by cluster); a chain that fails the check is
// recomputed in point order.  Either way the means are bit-identical.
// =============================================================================
constexpr int V2_MG = 4;  // member groups per warp in the parallel reduction

struct V2Smem {
    double* gbuf;
    long long* lscr;
    int* iscratch;
    double* dscratch;
    uint32_t* cnt_loc;   // [K] this slice
    uint32_t* cnt_all;   // [K] cluster total
    uint32_t* moff;      // [K] member-list offsets
    uint32_t* run;       // [K] scatter cursors
    uint32_t* wcnt;      // [KM_WARPS][K]
    float* cenf;         // [K*D]
    float* cnorm;        // [K]
    double* cen64;       // [K*D]
    double* dseed2;      // [K] squared distance of seed j to the newest seed
    float* delta;        // [K] centroid movement of the last update (rounded up)
    float* ncf;          // [K] |cf|^2 in fp32
    float* cenfg;        // [K*D] cenf in group order (Yinyang)
    float* cnormg;       // [K] cnorm in group order
    int* grp;            // [K] group of centroid c
    int* gorder;         // [K] centroid at group-order position
    uint32_t* lrun;      // [K] CTA-local member-list cursors
};

__host__ __device__ inline size_t v2_smem_bytes(int K, int D) {
    size_t b = (size_t)KM_THREADS * 4 * 8 + 32 * 8 + 64 * 4 + 64 * 8;
    b += (size_t)4 * K * 4 + (size_t)KM_WARPS * K * 4;
    b = (b + 15) / 16 * 16;
    b += (size_t)K * D * 4 + (size_t)K * 4;
    b = (b + 15) / 16 * 16;
    b += (size_t)K * D * 8 + (size_t)K * 8 + (size_t)K * 4 + (size_t)K * 4;
    b = (b + 15) / 16 * 16;
    b += (size_t)K * D * 4 + (size_t)K * 4 * 4;  // Yinyang tables
    return b;
}

// Two CTAs per SM for D <= 64: the seeding, update and assign loops are
// latency-bound row gathers, so warps in flight matter more than registers
// (D = 128 rows would spill).
constexpr int km_v2_occ(int dim) { return dim >= 128 ? 1 : 2; }
template <int D>
__global__ void __launch_bounds__(KM_THREADS, km_v2_occ(D)) kmeans_cluster_kernel(KmArgs a, uint32_t* members_g) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int R = (int)cl.num_blocks();
    const int r = (int)cl.block_rank();
    const int q = blockIdx.x / R;
    const int n = a.n, K = a.K, T = a.T;
    const long long KD = (long long)K * D;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int per = (n + R - 1) / R;
    const int lo = min(n, r * per), hi = min(n, lo + per);

    extern __shared__ __align__(16) unsigned char smem_raw[];
    V2Smem s;
    {
        unsigned char* p = smem_raw;
        s.gbuf = reinterpret_cast<double*>(p); p += KM_THREADS * 4 * 8;
        s.lscr = reinterpret_cast<long long*>(p); p += 32 * 8;
        s.iscratch = reinterpret_cast<int*>(p); p += 64 * 4;
        s.dscratch = reinterpret_cast<double*>(p); p += 64 * 8;
        s.cnt_loc = reinterpret_cast<uint32_t*>(p); p += K * 4;
        s.cnt_all = reinterpret_cast<uint32_t*>(p); p += K * 4;
        s.moff = reinterpret_cast<uint32_t*>(p); p += K * 4;
        s.run = reinterpret_cast<uint32_t*>(p); p += K * 4;
        s.wcnt = reinterpret_cast<uint32_t*>(p); p += KM_WARPS * K * 4;
        p = smem_raw + (p - smem_raw + 15) / 16 * 16;
        s.cenf = reinterpret_cast<float*>(p); p += KD * 4;
        s.cnorm = reinterpret_cast<float*>(p); p += K * 4;
        p = smem_raw + (p - smem_raw + 15) / 16 * 16;
        s.cen64 = reinterpret_cast<double*>(p); p += KD * 8;
        s.dseed2 = reinterpret_cast<double*>(p); p += K * 8;
        s.delta = reinterpret_cast<float*>(p); p += K * 4;
        s.ncf = reinterpret_cast<float*>(p); p += K * 4;
        p = smem_raw + (p - smem_raw + 15) / 16 * 16;
        s.cenfg = reinterpret_cast<float*>(p); p += KD * 4;
        s.cnormg = reinterpret_cast<float*>(p); p += K * 4;
        s.grp = reinterpret_cast<int*>(p); p += K * 4;
        s.gorder = reinterpret_cast<int*>(p); p += K * 4;
        s.lrun = reinterpret_cast<uint32_t*>(p);
    }
    const bool yy = a.glb != nullptr;  // group bounds active for this launch
    __shared__ int g_start[KG + 1];
    __shared__ float g_delta[KG];
    bool groups_ready = false;
    uint32_t* lmem = yy ? a.lmem + (long long)q * n : nullptr;
    float* glbp = yy ? a.glb + (long long)q * n * KG : nullptr;
    bool lists_ready = false;  // lmem holds this CTA's points in assigned-centroid order
    uint32_t* asg = a.asg0 + (long long)q * n;
    uint32_t* nxt = a.asg1 + (long long)q * n;
    double* aux0 = a.aux0 + (long long)q * n;
    double* aux1 = a.aux1 + (long long)q * n;
    uint32_t* queue = a.queue + (long long)q * n;
    uint32_t* mem = members_g + (long long)q * n;
    uint16_t* nears = a.nearseed + (long long)q * n;
    float* ubd = a.ubound + (long long)q * n;
    float* lbd = a.lbound + (long long)q * n;
    __shared__ float sh_dmax1, sh_dmax2;
    __shared__ int sh_dargmax;
    bool bounds_valid = false;
    double* gcen = a.cen64 + q * KD;
    __shared__ int sh_int[8];
    __shared__ float sh_cmax;
    __shared__ int sh_flag;
    unsigned long long t_acc[6] = {0, 0, 0, 0, 0, 0};
    unsigned long long t_last = clock64();
    auto tick = [&](int ph) {
        if (tid == 0) {
            unsigned long long now = clock64();
            t_acc[ph] += now - t_last;
            t_last = now;
        }
    };
    auto cluster_or = [&](int v) -> int {
        int mine = __syncthreads_or(v);
        if (tid == 0) sh_flag = mine;
        cl.sync();
        int any = 0;
        for (int rr = 0; rr < R; ++rr) any |= *cl.map_shared_rank(&sh_flag, rr);
        cl.sync();  // sh_flag may be rewritten after this
        return any;
    };
    auto refresh_f32 = [&]() {
        for (long long e = tid; e < KD; e += KM_THREADS) s.cenf[e] = (float)s.cen64[e];
        if (tid == 0) sh_cmax = 0.f;
        __syncthreads();
        for (int c = tid; c < K; c += KM_THREADS) {
            float acc = 0.f;
            for (int t = 0; t < D; ++t) acc = fmaf(s.cenf[c * D + t], s.cenf[c * D + t], acc);
            float nrm = sqrtf(acc) * (1.0f + 9.6e-7f) + 1e-30f;
            s.cnorm[c] = nrm;
            s.ncf[c] = acc;
            atomicMax(reinterpret_cast<int*>(&sh_cmax), __float_as_int(nrm));
        }
        __syncthreads();
        if (groups_ready) {  // group-ordered copy for the Yinyang assign
            for (long long e = tid; e < KD; e += KM_THREADS) {
                const int pos = (int)(e / D), t = (int)(e % D);
                s.cenfg[e] = s.cenf[(long long)s.gorder[pos] * D + t];
            }
            for (int pos = tid; pos < K; pos += KM_THREADS) s.cnormg[pos] = s.cnorm[s.gorder[pos]];
            __syncthreads();
        }
    };
    // Centroid groups (Yinyang): KG Lloyd steps over the K centroids from the
    // first KG seeds (k-means++ spreads them); deterministic, CTA-local.
    auto form_groups = [&]() {
        __shared__ float gctr[KG][D];
        __shared__ int gcnt[KG];
        for (int e = tid; e < KG * D; e += KM_THREADS) gctr[e / D][e % D] = s.cenf[(e / D) * D + e % D];
        __syncthreads();
        for (int it = 0; it < 4; ++it) {
            for (int c = tid; c < K; c += KM_THREADS) {
                float best = FLT_MAX;
                int bg = 0;
                for (int g = 0; g < KG; ++g) {
                    float acc = 0.f;
                    for (int t = 0; t < D; ++t) {
                        const float d = s.cenf[c * D + t] - gctr[g][t];
                        acc = fmaf(d, d, acc);
                    }
                    if (acc < best) { best = acc; bg = g; }
                }
                s.grp[c] = bg;
            }
            __syncthreads();
            if (it == 3) break;
            for (int e = tid; e < KG * D; e += KM_THREADS) {
                const int g = e / D, t = e % D;
                float sum = 0.f;
                int cnt = 0;
                for (int c = 0; c < K; ++c)
                    if (s.grp[c] == g) { sum += s.cenf[c * D + t]; ++cnt; }
                if (cnt) gctr[g][t] = sum / (float)cnt;
            }
            __syncthreads();
        }
        if (tid == 0) {  // stable group order
            for (int g = 0; g < KG; ++g) gcnt[g] = 0;
            for (int c = 0; c < K; ++c) ++gcnt[s.grp[c]];
            int run = 0;
            for (int g = 0; g < KG; ++g) { g_start[g] = run; run += gcnt[g]; gcnt[g] = g_start[g]; }
            g_start[KG] = run;
            for (int c = 0; c < K; ++c) s.gorder[gcnt[s.grp[c]]++] = c;
        }
        __syncthreads();
        groups_ready = true;
    };
    auto merge_counts = [&]() {
        cl.sync();
        for (int c = tid; c < K; c += KM_THREADS) {
            uint32_t t = 0;
            for (int rr = 0; rr < R; ++rr) t += cl.map_shared_rank(s.cnt_loc, rr)[c];
            s.cnt_all[c] = t;
        }
        __syncthreads();
    };

    // ---- assignment pass over this CTA's slice (+ cluster-wide repair) ----
    // Hamerly bounds (certified): a point whose moved upper bound stays below
    // its moved lower bound keeps its centroid -- it is provably the unique
    // nearest in exact arithmetic and the fp64 margins exceed rounding -- so
    // neither its row nor any distance is touched.
    auto assign_pass = [&](uint32_t* out, const uint32_t* prev) {
        for (int c = tid; c < K; c += KM_THREADS) s.cnt_loc[c] = 0;
        if (tid == 0) { sh_int[0] = 0; sh_int[4] = 0; }
        __syncthreads();
        const float cmax = sh_cmax;
        const float dm1 = sh_dmax1, dm2 = sh_dmax2;
        const int dma = sh_dargmax;
        if (groups_ready) {
            // ---- Yinyang pass: points in assigned-centroid order (coherent warps) ----
            for (int j = lo + tid; j < hi; j += KM_THREADS) {
                const int i = lists_ready ? (int)lmem[j] : j;
                float* gl = glbp + (long long)i * KG;
                float lg[KG];
                float u = INFINITY;
                int ga = -1;
                if (bounds_valid) {
                    const uint32_t ap = prev[i];
                    ga = s.grp[ap];
                    u = __fadd_ru(ubd[i], s.delta[ap]);
                    const float4 l0 = reinterpret_cast<const float4*>(gl)[0], l1 = reinterpret_cast<const float4*>(gl)[1];
                    const float lv[KG] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
                    float lmin = INFINITY;
#pragma unroll
                    for (int g = 0; g < KG; ++g) {
                        lg[g] = __fsub_rd(lv[g], g_delta[g]);
                        lmin = fminf(lmin, lg[g]);
                    }
                    if (__fmul_ru(u, 1.000001f) < lmin) {  // keeps its centroid (Hamerly over groups)
                        out[i] = ap;
                        atomicAdd(&s.cnt_loc[ap], 1u);
                        ubd[i] = u;
                        reinterpret_cast<float4*>(gl)[0] = make_float4(lg[0], lg[1], lg[2], lg[3]);
                        reinterpret_cast<float4*>(gl)[1] = make_float4(lg[4], lg[5], lg[6], lg[7]);
                        atomicAdd(&sh_int[4], 1);
                        continue;
                    }
                } else {
#pragma unroll
                    for (int g = 0; g < KG; ++g) lg[g] = -INFINITY;
                }
                float x[D];
                load_point<D>(point_ptr(a, q, i), x, a.vec4);
                const float uu = __fmul_ru(u, 1.000001f);
                float b1 = FLT_MAX, e1 = 0.f;
                int i1 = -1;
                float low1[KG], low2[KG];
                int idx1[KG];
                unsigned evald = 0;
#pragma unroll
                for (int g = 0; g < KG; ++g) {
                    low1[g] = INFINITY;
                    low2[g] = INFINITY;
                    idx1[g] = -1;
                    if (!(lg[g] <= uu) && g != ga) continue;  // every centroid of g is provably farther
                    evald |= 1u << g;
                    for (int pos = g_start[g]; pos < g_start[g + 1]; ++pos) {
                        const float v = dist_f<D>(x, s.cenfg + (long long)pos * D);
                        const float e = err_bound(v, s.cnormg[pos], D);
                        const int c = s.gorder[pos];
                        if (v < b1) { b1 = v; e1 = e; i1 = c; }
                        const float lo_v = v - e;
                        if (lo_v < low1[g]) { low2[g] = low1[g]; low1[g] = lo_v; idx1[g] = c; }
                        else if (lo_v < low2[g]) low2[g] = lo_v;
                    }
                }
                // certified iff every other centroid's lower bound exceeds the
                // best's upper bound (evaluated ones: their own error bounds;
                // skipped groups: the group bound)
                bool ok = i1 >= 0 && b1 < 1e37f;
                const float hi1 = b1 + e1;
#pragma unroll
                for (int g = 0; g < KG; ++g) {
                    if ((evald >> g) & 1u) {
                        const float ex = idx1[g] == i1 ? low2[g] : low1[g];
                        ok = ok && ex > hi1;
                    } else {
                        ok = ok && __fmul_rd(__fmul_rd(lg[g], lg[g]), 0.999999f) > hi1;
                    }
                }
                if (ok) {
                    out[i] = (uint32_t)i1;
                    atomicAdd(&s.cnt_loc[i1], 1u);
                    ubd[i] = __fsqrt_ru(__fmul_ru(__fadd_ru(b1, e1), 1.000001f));
                    float nl[KG];
#pragma unroll
                    for (int g = 0; g < KG; ++g) {
                        if ((evald >> g) & 1u) {
                            const float ex = idx1[g] == i1 ? low2[g] : low1[g];
                            nl[g] = ex >= INFINITY ? INFINITY : __fsqrt_rd(fmaxf(0.f, __fmul_rd(ex, 0.999999f)));
                        } else {
                            nl[g] = lg[g];
                        }
                    }
                    reinterpret_cast<float4*>(gl)[0] = make_float4(nl[0], nl[1], nl[2], nl[3]);
                    reinterpret_cast<float4*>(gl)[1] = make_float4(nl[4], nl[5], nl[6], nl[7]);
                } else {
                    queue[lo + atomicAdd(&sh_int[0], 1)] = (uint32_t)i;
                    ubd[i] = INFINITY;  // re-scan next pass
                    reinterpret_cast<float4*>(gl)[0] = make_float4(0.f, 0.f, 0.f, 0.f);
                    reinterpret_cast<float4*>(gl)[1] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
        } else
        for (int i = lo + tid; i < hi; i += KM_THREADS) {
            if (bounds_valid) {
                const uint32_t ap = prev[i];
                const float u = __fadd_ru(ubd[i], s.delta[ap]);
                const float l = __fsub_rd(lbd[i], (int)ap == dma ? dm2 : dm1);
                if (__fmul_ru(u, 1.000001f) < l) {
                    out[i] = ap;
                    atomicAdd(&s.cnt_loc[ap], 1u);
                    ubd[i] = u;
                    lbd[i] = l;
                    atomicAdd(&sh_int[4], 1);
                    continue;
                }
            }
            float x[D];
            load_point<D>(point_ptr(a, q, i), x, a.vec4);
            float ub, lb;
            // direct form: its bound scales with the distance itself; the
            // expanded form's (|x|^2 + |c|^2 - 2 x.c) scales with (|x| + |c|)^2,
            // which re-checked most points of the powerlaw keys
            int c = nearest_filtered_b<D>(x, s.cenf, s.cnorm, cmax, K, ub, lb);
            if (c >= 0) {
                out[i] = (uint32_t)c;
                atomicAdd(&s.cnt_loc[c], 1u);
                ubd[i] = ub;
                lbd[i] = lb;
            } else {
                queue[lo + atomicAdd(&sh_int[0], 1)] = (uint32_t)i;
            }
        }
        __syncthreads();
        const int qn = sh_int[0];
        for (int e = tid; e < qn; e += KM_THREADS) {
            const int i = (int)queue[lo + e];
            const uint32_t c = nearest_g(point_ptr(a, q, i), s.cen64, K, D);
            out[i] = c;
            atomicAdd(&s.cnt_loc[c], 1u);
            ubd[i] = INFINITY;  // re-scan next pass
            lbd[i] = 0.f;
        }
        if (tid == 0 && a.stats) {
            atomicAdd(&a.stats[0], (unsigned long long)qn);
            atomicAdd(&a.stats[1], (unsigned long long)(hi - lo));
            atomicAdd(&a.stats[2], (unsigned long long)sh_int[4]);
        }
        merge_counts();
        if (n < K) return;
        int empty = 0;
        for (int c = tid; c < K; c += KM_THREADS) empty |= (s.cnt_all[c] == 0);
        if (!__syncthreads_or(empty)) return;  // uniform: cnt_all is identical in every CTA
        // rare path (kmeans.cpp:111-127): rank 0 repairs over all points
        if (r == 0) {
            for (int i = tid; i < n; i += KM_THREADS)
                aux0[i] = dist2_g(point_ptr(a, q, i), s.cen64 + (long long)out[i] * D, D);
            __syncthreads();
            for (int c = 0; c < K; ++c) {
                if (s.cnt_all[c] != 0) continue;
                double best = -1.0;
                int bi = n;
                for (int i = tid; i < n; i += KM_THREADS) {
                    if (s.cnt_all[out[i]] < 2) continue;
                    double d = aux0[i];
                    if (d > best) { best = d; bi = i; }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    double ob = __shfl_xor_sync(FULL, best, o);
                    int oi = __shfl_xor_sync(FULL, bi, o);
                    if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
                }
                if (lane == 0) { s.dscratch[warp] = best; s.iscratch[warp] = bi; }
                __syncthreads();
                if (tid == 0) {
                    double b = s.dscratch[0];
                    int ii = s.iscratch[0];
                    for (int w = 1; w < KM_WARPS; ++w) {
                        double ob = s.dscratch[w];
                        int oi = s.iscratch[w];
                        if (ob > b || (ob == b && oi < ii)) { b = ob; ii = oi; }
                    }
                    sh_int[1] = ii;
                }
                __syncthreads();
                const int donor = sh_int[1];
                if (donor >= n) break;
                if (tid == 0) {
                    s.cnt_all[out[donor]] -= 1;
                    out[donor] = (uint32_t)c;
                    s.cnt_all[c] += 1;
                    ubd[donor] = INFINITY;  // not at its nearest centroid any more
                    lbd[donor] = 0.f;
                }
                __syncthreads();
            }
        }
        cl.sync();  // repaired assignment visible
        for (int c = tid; c < K; c += KM_THREADS) s.cnt_loc[c] = 0;
        __syncthreads();
        for (int i = lo + tid; i < hi; i += KM_THREADS) atomicAdd(&s.cnt_loc[out[i]], 1u);
        merge_counts();
    };

    // ---- update_means: member lists + certified order-free sums ----
    auto update_means = [&](const uint32_t* as) {
        // offsets: members of cluster c in point order, slices in rank order
        if (tid == 0) {
            uint32_t run = 0, lrun = (uint32_t)lo;
            for (int c = 0; c < K; ++c) {
                s.moff[c] = run;
                run += s.cnt_all[c];
                s.lrun[c] = lrun;  // this CTA's own list (Yinyang pass order)
                lrun += s.cnt_loc[c];
            }
        }
        __syncthreads();
        for (int c = tid; c < K; c += KM_THREADS) {
            uint32_t before = 0;
            for (int rr = 0; rr < r; ++rr) before += cl.map_shared_rank(s.cnt_loc, rr)[c];
            s.run[c] = s.moff[c] + before;
        }
        for (int e = tid; e < KM_WARPS * K; e += KM_THREADS) s.wcnt[e] = 0;
        __syncthreads();
        // stable scatter of this slice
        for (int b0 = lo; b0 < hi; b0 += KM_THREADS) {
            const int i = b0 + tid;
            const uint32_t c = i < hi ? as[i] : 0xffffffffu;
            const unsigned peers = __match_any_sync(FULL, c);
            const uint32_t wr = __popc(peers & lanemask_lt());
            if (c != 0xffffffffu && wr == 0) s.wcnt[warp * K + c] = __popc(peers);
            __syncthreads();
            if (c != 0xffffffffu) {
                uint32_t before = 0;
                for (int w = 0; w < warp; ++w) before += s.wcnt[w * K + c];
                mem[s.run[c] + before + wr] = (uint32_t)i;
                if (yy) lmem[s.lrun[c] + before + wr] = (uint32_t)i;
            }
            __syncthreads();
            for (int cc = tid; cc < K; cc += KM_THREADS) {
                uint32_t tot = 0;
                for (int w = 0; w < KM_WARPS; ++w) { tot += s.wcnt[w * K + cc]; s.wcnt[w * K + cc] = 0; }
                s.run[cc] += tot;
                s.lrun[cc] += tot;
            }
            __syncthreads();
        }
        cl.sync();  // every slice's member list is written
        tick(3);
        // sums: warp gw of the cluster owns clusters c = gw (mod KM_WARPS*R)
        constexpr int DG = 32 / V2_MG;                       // lanes per member group (8)
        constexpr int DPL = (D + DG - 1) / DG;               // dims per lane
        const int mg = lane / DG, dl = lane % DG;            // member group, lane in group
        const int gw = r * KM_WARPS + warp;
        for (int c = gw; c < K; c += KM_WARPS * R) {
            const uint32_t cnt = s.cnt_all[c];
            if (cnt == 0) continue;  // empty cluster keeps its centroid
            const uint32_t base = s.moff[c];
            double acc[DPL], aabs[DPL];
            int emin[DPL];
#pragma unroll
            for (int e = 0; e < DPL; ++e) { acc[e] = 0.0; aabs[e] = 0.0; emin[e] = 0x7fffffff; }
            // members mg, mg+4, ... ; 4 member rows per warp step, unrolled x4;
            // the next step's member indices are loaded one step ahead
            uint32_t idn[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t m = u * V2_MG + mg;
                idn[u] = m < cnt ? mem[base + m] : 0xffffffffu;
            }
            for (uint32_t m0 = 0; m0 < cnt; m0 += V2_MG * 4) {
                float xv[4][DPL];
                uint32_t idc[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    idc[u] = idn[u];
                    const uint32_t m = m0 + V2_MG * 4 + u * V2_MG + mg;
                    idn[u] = m < cnt ? mem[base + m] : 0xffffffffu;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float* xp = idc[u] != 0xffffffffu ? point_ptr(a, q, (int)idc[u]) : nullptr;
#pragma unroll
                    for (int e = 0; e < DPL; ++e) {
                        const int t = dl + DG * e;
                        xv[u][e] = (xp && t < D) ? __ldg(xp + t) : 0.0f;
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int e = 0; e < DPL; ++e) {
                        const float x = xv[u][e];
                        acc[e] += (double)x;
                        aabs[e] += (double)fabsf(x);
                        if (x != 0.0f) emin[e] = min(emin[e], (int)((__float_as_uint(x) >> 23) & 0xff));
                    }
            }
            // combine the member groups (lanes dl, dl+8, dl+16, dl+24)
#pragma unroll
            for (int e = 0; e < DPL; ++e)
#pragma unroll
                for (int o = DG; o < 32; o <<= 1) {
                    acc[e] += __shfl_xor_sync(FULL, acc[e], o);
                    aabs[e] += __shfl_xor_sync(FULL, aabs[e], o);
                    emin[e] = min(emin[e], __shfl_xor_sync(FULL, emin[e], o));
                }
            // certificate per dim: sum|x| < 2^52 * ulp_min (ulp of the smallest-exponent
            // member: 2^(e-150) for normal e, 2^-149 for subnormals)
            unsigned badm = 0;  // failing dims of this lane, bit e
#pragma unroll
            for (int e = 0; e < DPL; ++e) {
                if (dl + DG * e >= D || emin[e] == 0x7fffffff) continue;
                const int ue = emin[e] == 0 ? -149 : emin[e] - 150;
                if (!(aabs[e] * (1.0 + 1e-9) < ldexp(1.0, 52 + ue))) badm |= 1u << e;
            }
            if (mg == 0) {
#pragma unroll
                for (int e = 0; e < DPL; ++e) {
                    const int t = dl + DG * e;
                    if (t < D && !((badm >> e) & 1u)) gcen[(long long)c * D + t] = __ddiv_rn(acc[e], (double)cnt);
                }
            }
            // exact fallback for failing dims: the reference's order (points
            // ascending), 32 members per step -- indices and values fetched in
            // parallel, then folded serially through the warp
            unsigned any = __ballot_sync(FULL, mg == 0 && badm != 0);
            while (any) {
                const int src = __ffs(any) - 1;
                const unsigned bm = __shfl_sync(FULL, badm, src);
                const int e = __ffs(bm) - 1;
                const int t = (src % DG) + DG * e;
                double sacc = 0.0;
                for (uint32_t m0 = 0; m0 < cnt; m0 += 32) {
                    const uint32_t m = m0 + lane;
                    const float xv = m < cnt ? __ldg(point_ptr(a, q, (int)mem[base + m]) + t) : 0.0f;
                    const int nb = (int)min(32u, cnt - m0);
                    for (int l = 0; l < nb; ++l) sacc = __dadd_rn(sacc, (double)__shfl_sync(FULL, xv, l));
                }
                if (lane == 0) gcen[(long long)c * D + t] = __ddiv_rn(sacc, (double)cnt);
                // clear (src, e) and continue with the next failing dim
                if (lane == src) badm &= ~(1u << e);
                any = __ballot_sync(FULL, mg == 0 && badm != 0);
            }
        }
        cl.sync();  // new means visible in global memory
        // centroid movement (Hamerly): delta_c >= |mu_c(new) - mu_c(old)|
        for (int c = tid; c < K; c += KM_THREADS) {
            double dd = 0.0;
            for (int t = 0; t < D; ++t) {
                const double df = gcen[(long long)c * D + t] - s.cen64[(long long)c * D + t];
                dd = fma(df, df, dd);
            }
            s.delta[c] = __double2float_ru(__dsqrt_ru(dd * (1.0 + 1e-12)));
        }
        __syncthreads();
        if (warp == 0) {  // largest and second largest movement
            float m1 = 0.f, m2 = 0.f;
            int i1 = -1;
            for (int c = lane; c < K; c += 32) {
                const float v = s.delta[c];
                if (v > m1) { m2 = m1; m1 = v; i1 = c; }
                else if (v > m2) m2 = v;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float om1 = __shfl_xor_sync(FULL, m1, o), om2 = __shfl_xor_sync(FULL, m2, o);
                const int oi = __shfl_xor_sync(FULL, i1, o);
                if (om1 > m1) { m2 = fmaxf(m1, om2); m1 = om1; i1 = oi; }
                else m2 = fmaxf(m2, om1);
            }
            if (lane == 0) { sh_dmax1 = m1; sh_dmax2 = m2; sh_dargmax = i1; }
        }
        if (groups_ready && tid < KG) {  // largest drift per group (already rounded up)
            float mx = 0.f;
            for (int pos = g_start[tid]; pos < g_start[tid + 1]; ++pos) mx = fmaxf(mx, s.delta[s.gorder[pos]]);
            g_delta[tid] = mx;
        }
        if (yy) lists_ready = true;
        for (long long e = tid; e < KD; e += KM_THREADS) s.cen64[e] = gcen[e];
        __syncthreads();
    };

    // =====================================================================
    // 1. seeding
    // =====================================================================
    const unsigned long long* draws = a.draws + (long long)q * K;
    if (n <= K) {
        if (r == 0) {  // seed_from_distinct (kmeans.cpp:44-57), small
            for (int i = tid; i < n; i += KM_THREADS) {
                const uint32_t* xi = reinterpret_cast<const uint32_t*>(point_ptr(a, q, i));
                int seen = 0;
                for (int j = 0; j < i && !seen; ++j) {
                    const uint32_t* xj = reinterpret_cast<const uint32_t*>(point_ptr(a, q, j));
                    int eq = 1;
                    for (int t = 0; t < D && eq; ++t) eq = (xi[t] == xj[t]);
                    seen = eq;
                }
                asg[i] = seen ? 0u : 1u;
            }
            __syncthreads();
            if (tid == 0) {
                int nd = 0;
                for (int i = 0; i < n; ++i)
                    if (asg[i]) nxt[nd++] = (uint32_t)i;
                sh_int[2] = nd;
            }
            __syncthreads();
            const int nd = sh_int[2];
            for (long long e = tid; e < KD; e += KM_THREADS) {
                const int c = (int)(e / D), t = (int)(e % D);
                const int src = (int)nxt[c < nd - 1 ? c : nd - 1];
                gcen[e] = (double)point_ptr(a, q, src)[t];
            }
        }
        cl.sync();
        for (long long e = tid; e < KD; e += KM_THREADS) s.cen64[e] = gcen[e];
        __syncthreads();
    } else {
        const int c0 = (int)(draws[0] % (unsigned long long)n);
        for (int t = tid; t < D; t += KM_THREADS) s.cen64[t] = (double)point_ptr(a, q, c0)[t];
        __syncthreads();
        for (int i = lo + tid; i < hi; i += KM_THREADS) {
            aux0[i] = dist2_g(point_ptr(a, q, i), s.cen64, D);
            nears[i] = 0;
        }
        if (tid == 0) sh_int[5] = 0;
        for (int c = 1; c < K; ++c) {
            cl.sync();  // every slice's min_d2 is final for this step
            tick(1);
            // k-means++ running sums (kmeans.cpp:64-65, 70-71), split over the
            // cluster: rank 0 runs the serial-exact sum over its slice while
            // every other rank turns its slice into an integer prefix in the
            // binade its entry value must lie in (slice_increments); the
            // entries are then chained exactly, slices that cannot be
            // certified are summed serially from their exact entry.
            double total;
            if (R == 1) {
                total = exact_running_sum(aux0, n, aux1, s.gbuf, s.lscr, s.dscratch);
                __syncthreads();  // aux1 (prefix) visible to warp 0's search
            } else {
                __shared__ double rs_pub[4];  // [0] approx slice sum, [1] u, [2] exit S (rank 0)
                __shared__ long long rs_iend;
                __shared__ int rs_ok;
                {
                    double part = 0.0;
                    for (int i = lo + tid; i < hi; i += KM_THREADS) part += aux0[i];
                    part = warp_sum(part);
                    if (lane == 0) s.dscratch[warp] = part;
                    __syncthreads();
                    if (tid == 0) {
                        double t = 0.0;
                        for (int w = 0; w < KM_WARPS; ++w) t += s.dscratch[w];
                        rs_pub[0] = t;
                    }
                }
                cl.sync();  // approximate slice sums published
                double P = 0.0;
                for (int rr = 0; rr < r; ++rr) P += *cl.map_shared_rank(&rs_pub[0], rr);
                if (r == 0) {
                    const double ex = exact_running_sum(aux0, hi, aux1, s.gbuf, s.lscr, s.dscratch);
                    if (tid == 0) rs_pub[2] = ex;
                } else {
                    double u;
                    long long iend;
                    const bool ok = slice_increments(aux0 + lo, hi - lo, P, aux1 + lo, s.lscr, &u, &iend);
                    if (tid == 0) { rs_ok = ok ? 1 : 0; rs_pub[1] = u; rs_iend = iend; }
                }
                cl.sync();  // rank 0's exit and the speculative slices are ready
                // chain the exact entries in rank order (identical in every CTA)
                double S = *cl.map_shared_rank(&rs_pub[2], 0);
                double my_entry = 0.0;
                bool my_serial = false;
                for (int rr = 1; rr < R; ++rr) {
                    const int okr = *cl.map_shared_rank(&rs_ok, rr);
                    const double ur = *cl.map_shared_rank(&rs_pub[1], rr);
                    const long long ir = *cl.map_shared_rank(&rs_iend, rr);
                    const int lor = min(n, rr * per), hir = min(n, lor + per);
                    const double lo_edge = __longlong_as_double(__double_as_longlong(ur) + (52ll << 52));
                    const bool fits = okr && S >= lo_edge && S + (double)ir * ur < 2.0 * lo_edge;
                    if (rr == r) { my_entry = S; my_serial = !fits; }
                    if (fits) {
                        S = S + (double)ir * ur;
                    } else {  // rare: rank rr sums its slice serially from the exact entry
                        if (rr == r) {
                            const double ex = exact_running_sum(aux0 + lor, hir - lor, aux1 + lor, s.gbuf, s.lscr,
                                                                s.dscratch, S);
                            if (tid == 0) rs_pub[2] = ex;
                        }
                        cl.sync();
                        S = *cl.map_shared_rank(&rs_pub[2], rr);
                    }
                }
                total = S;
                if (r > 0 && !my_serial) {  // integer prefix -> exact running sums
                    const double ur = rs_pub[1];
                    for (int i = lo + tid; i < hi; i += KM_THREADS) aux1[i] = my_entry + aux1[i] * ur;
                }
                cl.sync();  // every slice's running sums are written
            }
            if (r == 0) {
                if (warp == 0) {
                    int chosen;
                    if (total > 0.0) {
                        const double u = (double)(draws[c] >> 11) * 0x1.0p-53;
                        chosen = warp_lower_bound(aux1, n, __dmul_rn(u, total));
                    } else {
                        chosen = (int)(draws[c] % (unsigned long long)n);
                    }
                    if (lane == 0) sh_int[3] = chosen;
                }
            }
            cl.sync();
            const int chosen = *cl.map_shared_rank(&sh_int[3], 0);
            tick(0);
            for (int t = tid; t < D; t += KM_THREADS)
                s.cen64[(long long)c * D + t] = (double)point_ptr(a, q, chosen)[t];
            __syncthreads();
            const double* cc = s.cen64 + (long long)c * D;
            // triangle inequality: d(x, mu_c) >= d(mu_j, mu_c) - d(x, mu_j) with j the
            // seed behind min_d2(x); if d(mu_j, mu_c)^2 >= 4 min_d2 (+ margin for
            // fp64 rounding) then min(min_d2, dist2(x, mu_c)) == min_d2: skip x.
            for (int j = tid; j < c; j += KM_THREADS) {
                double acc = 0.0;
                for (int t = 0; t < D; ++t) {
                    const double df = s.cen64[(long long)j * D + t] - cc[t];
                    acc = fma(df, df, acc);
                }
                s.dseed2[j] = acc * (1.0 - 1e-12);
            }
            float cf[D];
            float cn = 0.f;
#pragma unroll
            for (int t = 0; t < D; ++t) { cf[t] = (float)cc[t]; cn = fmaf(cf[t], cf[t], cn); }
            cn = sqrtf(cn) * (1.0f + 9.6e-7f) + 1e-30f;
            __syncthreads();
            int nskip = 0;
            for (int i0 = lo + tid; i0 < hi; i0 += 4 * KM_THREADS) {
              double mdv[4];
              uint16_t nrv[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                  const int i = i0 + u * KM_THREADS;
                  mdv[u] = i < hi ? aux0[i] : 0.0;
                  nrv[u] = i < hi ? nears[i] : (uint16_t)0;
              }
#pragma unroll 1
              for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * KM_THREADS;
                if (i >= hi) break;
                const double md = mdv[u];
                if (s.dseed2[nrv[u]] >= 4.0 * md * (1.0 + 1e-7) + 1e-300) {
                    ++nskip;
                    continue;
                }
                const float* xp = point_ptr(a, q, i);
                float xr[D];
                load_point<D>(xp, xr, a.vec4);
                float acc = 0.f;
#pragma unroll
                for (int t = 0; t < D; ++t) {
                    const float d = xr[t] - cf[t];
                    acc = fmaf(d, d, acc);
                }
                const double old = md;
                if (acc < 1e37f && (double)(acc - err_bound(acc, cn, D)) > old) continue;
                // dist2 (kmeans.cpp:14-21) from the row already in registers:
                // fp64, separate sub / mul / add, ascending t
                double d = 0.0;
#pragma unroll
                for (int t = 0; t < D; ++t) {
                    const double df = __dsub_rn((double)xr[t], cc[t]);
                    d = __dadd_rn(d, __dmul_rn(df, df));
                }
                if (d < old) {
                    aux0[i] = d;
                    nears[i] = (uint16_t)c;
                }
              }
            }
            if (nskip) atomicAdd(&sh_int[5], nskip);
        }
        cl.sync();
        tick(1);
        if (tid == 0 && a.stats) atomicAdd(&a.stats[3], (unsigned long long)sh_int[5]);
        if (r == 0)
            for (long long e = tid; e < KD; e += KM_THREADS) gcen[e] = s.cen64[e];
        // (no sync needed: gcen is read after the next cluster barrier)
    }
    refresh_f32();
    tick(5);

    // =====================================================================
    // 2. Lloyd iterations (kmeans.cpp:174-183)
    // =====================================================================
    if (yy) {
        form_groups();
        refresh_f32();
    }
    assign_pass(asg, nullptr);
    bounds_valid = true;
    tick(2);
    int iters = 0;
    for (int iter = 1; iter <= T; ++iter) {
        update_means(asg);
        tick(4);
        if (a.inertia) {
            for (int i = lo + tid; i < hi; i += KM_THREADS)
                aux0[i] = dist2_g(point_ptr(a, q, i), s.cen64 + (long long)asg[i] * D, D);
            cl.sync();
            if (r == 0 && warp == 0) {
                double tot = warp_serial_sum(aux0, n, nullptr);
                if (lane == 0) a.inertia[(long long)q * T + iter - 1] = tot;
            }
            cl.sync();
        }
        iters = iter;
        refresh_f32();
        tick(5);
        assign_pass(nxt, asg);
        tick(2);
        int changed = 0;
        for (int i = lo + tid; i < hi; i += KM_THREADS) changed |= (nxt[i] != asg[i]);
        if (!cluster_or(changed)) break;
        uint32_t* t = asg;
        asg = nxt;
        nxt = t;
    }

    // =====================================================================
    // 3. emit
    // =====================================================================
    if (r == 0)
        for (long long e = tid; e < KD; e += KM_THREADS) a.centroids_out[q * KD + e] = (float)s.cen64[e];
    if (a.assign_out)
        for (int i = lo + tid; i < hi; i += KM_THREADS) a.assign_out[(long long)q * n + i] = asg[i];
    if (a.codes) {
        const int head = q / a.m_sub, j = q % a.m_sub;
        uint16_t* cd = a.codes + (long long)head * a.codes_head_stride + j;
        for (int i = lo + tid; i < hi; i += KM_THREADS) cd[(long long)i * a.m_sub] = (uint16_t)asg[i];
    }
    if (a.iterations && tid == 0 && r == 0) a.iterations[q] = (uint32_t)iters;
    tick(5);
    if (tid == 0 && r == 0 && a.timers)
        for (int ph = 0; ph < 6; ++ph) a.timers[(long long)q * 8 + ph] = t_acc[ph];
    cl.sync();  // keep smem alive for remote readers
}

template <int D>
void launch_cluster_v2(const KmArgs& a, uint32_t* members, int problems, int R, size_t smem, cudaStream_t st) {
    auto kern = kmeans_cluster_kernel<D>;
    PQKV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(problems * R));
    cfg.blockDim = dim3(KM_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)R;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (std::getenv("PQKV_DEBUG_CLUSTERS")) {
        int nc = -1;
        cudaOccupancyMaxActiveClusters(&nc, kern, &cfg);
        std::fprintf(stderr, "kmeans_cluster_kernel<%d>: %d problems x cluster %d, smem %zu -> max active clusters %d\n",
                     D, problems, R, smem, nc);
    }
    PQKV_CUDA(cudaLaunchKernelEx(&cfg, kern, a, members));
    PQKV_LAUNCHED("kmeans_cluster_kernel");
}

template <int D, bool F>
void launch_problem(const KmArgs& a, int problems, size_t smem, cudaStream_t st) {
    auto kern = kmeans_problem_kernel<D, F>;
    PQKV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<problems, KM_THREADS, smem, st>>>(a);
    PQKV_LAUNCHED("kmeans_problem_kernel");
}

}  // namespace

void launch_kmeans(pqkv_ctx* ctx, const KmeansBatch& b, cudaStream_t st) {
    const size_t Q = b.n_problems, n = b.n, dim = b.dim, K = b.k;
    if (Q == 0) return;
    if (n > 0x7fffffff || K > 0x7fffffff) fail(PQKV_EINVAL, "kmeans: problem too large");
    const bool exact = ctx->assign_mode == PQKV_ASSIGN_EXACT;
    // pick the compile-time dimension
    int D = 0;
    for (int d : {2, 4, 8, 16, 32, 64, 128})
        if ((size_t)d == dim) D = d;
    bool filter = !exact && D > 0;
    if (!filter && D > 64) D = 0;  // fp64 point registers would spill

    // shared-memory plan (same carve order as the kernel)
    const size_t KD = K * dim;
    const size_t budget = 200 * 1024;
    size_t smem = KM_THREADS * 4 * 8 + 32 * 8 + 64 * 4 + 64 * 8;
    int counts_smem = 0, sums_smem = 0, cen64_smem = 0, cenf_smem = 0;
    auto take = [&](size_t bytes, int& flag) {
        bytes = round_up(bytes, 16);
        if (smem + bytes <= budget) { smem += bytes; flag = 1; }
    };
    take(K * 4, counts_smem);
    if (filter) {
        // the filter needs the f32 table in smem; fp64 centroids may stay global
        size_t need = round_up(KD * 4, 16) + round_up(K * 4, 16);
        if (smem + need > budget) { filter = false; if (D > 64) D = 0; }
    }
    if (filter) {
        take(KD * 8, sums_smem);
        size_t need = round_up(KD * 4, 16) + round_up(K * 4, 16);
        smem += need;
        cenf_smem = 1;
        take(KD * 8, cen64_smem);
    } else {
        take(KD * 8, cen64_smem);
        take(KD * 8, sums_smem);
        if (D > 0 && !cen64_smem) D = 0;  // register path reads smem centroids
    }

    // v2 (cluster of R CTAs per problem) for the filtered path with smem tables
    const bool v2 = filter && D >= 8 && K <= 1024 && K <= 65536 && v2_smem_bytes((int)K, D) <= 200 * 1024 &&
                    std::getenv("PQKV_KMEANS_V1") == nullptr;
    int R = 1;
    if (v2) {
        // CTAs per SM: two for D <= 64 when both fit in shared memory
        const int occ = km_v2_occ(D) == 2 && 2 * (v2_smem_bytes((int)K, D) + 2048) <= 227 * 1024 ? 2 : 1;
        R = (int)std::max<size_t>(1, (size_t)ctx->sm_count * occ / Q);
        R = std::min(R, 8);
        R = (int)std::min<size_t>((size_t)R, std::max<size_t>(1, ceil_div(n, 4096)));
        while (R & (R - 1)) --R;  // power of two
    }

    Scratch sc(ctx);
    size_t h_mem = sc.plan<uint32_t>(v2 ? Q * n : 1);
    size_t h_near = sc.plan<uint16_t>(v2 ? Q * n : 1);
    size_t h_ub = sc.plan<float>(v2 ? Q * n : 1), h_lb = sc.plan<float>(v2 ? Q * n : 1);
    // group bounds (Yinyang) when there are enough centroids to group
    const bool yy = v2 && K >= 4 * (size_t)KG && std::getenv("PQKV_KMEANS_NOGROUPS") == nullptr;
    size_t h_glb = sc.plan<float>(yy ? Q * n * KG : 4), h_lmem = sc.plan<uint32_t>(yy ? Q * n : 1);
    size_t h_draws = sc.plan<unsigned long long>(Q * K);
    size_t h_a0 = sc.plan<uint32_t>(Q * n), h_a1 = sc.plan<uint32_t>(Q * n);
    size_t h_x0 = sc.plan<double>(Q * n), h_x1 = sc.plan<double>(Q * n);
    size_t h_cen = sc.plan<double>(Q * KD);
    size_t h_sums = sc.plan<double>(sums_smem ? 1 : Q * KD);
    size_t h_cnt = sc.plan<uint32_t>(counts_smem ? 1 : Q * K);
    size_t h_q = sc.plan<uint32_t>(Q * n);
    size_t h_tm = sc.plan<unsigned long long>(Q * 8);
    sc.commit();

    // mt19937_64 draws (rng.hpp:13-33): k-means++ consumes exactly K raw
    // draws per problem regardless of the data (kmeans.cpp:60, 68, 78).
    std::vector<unsigned long long> draws(Q * K, 0ull);
    for (size_t q = 0; q < Q; ++q) {
        if (n <= K) continue;
        std::mt19937_64 eng(b.seeds[q]);
        for (size_t c = 0; c < K; ++c) draws[q * K + c] = eng();
    }
    PQKV_CUDA(cudaMemcpyAsync(sc.get<unsigned long long>(h_draws), draws.data(),
                              draws.size() * 8, cudaMemcpyHostToDevice, st));
    PQKV_CUDA(cudaMemsetAsync(ctx->d_stats, 0, 4 * sizeof(unsigned long long), st));

    KmArgs a{};
    a.points = b.points;
    a.problem_stride = (long long)b.problem_stride;
    a.row_stride = (long long)b.row_stride;
    a.m_sub = (int)b.m_sub;
    a.n = (int)n;
    a.dim = (int)dim;
    a.K = (int)K;
    a.T = (int)b.max_iter;
    a.draws = sc.get<unsigned long long>(h_draws);
    a.centroids_out = b.centroids;
    a.assign_out = b.assign;
    a.codes = b.codes;
    a.codes_head_stride = (long long)b.codes_head_stride;
    a.iterations = b.iterations;
    a.inertia = b.inertia;
    a.asg0 = sc.get<uint32_t>(h_a0);
    a.asg1 = sc.get<uint32_t>(h_a1);
    a.aux0 = sc.get<double>(h_x0);
    a.aux1 = sc.get<double>(h_x1);
    a.cen64 = sc.get<double>(h_cen);
    a.gsums = sc.get<double>(h_sums);
    a.gcounts = sc.get<uint32_t>(h_cnt);
    a.queue = sc.get<uint32_t>(h_q);
    a.stats = ctx->d_stats;
    a.timers = sc.get<unsigned long long>(h_tm);
    a.nearseed = sc.get<uint16_t>(h_near);
    a.ubound = sc.get<float>(h_ub);
    a.lbound = sc.get<float>(h_lb);
    a.glb = yy ? sc.get<float>(h_glb) : nullptr;
    a.lmem = yy ? sc.get<uint32_t>(h_lmem) : nullptr;
    a.counts_smem = counts_smem;
    a.sums_smem = sums_smem;
    a.cen64_smem = cen64_smem;
    a.cenf_smem = cenf_smem;
    a.vec4 = ((reinterpret_cast<uintptr_t>(b.points) & 15) == 0) && (b.row_stride % 4 == 0) &&
             (b.problem_stride % 4 == 0) && (dim % 4 == 0);

    bind_device(ctx);
    int P = (int)Q;
    if (v2) {
        const size_t smem2 = v2_smem_bytes((int)K, D);
        uint32_t* members = sc.get<uint32_t>(h_mem);
        switch (D) {
            case 8: launch_cluster_v2<8>(a, members, P, R, smem2, st); break;
            case 16: launch_cluster_v2<16>(a, members, P, R, smem2, st); break;
            case 32: launch_cluster_v2<32>(a, members, P, R, smem2, st); break;
            case 64: launch_cluster_v2<64>(a, members, P, R, smem2, st); break;
            case 128: launch_cluster_v2<128>(a, members, P, R, smem2, st); break;
            default: fail(PQKV_ERUNTIME, "kmeans: bad v2 dim");
        }
    } else if (filter) {
        switch (D) {
            case 2: launch_problem<2, true>(a, P, smem, st); break;
            case 4: launch_problem<4, true>(a, P, smem, st); break;
            case 8: launch_problem<8, true>(a, P, smem, st); break;
            case 16: launch_problem<16, true>(a, P, smem, st); break;
            case 32: launch_problem<32, true>(a, P, smem, st); break;
            case 64: launch_problem<64, true>(a, P, smem, st); break;
            case 128: launch_problem<128, true>(a, P, smem, st); break;
            default: fail(PQKV_ERUNTIME, "kmeans: bad filter dim");
        }
    } else {
        switch (D) {
            case 2: launch_problem<2, false>(a, P, smem, st); break;
            case 4: launch_problem<4, false>(a, P, smem, st); break;
            case 8: launch_problem<8, false>(a, P, smem, st); break;
            case 16: launch_problem<16, false>(a, P, smem, st); break;
            case 32: launch_problem<32, false>(a, P, smem, st); break;
            case 64: launch_problem<64, false>(a, P, smem, st); break;
            default: launch_problem<0, false>(a, P, smem, st); break;
        }
    }
    unsigned long long stats[4] = {0, 0, 0, 0};
    PQKV_CUDA(cudaMemcpyAsync(stats, ctx->d_stats, sizeof(stats), cudaMemcpyDeviceToHost, st));
    PQKV_CUDA(cudaMemcpyAsync(ctx->last_phase_cycles, a.timers, 8 * sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, st));
    PQKV_CUDA(cudaStreamSynchronize(st));
    ctx->last_rechecked = stats[0];
    ctx->last_total = stats[1];
    ctx->last_phase_cycles[6] = stats[2];  // Hamerly-skipped point visits
    ctx->last_phase_cycles[7] = stats[3];  // k-means++ triangle-skipped point visits
}

void launch_encode(pqkv_ctx* ctx, const float* keys, size_t n_heads, size_t key_stride,
                   size_t d_h, size_t m, size_t C, const float* centroids, uint16_t* codes,
                   size_t codes_head_stride, size_t row, cudaStream_t st) {
    bind_device(ctx);
    int threads = (int)std::min<size_t>(32 * m, 256);
    encode_kernel<<<(unsigned)n_heads, threads, 0, st>>>(keys, (long long)key_stride, (int)d_h,
                                                         (int)m, (int)C, centroids, codes,
                                                         (long long)codes_head_stride, (long long)row);
    PQKV_LAUNCHED("encode_kernel");
}

void launch_assign_nearest(pqkv_ctx* ctx, const float* points, size_t n, size_t dim,
                           const float* centroids, size_t k, uint32_t* assign, cudaStream_t st) {
    bind_device(ctx);
    if (n == 0) return;
    assign_nearest_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(points, (int)n, (int)dim,
                                                                     centroids, (int)k, assign);
    PQKV_LAUNCHED("assign_nearest_kernel");
}

}  // namespace pqkv_dev
