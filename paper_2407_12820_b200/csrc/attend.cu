// attend.cu -- K/V gather + sparse softmax attention on sm_100a (hot path B).
//
// selective_attention (attention.cpp:62-91) attends over init [0,n_init) ++
// the selected middle tokens in ascending id ++ the local window: on the flat
// per-head layout that is simply the selected token ids in ascending order.
//
// Fast path (d_h = 128, fp32, PQKV_PREC_F32) -- the decode hot loop:
//   grid = (chunks + 1) x heads.  CTA c of a head owns middle rows
//   [c*CHUNK, (c+1)*CHUNK); it expands that slice of the selection bitmap
//   into row ids in shared memory, then every 8-lane group of a warp gathers
//   one 512 B K row and one V row per step with coalesced 128-bit loads
//   (16 floats per lane) and folds it into a warp-level online softmax
//   (log2 domain, exp2f).  The last CTA of a head takes the init + local
//   rows.  Groups, then warps, then CTAs are merged with the usual
//   (max, sum, acc) rescaling; combine_kernel merges the per-CTA partials.
//
// Exact path (PQKV_PREC_F64, any d_h) -- the C++ API drop-in:
//   exact_scores (attention.cpp:11-26) in fp64 with the same summation order
//   (bit-identical f32 scores), max-subtracted fp64 exp, the serial fp64 total
//   and the row-ordered fp64 accumulation of softmax_attention
//   (attention.cpp:35-60).  Only exp() differs in implementation from libm.
#include <cfloat>
#include <cmath>

#include "internal.cuh"

namespace pqkv_dev {
namespace {

constexpr int AT_THREADS = 256;
constexpr int AT_WARPS = AT_THREADS / 32;
constexpr int CHUNK = 4096;  // middle rows per CTA (bitmap mode) / list positions (rows mode)
constexpr int DH = 128;

struct AtArgs {
    const float* queries;  // [P][G][128]
    const float* keys;
    const float* values;
    long long kv_head_stride;
    // bitmap mode
    const uint32_t* bitmap;  // [P][words]
    int words, s_mid, n_init, n_local, total;
    // rows mode
    const int64_t* rows;  // [P][t]
    int t;
    int n_chunks;          // chunks per head including the init/local chunk (bitmap mode)
    float scale_log2;      // log2(e) / sqrt(d_h)
    float* part;           // [P][n_chunks][G][DH + 2]
    unsigned* arrivals;    // [P] zero on entry; reset by the combining CTA
    float* out;            // [P][G][DH]
};

__device__ __forceinline__ float safe_scale(float m_old, float m_new) {
    return m_old == -INFINITY ? 0.0f : exp2f(m_old - m_new);
}

template <int G, int RPI>
__global__ void __launch_bounds__(AT_THREADS) attend_kernel(AtArgs a) {
    __shared__ int rows_s[CHUNK + 128];
    __shared__ int nrows_s;
    __shared__ uint32_t wcnt[CHUNK / 32];
    __shared__ float wm[AT_WARPS][G], wl[AT_WARPS][G];
    // wacc (warp partials) reuses rows_s once the gather loop is done
    static_assert(AT_WARPS * G * DH <= CHUNK + 128, "warp partials must fit the row buffer");

    const int p = blockIdx.y, c = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int grp = lane >> 3, gl = lane & 7;

    // ---- 1. this CTA's row list ----
    if (a.bitmap) {
        const int last = a.n_chunks - 1;
        if (c < last) {
            const int w0 = c * (CHUNK / 32);
            const int nw = min(CHUNK / 32, a.words - w0);
            uint32_t bits = 0;
            if (tid < CHUNK / 32) {
                bits = tid < nw ? a.bitmap[(long long)p * a.words + w0 + tid] : 0u;
                wcnt[tid] = __popc(bits);
            }
            __syncthreads();
            if (tid == 0) {  // exclusive scan of 128 word counts
                uint32_t run = 0;
                for (int w = 0; w < CHUNK / 32; ++w) { uint32_t v = wcnt[w]; wcnt[w] = run; run += v; }
                nrows_s = (int)run;
            }
            __syncthreads();
            if (tid < CHUNK / 32) {
                int off = (int)wcnt[tid];
                int base = a.n_init + (w0 + tid) * 32;
                while (bits) {
                    int b = __ffs(bits) - 1;
                    bits &= bits - 1;
                    rows_s[off++] = base + b;
                }
            }
        } else {
            const int ni = a.n_init, nl = a.n_local;
            for (int e = tid; e < ni + nl; e += AT_THREADS)
                rows_s[e] = e < ni ? e : a.total - nl + (e - ni);
            if (tid == 0) nrows_s = ni + nl;
        }
    } else {
        const int b0 = c * CHUNK;
        const int cnt = min(CHUNK, a.t - b0);
        for (int e = tid; e < cnt; e += AT_THREADS) rows_s[e] = (int)a.rows[(long long)p * a.t + b0 + e];
        if (tid == 0) nrows_s = max(cnt, 0);
    }
    __syncthreads();
    const int nrows = nrows_s;

    // ---- 2. queries in the lane layout: dims {32j + 4gl + e} ----
    float q[G][16];
#pragma unroll
    for (int r = 0; r < G; ++r) {
        const float4* qp = reinterpret_cast<const float4*>(a.queries + ((long long)p * G + r) * DH);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float4 v = __ldg(qp + j * 8 + gl);
            q[r][4 * j + 0] = v.x * a.scale_log2;
            q[r][4 * j + 1] = v.y * a.scale_log2;
            q[r][4 * j + 2] = v.z * a.scale_log2;
            q[r][4 * j + 3] = v.w * a.scale_log2;
        }
    }
    float m[G], l[G], acc[G][16];
#pragma unroll
    for (int r = 0; r < G; ++r) {
        m[r] = -INFINITY;
        l[r] = 0.f;
#pragma unroll
        for (int e = 0; e < 16; ++e) acc[r][e] = 0.f;
    }

    const float* kbase = a.keys + (long long)p * a.kv_head_stride;
    const float* vbase = a.values + (long long)p * a.kv_head_stride;
    const int slot = warp * 4 + grp;        // 0..31
    const int stride = AT_WARPS * 4 * RPI;  // rows per CTA step

    // ---- 3. gather + online softmax ----
    for (int base = 0; base < nrows; base += stride) {
        float4 kr[RPI][4], vr[RPI][4];
        bool valid[RPI];
#pragma unroll
        for (int u = 0; u < RPI; ++u) {
            int ri = base + u * AT_WARPS * 4 + slot;
            valid[u] = ri < nrows;
            int row = valid[u] ? rows_s[ri] : rows_s[0];
            const float4* kp = reinterpret_cast<const float4*>(kbase + (long long)row * DH);
            const float4* vp = reinterpret_cast<const float4*>(vbase + (long long)row * DH);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                kr[u][j] = __ldg(kp + j * 8 + gl);
                vr[u][j] = __ldg(vp + j * 8 + gl);
            }
        }
#pragma unroll
        for (int r = 0; r < G; ++r) {
            float s[RPI];
#pragma unroll
            for (int u = 0; u < RPI; ++u) {
                float d = 0.f;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    d = fmaf(q[r][4 * j + 0], kr[u][j].x, d);
                    d = fmaf(q[r][4 * j + 1], kr[u][j].y, d);
                    d = fmaf(q[r][4 * j + 2], kr[u][j].z, d);
                    d = fmaf(q[r][4 * j + 3], kr[u][j].w, d);
                }
                d += __shfl_xor_sync(FULL, d, 1);
                d += __shfl_xor_sync(FULL, d, 2);
                d += __shfl_xor_sync(FULL, d, 4);
                s[u] = valid[u] ? d : -INFINITY;
            }
            float mn = m[r];
#pragma unroll
            for (int u = 0; u < RPI; ++u) mn = fmaxf(mn, s[u]);
            if (mn == -INFINITY) continue;
            float alpha = safe_scale(m[r], mn);
            float pw[RPI];
            float lsum = 0.f;
#pragma unroll
            for (int u = 0; u < RPI; ++u) { pw[u] = exp2f(s[u] - mn); lsum += pw[u]; }
            l[r] = l[r] * alpha + lsum;
            m[r] = mn;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                float o0 = acc[r][4 * j + 0] * alpha, o1 = acc[r][4 * j + 1] * alpha;
                float o2 = acc[r][4 * j + 2] * alpha, o3 = acc[r][4 * j + 3] * alpha;
#pragma unroll
                for (int u = 0; u < RPI; ++u) {
                    o0 = fmaf(pw[u], vr[u][j].x, o0);
                    o1 = fmaf(pw[u], vr[u][j].y, o1);
                    o2 = fmaf(pw[u], vr[u][j].z, o2);
                    o3 = fmaf(pw[u], vr[u][j].w, o3);
                }
                acc[r][4 * j + 0] = o0;
                acc[r][4 * j + 1] = o1;
                acc[r][4 * j + 2] = o2;
                acc[r][4 * j + 3] = o3;
            }
        }
    }

    // ---- 4. merge the 4 groups of the warp (lanes gl, gl+8, gl+16, gl+24) ----
#pragma unroll
    for (int r = 0; r < G; ++r) {
#pragma unroll
        for (int o = 8; o <= 16; o <<= 1) {
            float mo = __shfl_xor_sync(FULL, m[r], o);
            float lo = __shfl_xor_sync(FULL, l[r], o);
            float mn = fmaxf(m[r], mo);
            float sa = safe_scale(m[r], mn), sb = safe_scale(mo, mn);
            l[r] = l[r] * sa + lo * sb;
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                float ao = __shfl_xor_sync(FULL, acc[r][e], o);
                acc[r][e] = acc[r][e] * sa + ao * sb;
            }
            m[r] = mn;
        }
    }
    __syncthreads();  // every warp is past the gather loop: rows_s is free
    float* wacc = reinterpret_cast<float*>(rows_s);
#pragma unroll
    for (int r = 0; r < G; ++r) {
        if (grp == 0) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) wacc[(warp * G + r) * DH + 32 * j + 4 * gl + e] = acc[r][4 * j + e];
            if (gl == 0) { wm[warp][r] = m[r]; wl[warp][r] = l[r]; }
        }
    }
    __syncthreads();

    // ---- 5. merge warps, write this CTA's partial ----
    for (int e = tid; e < G * DH; e += AT_THREADS) {
        int r = e / DH, d = e % DH;
        float M = -INFINITY;
        for (int w = 0; w < AT_WARPS; ++w) M = fmaxf(M, wm[w][r]);
        float L = 0.f, O = 0.f;
        if (M != -INFINITY) {
            for (int w = 0; w < AT_WARPS; ++w) {
                float sc = safe_scale(wm[w][r], M);
                L += wl[w][r] * sc;
                O += wacc[(w * G + r) * DH + d] * sc;
            }
        }
        float* out = a.part + (((long long)p * a.n_chunks + c) * G + r) * (DH + 2);
        out[2 + d] = O;
        if (d == 0) { out[0] = M; out[1] = L; }
    }

    // ---- 6. the last CTA of this head merges all partials (no extra launch) ----
    __shared__ unsigned ticket;
    __threadfence();
    __syncthreads();
    if (tid == 0) ticket = atomicAdd(&a.arrivals[p], 1u);
    __syncthreads();
    if (ticket != (unsigned)a.n_chunks - 1) return;
    __threadfence();
    float* sc = reinterpret_cast<float*>(rows_s);  // [G][n_chunks] scale, then [G] sums
    const int nc = a.n_chunks;
    const float* pb = a.part + (long long)p * nc * G * (DH + 2);
    for (int r = warp; r < G; r += AT_WARPS) {
        float M = -INFINITY;
        for (int cc = lane; cc < nc; cc += 32) M = fmaxf(M, __ldcg(pb + ((long long)cc * G + r) * (DH + 2)));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(FULL, M, o));
        float L = 0.f;
        for (int cc = lane; cc < nc; cc += 32) {
            const float* pc = pb + ((long long)cc * G + r) * (DH + 2);
            float f = safe_scale(__ldcg(pc), M);
            sc[r * nc + cc] = f;
            L += __ldcg(pc + 1) * f;
        }
        L = warp_sum(L);
        if (lane == 0) sc[G * nc + r] = L;
    }
    __syncthreads();
    for (int e = tid; e < G * DH; e += AT_THREADS) {
        const int r = e / DH, d = e % DH;
        float O = 0.f;
#pragma unroll 4
        for (int cc = 0; cc < nc; ++cc) O = fmaf(__ldcg(pb + ((long long)cc * G + r) * (DH + 2) + 2 + d), sc[r * nc + cc], O);
        a.out[((long long)p * G + r) * DH + d] = O / sc[G * nc + r];
    }
    if (tid == 0) a.arrivals[p] = 0;  // ready for the next launch on this stream
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

// softmax_attention (attention.cpp:35-60) given the f32 scores.
__global__ void softmax_exact_kernel(const float* scores, int G, int d_h, const float* values,
                                     long long kv_head_stride, const int64_t* rows, int t,
                                     double* w, float* out) {
    const int pr = blockIdx.x, p = pr / G;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float* sc = scores + (long long)pr * t;
    double* wr = w + (long long)pr * t;
    __shared__ float smax[32];
    __shared__ double stotal;
    // max_element: first maximal f32 score
    float mx = -INFINITY;
    for (int i = tid; i < t; i += blockDim.x) mx = fmaxf(mx, sc[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, o));
    if (lane == 0) smax[warp] = mx;
    __syncthreads();
    if (tid == 0) {
        float v = smax[0];
        for (int e = 1; e < (int)(blockDim.x >> 5); ++e) v = fmaxf(v, smax[e]);
        smax[0] = v;
    }
    __syncthreads();
    const double max_score = (double)smax[0];
    for (int i = tid; i < t; i += blockDim.x) wr[i] = exp(__dsub_rn((double)sc[i], max_score));
    __syncthreads();
    if (warp == 0) {  // serial total in row order
        double total = 0.0;
        for (int i0 = 0; i0 < t; i0 += 32) {
            double v = (i0 + lane < t) ? wr[i0 + lane] : 0.0;
            int cnt = min(32, t - i0);
            for (int e = 0; e < cnt; ++e) total = __dadd_rn(total, __shfl_sync(FULL, v, e));
        }
        if (lane == 0) stotal = total;
    }
    __syncthreads();
    const double total = stotal;
    for (int i = tid; i < t; i += blockDim.x) wr[i] = __ddiv_rn(wr[i], total);
    __syncthreads();
    const float* vb = values + p * kv_head_stride;
    const int64_t* rr = rows + (long long)p * t;
    for (int j = tid; j < d_h; j += blockDim.x) {
        double accv = 0.0;
        for (int i = 0; i < t; ++i)
            accv = __dadd_rn(accv, __dmul_rn(wr[i], (double)__ldg(vb + rr[i] * d_h + j)));
        out[(long long)pr * d_h + j] = (float)accv;
    }
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

template <int G>
void launch_fast(const AtArgs& a, dim3 grid, cudaStream_t st) {
    if constexpr (G <= 2)
        attend_kernel<G, 2><<<grid, AT_THREADS, 0, st>>>(a);
    else
        attend_kernel<G, 1><<<grid, AT_THREADS, 0, st>>>(a);
    PQKV_LAUNCHED("attend_kernel");
}

bool launch_fast_any(int G, const AtArgs& a, dim3 grid, cudaStream_t st) {
    switch (G) {
        case 1: launch_fast<1>(a, grid, st); return true;
        case 2: launch_fast<2>(a, grid, st); return true;
        case 4: launch_fast<4>(a, grid, st); return true;
        default: return false;
    }
}

}  // namespace

void launch_exact(pqkv_ctx* ctx, const float* queries, size_t P, size_t G, size_t d_h,
                  const float* keys, const float* values, size_t kv_head_stride,
                  const int64_t* rows, size_t t, float* out, cudaStream_t st) {
    Scratch sc(ctx);
    size_t h_s = sc.plan<float>(P * G * t), h_w = sc.plan<double>(P * G * t);
    sc.commit();
    float* scores = sc.get<float>(h_s);
    double* w = sc.get<double>(h_w);
    double scale = 1.0 / std::sqrt(static_cast<double>(d_h));
    dim3 g1((unsigned)ceil_div(t, 128), (unsigned)(P * G));
    exact_scores_kernel<<<g1, 128, 0, st>>>(queries, (int)G, (int)d_h, keys, (long long)kv_head_stride,
                                           rows, (int)t, scale, scores);
    PQKV_LAUNCHED("exact_scores_kernel");
    int threads = (int)std::min<size_t>(1024, std::max<size_t>(128, round_up(d_h, 32)));
    softmax_exact_kernel<<<(unsigned)(P * G), threads, 0, st>>>(scores, (int)G, (int)d_h, values,
                                                               (long long)kv_head_stride, rows,
                                                               (int)t, w, out);
    PQKV_LAUNCHED("softmax_exact_kernel");
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
    const int chunks = (int)ceil_div(t, CHUNK);
    Scratch sc(ctx);
    size_t h_part = sc.plan<float>(P * chunks * G * (DH + 2));
    sc.commit();
    AtArgs a{};
    a.queries = queries;
    a.keys = keys;
    a.values = values;
    a.kv_head_stride = (long long)kv_head_stride;
    a.rows = rows;
    a.t = (int)t;
    a.n_chunks = chunks;
    a.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)d_h));
    a.part = sc.get<float>(h_part);
    a.arrivals = arrival_counters(ctx, P, st);
    a.out = out;
    launch_fast_any((int)G, a, dim3((unsigned)chunks, (unsigned)P), st);
}

bool launch_decode_attend(pqkv_ctx* ctx, const pqkv_layer& L, const float* queries, size_t G,
                          const uint32_t* bitmap, float* out, cudaStream_t st, int* launches) {
    bind_device(ctx);
    const size_t s_mid = L.total - L.n_init - L.n_local;
    const size_t words = ceil_div(s_mid, 32);
    bool fast = L.d_h == DH && (G == 1 || G == 2 || G == 4) && L.kv_head_stride % 4 == 0;
    if (fast) {
        const int mid_chunks = (int)ceil_div(s_mid, CHUNK);
        const int chunks = mid_chunks + 1;
        Scratch sc(ctx);
        size_t h_part = sc.plan<float>(L.n_heads * chunks * G * (DH + 2));
        sc.commit();
        AtArgs a{};
        a.queries = queries;
        a.keys = L.keys;
        a.values = L.values;
        a.kv_head_stride = (long long)L.kv_head_stride;
        a.bitmap = bitmap;
        a.words = (int)words;
        a.s_mid = (int)s_mid;
        a.n_init = (int)L.n_init;
        a.n_local = (int)L.n_local;
        a.total = (int)L.total;
        a.n_chunks = chunks;
        a.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)L.d_h));
        a.part = sc.get<float>(h_part);
        a.arrivals = arrival_counters(ctx, L.n_heads, st);
        a.out = out;
        launch_fast_any((int)G, a, dim3((unsigned)chunks, (unsigned)L.n_heads), st);
        if (launches) *launches = 1;
        return true;
    }
    return false;  // caller materialises row lists and runs the exact kernels
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
