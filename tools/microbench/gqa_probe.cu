// GQA gather probe (cfg3 geometry: 8 kv heads x g = 4, 26282 selected rows
// per head of 131072, fp32 K/V): attention over row lists, two designs.
//   H  half-warp per row, per-lane cp.async ring (attend_kernel's g > 1 path)
//   W  warp per row, per-warp ring of D rows staged by cp.async.bulk (one
//      lane issues two 512 B bulk copies per row, completion on an mbarrier),
//      g dot products reduced by a transpose-reduce (6 shuffles for g = 4)
// Each variant writes per-CTA partials (m, l, acc); a check kernel merges
// them and compares with a naive fp32 reference.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cmath>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int P = 8, S = 131072, DH = 128, SEL = 26282, G = 4;
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ float safe_scale(float mo, float mn) { return mo == -INFINITY ? 0.f : exp2f(mo - mn); }

// ---- mbarrier / bulk-copy helpers ----
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar, uint64_t pol) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n"
                 ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ uint64_t evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// ---- W: warp per row, bulk-copy ring ----
template <int D, int MINB>
__global__ void __launch_bounds__(256, MINB) gqa_w(const float* __restrict__ K, const float* __restrict__ V,
                                                   const int* __restrict__ rows, int per_cta, const float* __restrict__ Q,
                                                   float scale_log2, float* part) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int p = blockIdx.y, c = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    float4* ring = reinterpret_cast<float4*>(sm) + (size_t)warp * D * 64;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + 8 * D * 1024) + warp * D;
    const int r0 = c * per_cta, n = max(0, min(per_cta, SEL - r0));
    const int* rl = rows + (size_t)p * SEL + r0;
    const float* kb = K + (size_t)p * S * DH;
    const float* vb = V + (size_t)p * S * DH;
    const uint64_t pol = evict_first();
    if (lane == 0)
        for (int s = 0; s < D; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    auto issue = [&](int i, int s) {  // lane 0 only
        const long long row = rl[i];
        mbar_expect_tx(&bars[s], 1024);
        bulk_g2s(ring + s * 64, kb + row * DH, 512, &bars[s], pol);
        bulk_g2s(ring + s * 64 + 32, vb + row * DH, 512, &bars[s], pol);
    };
    const int mine = n > warp ? (n - warp + 7) / 8 : 0;  // rows warp, warp+8, ...
    if (lane == 0)
        for (int s = 0; s < D && s < mine; ++s) issue(warp + 8 * s, s);
    float4 q[G];
#pragma unroll
    for (int r = 0; r < G; ++r) {
        float4 v = reinterpret_cast<const float4*>(Q + ((size_t)p * G + r) * DH)[lane];
        q[r] = make_float4(v.x * scale_log2, v.y * scale_log2, v.z * scale_log2, v.w * scale_log2);
    }
    const bool b4 = lane & 16, b3 = lane & 8;
    const int own = (b4 ? 2 : 0) + (b3 ? 1 : 0);  // query row this lane's group reduces
    float m_own = -INFINITY, l_own = 0.f;
    float4 acc[G];
#pragma unroll
    for (int r = 0; r < G; ++r) acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int it = 0; it < mine; ++it) {
        const int s = it % D;
        mbar_wait(&bars[s], (it / D) & 1);
        const float4 k = ring[s * 64 + lane], v = ring[s * 64 + 32 + lane];
        __syncwarp();
        if (lane == 0 && it + D < mine) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(warp + 8 * (it + D), s);
        }
        float d[G];
#pragma unroll
        for (int r = 0; r < G; ++r) d[r] = fmaf(q[r].x, k.x, fmaf(q[r].y, k.y, fmaf(q[r].z, k.z, q[r].w * k.w)));
        // transpose-reduce: after xor 16 / 8 a lane holds a 4-lane partial of
        // row `own`; xor 4 / 2 / 1 complete it
        float a0 = b4 ? d[2] : d[0], a1 = b4 ? d[3] : d[1];
        const float s0 = b4 ? d[0] : d[2], s1 = b4 ? d[1] : d[3];
        a0 += __shfl_xor_sync(FULL, s0, 16);
        a1 += __shfl_xor_sync(FULL, s1, 16);
        float x = b3 ? a1 : a0;
        x += __shfl_xor_sync(FULL, b3 ? a0 : a1, 8);
        x += __shfl_xor_sync(FULL, x, 4);
        x += __shfl_xor_sync(FULL, x, 2);
        x += __shfl_xor_sync(FULL, x, 1);
        float alpha = 1.f;
        if (x > m_own) {
            alpha = safe_scale(m_own, x);
            l_own *= alpha;
            m_own = x;
        }
        const float pw = exp2f(x - m_own);
        l_own += pw;
        const bool grew = __any_sync(FULL, alpha != 1.f);
#pragma unroll
        for (int r = 0; r < G; ++r) {
            const float pr = __shfl_sync(FULL, pw, 8 * r);
            if (grew) {
                const float ar = __shfl_sync(FULL, alpha, 8 * r);
                acc[r].x *= ar; acc[r].y *= ar; acc[r].z *= ar; acc[r].w *= ar;
            }
            acc[r].x = fmaf(pr, v.x, acc[r].x);
            acc[r].y = fmaf(pr, v.y, acc[r].y);
            acc[r].z = fmaf(pr, v.z, acc[r].z);
            acc[r].w = fmaf(pr, v.w, acc[r].w);
        }
    }
    // per-warp partials -> part[p][c][warp][r][DH+2]
    float* o = part + ((((size_t)p * gridDim.x + c) * 8 + warp) * G) * (DH + 2);
#pragma unroll
    for (int r = 0; r < G; ++r) {
        const float mr = __shfl_sync(FULL, m_own, 8 * r), lr = __shfl_sync(FULL, l_own, 8 * r);
        float* orow = o + r * (DH + 2);
        if (lane == 0) { orow[0] = mr; orow[1] = lr; }
        reinterpret_cast<float*>(orow + 2)[4 * lane + 0] = acc[r].x;
        reinterpret_cast<float*>(orow + 2)[4 * lane + 1] = acc[r].y;
        reinterpret_cast<float*>(orow + 2)[4 * lane + 2] = acc[r].z;
        reinterpret_cast<float*>(orow + 2)[4 * lane + 3] = acc[r].w;
    }
}

// ---- H: half-warp per row, per-lane cp.async ring (depth 4) ----
__device__ __forceinline__ void cp16(void* s, const void* g, uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_u32(s)), "l"(g), "l"(pol) : "memory");
}
__global__ void __launch_bounds__(256, 2) gqa_h(const float* __restrict__ K, const float* __restrict__ V,
                                                const int* __restrict__ rows, int per_cta, const float* __restrict__ Q,
                                                float scale_log2, float* part) {
    extern __shared__ __align__(128) unsigned char sm[];
    constexpr int RING = 4, LPR = 16, VPL = 2, STEP = 16;
    const int p = blockIdx.y, c = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int half = lane >> 4, hl = lane & 15, slot = warp * 2 + half;
    const int r0 = c * per_cta, n = max(0, min(per_cta, SEL - r0));
    const int* rl = rows + (size_t)p * SEL + r0;
    const float4* kb = reinterpret_cast<const float4*>(K + (size_t)p * S * DH);
    const float4* vb = reinterpret_cast<const float4*>(V + (size_t)p * S * DH);
    float4* ring = reinterpret_cast<float4*>(sm) + (size_t)slot * RING * 64;
    const uint64_t pol = evict_first();
    float q[G][8];
    for (int r = 0; r < G; ++r)
        for (int j = 0; j < VPL; ++j) {
            float4 v = reinterpret_cast<const float4*>(Q + ((size_t)p * G + r) * DH)[j * LPR + hl];
            q[r][4 * j] = v.x * scale_log2; q[r][4 * j + 1] = v.y * scale_log2;
            q[r][4 * j + 2] = v.z * scale_log2; q[r][4 * j + 3] = v.w * scale_log2;
        }
    float m[G], l[G], acc[G][8];
    for (int r = 0; r < G; ++r) { m[r] = -INFINITY; l[r] = 0.f; for (int e = 0; e < 8; ++e) acc[r][e] = 0.f; }
    auto issue = [&](int rr, int u) {
        if (rr < n) {
            const long long row = rl[rr];
            for (int j = 0; j < VPL; ++j) {
                cp16(ring + u * 64 + j * LPR + hl, kb + row * 32 + j * LPR + hl, pol);
                cp16(ring + u * 64 + 32 + j * LPR + hl, vb + row * 32 + j * LPR + hl, pol);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int u = 0; u < RING; ++u) issue(slot + u * STEP, u);
    for (int it = 0, ri = slot; ri < n; ri += STEP, ++it) {
        asm volatile("cp.async.wait_group 3;" ::: "memory");
        const int u = it & 3;
        float4 kc[2], vc[2];
        for (int j = 0; j < 2; ++j) { kc[j] = ring[u * 64 + j * LPR + hl]; vc[j] = ring[u * 64 + 32 + j * LPR + hl]; }
        issue(ri + RING * STEP, u);
#pragma unroll
        for (int r = 0; r < G; ++r) {
            float d = 0.f;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                d = fmaf(q[r][4 * j], kc[j].x, d); d = fmaf(q[r][4 * j + 1], kc[j].y, d);
                d = fmaf(q[r][4 * j + 2], kc[j].z, d); d = fmaf(q[r][4 * j + 3], kc[j].w, d);
            }
            for (int o = 1; o < 16; o <<= 1) d += __shfl_xor_sync(0xffffu << (half * 16), d, o, 16);
            if (d > m[r]) { float a = safe_scale(m[r], d); l[r] *= a; for (int e = 0; e < 8; ++e) acc[r][e] *= a; m[r] = d; }
            const float pw = exp2f(d - m[r]);
            l[r] += pw;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                acc[r][4 * j] = fmaf(pw, vc[j].x, acc[r][4 * j]); acc[r][4 * j + 1] = fmaf(pw, vc[j].y, acc[r][4 * j + 1]);
                acc[r][4 * j + 2] = fmaf(pw, vc[j].z, acc[r][4 * j + 2]); acc[r][4 * j + 3] = fmaf(pw, vc[j].w, acc[r][4 * j + 3]);
            }
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    // per half-warp partial: 16 slots -> stored as "warp" entries 0..15 (part sized for 16)
    float* o = part + ((((size_t)p * gridDim.x + c) * 16 + slot) * G) * (DH + 2);
    for (int r = 0; r < G; ++r) {
        float* orow = o + r * (DH + 2);
        if (hl == 0) { orow[0] = m[r]; orow[1] = l[r]; }
        for (int j = 0; j < 2; ++j)
            for (int e = 0; e < 4; ++e) orow[2 + 64 * j + 4 * hl + e] = acc[r][4 * j + e];
    }
}


// ---- W2: warp per row, per-lane cp.async ring of D rows (no TMA) ----
template <int D, int MINB>
__global__ void __launch_bounds__(256, MINB) gqa_w2(const float* __restrict__ K, const float* __restrict__ V,
                                                    const int* __restrict__ rows, int per_cta, const float* __restrict__ Q,
                                                    float scale_log2, float* part) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int p = blockIdx.y, c = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    float4* ring = reinterpret_cast<float4*>(sm) + (size_t)warp * D * 64;
    const int r0 = c * per_cta, n = max(0, min(per_cta, SEL - r0));
    const int* rl = rows + (size_t)p * SEL + r0;
    const float4* kb = reinterpret_cast<const float4*>(K + (size_t)p * S * DH);
    const float4* vb = reinterpret_cast<const float4*>(V + (size_t)p * S * DH);
    const uint64_t pol = evict_first();
    const int mine = n > warp ? (n - warp + 7) / 8 : 0;
    auto issue = [&](int it, int s) {
        if (it < mine) {
            const long long row = rl[warp + 8 * it];
            cp16(ring + s * 64 + lane, kb + row * 32 + lane, pol);
            cp16(ring + s * 64 + 32 + lane, vb + row * 32 + lane, pol);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
#pragma unroll
    for (int s = 0; s < D; ++s) issue(s, s);
    float4 q[G];
#pragma unroll
    for (int r = 0; r < G; ++r) {
        float4 v = reinterpret_cast<const float4*>(Q + ((size_t)p * G + r) * DH)[lane];
        q[r] = make_float4(v.x * scale_log2, v.y * scale_log2, v.z * scale_log2, v.w * scale_log2);
    }
    const bool b4 = lane & 16, b3 = lane & 8;
    float m_own = -INFINITY, l_own = 0.f;
    float4 acc[G];
#pragma unroll
    for (int r = 0; r < G; ++r) acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int it = 0; it < mine; ++it) {
        const int s = it % D;
        asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
        const float4 k = ring[s * 64 + lane], v = ring[s * 64 + 32 + lane];
        issue(it + D, s);
        float d[G];
#pragma unroll
        for (int r = 0; r < G; ++r) d[r] = fmaf(q[r].x, k.x, fmaf(q[r].y, k.y, fmaf(q[r].z, k.z, q[r].w * k.w)));
        float a0 = b4 ? d[2] : d[0], a1 = b4 ? d[3] : d[1];
        const float s0 = b4 ? d[0] : d[2], s1 = b4 ? d[1] : d[3];
        a0 += __shfl_xor_sync(FULL, s0, 16);
        a1 += __shfl_xor_sync(FULL, s1, 16);
        float x = b3 ? a1 : a0;
        x += __shfl_xor_sync(FULL, b3 ? a0 : a1, 8);
        x += __shfl_xor_sync(FULL, x, 4);
        x += __shfl_xor_sync(FULL, x, 2);
        x += __shfl_xor_sync(FULL, x, 1);
        float alpha = 1.f;
        if (x > m_own) {
            alpha = safe_scale(m_own, x);
            l_own *= alpha;
            m_own = x;
        }
        const float pw = exp2f(x - m_own);
        l_own += pw;
        const bool grew = __any_sync(FULL, alpha != 1.f);
#pragma unroll
        for (int r = 0; r < G; ++r) {
            const float pr = __shfl_sync(FULL, pw, 8 * r);
            if (grew) {
                const float ar = __shfl_sync(FULL, alpha, 8 * r);
                acc[r].x *= ar; acc[r].y *= ar; acc[r].z *= ar; acc[r].w *= ar;
            }
            acc[r].x = fmaf(pr, v.x, acc[r].x);
            acc[r].y = fmaf(pr, v.y, acc[r].y);
            acc[r].z = fmaf(pr, v.z, acc[r].z);
            acc[r].w = fmaf(pr, v.w, acc[r].w);
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    float* o = part + ((((size_t)p * gridDim.x + c) * 8 + warp) * G) * (DH + 2);
#pragma unroll
    for (int r = 0; r < G; ++r) {
        const float mr = __shfl_sync(FULL, m_own, 8 * r), lr = __shfl_sync(FULL, l_own, 8 * r);
        float* orow = o + r * (DH + 2);
        if (lane == 0) { orow[0] = mr; orow[1] = lr; }
        orow[2 + 4 * lane + 0] = acc[r].x;
        orow[2 + 4 * lane + 1] = acc[r].y;
        orow[2 + 4 * lane + 2] = acc[r].z;
        orow[2 + 4 * lane + 3] = acc[r].w;
    }
}


// ---- W2P: W2 with packed fp32 (FFMA2 / FMUL2) dots and accumulators ----
template <int D, int MINB>
__global__ void __launch_bounds__(256, MINB) gqa_w2p(const float* __restrict__ K, const float* __restrict__ V,
                                                    const int* __restrict__ rows, int per_cta, const float* __restrict__ Q,
                                                    float scale_log2, float* part) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int p = blockIdx.y, c = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    float4* ring = reinterpret_cast<float4*>(sm) + (size_t)warp * D * 64;
    const int r0 = c * per_cta, n = max(0, min(per_cta, SEL - r0));
    const int* rl = rows + (size_t)p * SEL + r0;
    const float4* kb = reinterpret_cast<const float4*>(K + (size_t)p * S * DH);
    const float4* vb = reinterpret_cast<const float4*>(V + (size_t)p * S * DH);
    const uint64_t pol = evict_first();
    const int mine = n > warp ? (n - warp + 7) / 8 : 0;
    auto issue = [&](int it, int s) {
        if (it < mine) {
            const long long row = rl[warp + 8 * it];
            cp16(ring + s * 64 + lane, kb + row * 32 + lane, pol);
            cp16(ring + s * 64 + 32 + lane, vb + row * 32 + lane, pol);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
#pragma unroll
    for (int s = 0; s < D; ++s) issue(s, s);
    float4 q[G];
#pragma unroll
    for (int r = 0; r < G; ++r) {
        float4 v = reinterpret_cast<const float4*>(Q + ((size_t)p * G + r) * DH)[lane];
        q[r] = make_float4(v.x * scale_log2, v.y * scale_log2, v.z * scale_log2, v.w * scale_log2);
    }
    const bool b4 = lane & 16, b3 = lane & 8;
    float m_own = -INFINITY, l_own = 0.f;
    float4 acc[G];
#pragma unroll
    for (int r = 0; r < G; ++r) acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int it = 0; it < mine; ++it) {
        const int s = it % D;
        asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
        const float4 k = ring[s * 64 + lane], v = ring[s * 64 + 32 + lane];
        issue(it + D, s);
        float d[G];
        const float2 kxy = make_float2(k.x, k.y), kzw = make_float2(k.z, k.w);
#pragma unroll
        for (int r = 0; r < G; ++r) {
            const float2 t = __ffma2_rn(make_float2(q[r].z, q[r].w), kzw, __fmul2_rn(make_float2(q[r].x, q[r].y), kxy));
            d[r] = t.x + t.y;
        }
        float a0 = b4 ? d[2] : d[0], a1 = b4 ? d[3] : d[1];
        const float s0 = b4 ? d[0] : d[2], s1 = b4 ? d[1] : d[3];
        a0 += __shfl_xor_sync(FULL, s0, 16);
        a1 += __shfl_xor_sync(FULL, s1, 16);
        float x = b3 ? a1 : a0;
        x += __shfl_xor_sync(FULL, b3 ? a0 : a1, 8);
        x += __shfl_xor_sync(FULL, x, 4);
        x += __shfl_xor_sync(FULL, x, 2);
        x += __shfl_xor_sync(FULL, x, 1);
        float alpha = 1.f;
        if (x > m_own) {
            alpha = safe_scale(m_own, x);
            l_own *= alpha;
            m_own = x;
        }
        const float pw = exp2f(x - m_own);
        l_own += pw;
        const bool grew = __any_sync(FULL, alpha != 1.f);
#pragma unroll
        for (int r = 0; r < G; ++r) {
            const float pr = __shfl_sync(FULL, pw, 8 * r);
            float2 axy = make_float2(acc[r].x, acc[r].y), azw = make_float2(acc[r].z, acc[r].w);
            if (grew) {
                const float ar = __shfl_sync(FULL, alpha, 8 * r);
                axy = __fmul2_rn(axy, make_float2(ar, ar));
                azw = __fmul2_rn(azw, make_float2(ar, ar));
            }
            axy = __ffma2_rn(make_float2(pr, pr), make_float2(v.x, v.y), axy);
            azw = __ffma2_rn(make_float2(pr, pr), make_float2(v.z, v.w), azw);
            acc[r] = make_float4(axy.x, axy.y, azw.x, azw.y);
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    float* o = part + ((((size_t)p * gridDim.x + c) * 8 + warp) * G) * (DH + 2);
#pragma unroll
    for (int r = 0; r < G; ++r) {
        const float mr = __shfl_sync(FULL, m_own, 8 * r), lr = __shfl_sync(FULL, l_own, 8 * r);
        float* orow = o + r * (DH + 2);
        if (lane == 0) { orow[0] = mr; orow[1] = lr; }
        orow[2 + 4 * lane + 0] = acc[r].x;
        orow[2 + 4 * lane + 1] = acc[r].y;
        orow[2 + 4 * lane + 2] = acc[r].z;
        orow[2 + 4 * lane + 3] = acc[r].w;
    }
}


// ---- W3: W2 with two rows per warp iteration (independent reduction chains interleaved) ----
template <int D, int MINB>
__global__ void __launch_bounds__(256, MINB) gqa_w3(const float* __restrict__ K, const float* __restrict__ V,
                                                    const int* __restrict__ rows, int per_cta, const float* __restrict__ Q,
                                                    float scale_log2, float* part) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int p = blockIdx.y, c = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    float4* ring = reinterpret_cast<float4*>(sm) + (size_t)warp * D * 64;
    const int r0 = c * per_cta, n = max(0, min(per_cta, SEL - r0));
    const int* rl = rows + (size_t)p * SEL + r0;
    const float4* kb = reinterpret_cast<const float4*>(K + (size_t)p * S * DH);
    const float4* vb = reinterpret_cast<const float4*>(V + (size_t)p * S * DH);
    const uint64_t pol = evict_first();
    const int mine = n > warp ? (n - warp + 7) / 8 : 0;
    auto issue = [&](int it, int s) {
        if (it < mine) {
            const long long row = rl[warp + 8 * it];
            cp16(ring + s * 64 + lane, kb + row * 32 + lane, pol);
            cp16(ring + s * 64 + 32 + lane, vb + row * 32 + lane, pol);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
#pragma unroll
    for (int s = 0; s < D; ++s) issue(s, s);
    float4 q[G];
#pragma unroll
    for (int r = 0; r < G; ++r) {
        float4 v = reinterpret_cast<const float4*>(Q + ((size_t)p * G + r) * DH)[lane];
        q[r] = make_float4(v.x * scale_log2, v.y * scale_log2, v.z * scale_log2, v.w * scale_log2);
    }
    const bool b4 = lane & 16, b3 = lane & 8;
    float m_own = -INFINITY, l_own = 0.f;
    float4 acc[G];
#pragma unroll
    for (int r = 0; r < G; ++r) acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int it = 0; it < mine; it += 2) {
        const bool two = it + 1 < mine;
        const int s0 = it % D, s1 = (it + 1) % D;
        asm volatile("cp.async.wait_group %0;" ::"n"(D - 2) : "memory");
        const float4 k0 = ring[s0 * 64 + lane], v0 = ring[s0 * 64 + 32 + lane];
        const float4 k1 = two ? ring[s1 * 64 + lane] : make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 v1 = two ? ring[s1 * 64 + 32 + lane] : make_float4(0.f, 0.f, 0.f, 0.f);
        issue(it + D, s0);
        issue(it + 1 + D, s1);
        float x[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float4 k = h ? k1 : k0;
            float d[G];
#pragma unroll
            for (int r = 0; r < G; ++r) d[r] = fmaf(q[r].x, k.x, fmaf(q[r].y, k.y, fmaf(q[r].z, k.z, q[r].w * k.w)));
            float a0 = b4 ? d[2] : d[0], a1 = b4 ? d[3] : d[1];
            const float s0_ = b4 ? d[0] : d[2], s1_ = b4 ? d[1] : d[3];
            a0 += __shfl_xor_sync(FULL, s0_, 16);
            a1 += __shfl_xor_sync(FULL, s1_, 16);
            float xx = b3 ? a1 : a0;
            xx += __shfl_xor_sync(FULL, b3 ? a0 : a1, 8);
            xx += __shfl_xor_sync(FULL, xx, 4);
            xx += __shfl_xor_sync(FULL, xx, 2);
            xx += __shfl_xor_sync(FULL, xx, 1);
            x[h] = xx;
        }
        if (!two) x[1] = -INFINITY;
        const float mx = fmaxf(x[0], x[1]);
        float alpha = 1.f;
        if (mx > m_own) { alpha = safe_scale(m_own, mx); l_own *= alpha; m_own = mx; }
        const float pw0 = exp2f(x[0] - m_own), pw1 = two ? exp2f(x[1] - m_own) : 0.f;
        l_own += pw0 + pw1;
        const bool grew = __any_sync(FULL, alpha != 1.f);
#pragma unroll
        for (int r = 0; r < G; ++r) {
            const float p0 = __shfl_sync(FULL, pw0, 8 * r), p1 = __shfl_sync(FULL, pw1, 8 * r);
            if (grew) {
                const float ar = __shfl_sync(FULL, alpha, 8 * r);
                acc[r].x *= ar; acc[r].y *= ar; acc[r].z *= ar; acc[r].w *= ar;
            }
            acc[r].x = fmaf(p0, v0.x, fmaf(p1, v1.x, acc[r].x));
            acc[r].y = fmaf(p0, v0.y, fmaf(p1, v1.y, acc[r].y));
            acc[r].z = fmaf(p0, v0.z, fmaf(p1, v1.z, acc[r].z));
            acc[r].w = fmaf(p0, v0.w, fmaf(p1, v1.w, acc[r].w));
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    float* o = part + ((((size_t)p * gridDim.x + c) * 8 + warp) * G) * (DH + 2);
#pragma unroll
    for (int r = 0; r < G; ++r) {
        const float mr = __shfl_sync(FULL, m_own, 8 * r), lr = __shfl_sync(FULL, l_own, 8 * r);
        float* orow = o + r * (DH + 2);
        if (lane == 0) { orow[0] = mr; orow[1] = lr; }
        orow[2 + 4 * lane + 0] = acc[r].x;
        orow[2 + 4 * lane + 1] = acc[r].y;
        orow[2 + 4 * lane + 2] = acc[r].z;
        orow[2 + 4 * lane + 3] = acc[r].w;
    }
}

// merge partials [P][n_parts][G][DH+2] -> out [P][G][DH]

// ---- W2D: W2 with NW warps per CTA claiming rows dynamically (smem counter,
// CB rows per claim) -- fewer, larger CTAs whose warps all finish together ----
template <int D, int NW, int CB>
__global__ void __launch_bounds__(NW * 32, 32 / NW) gqa_w2d(const float* __restrict__ K, const float* __restrict__ V,
                                                      const int* __restrict__ rows, int per_cta, const float* __restrict__ Q,
                                                      float scale_log2, float* part) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ int ctr;
    const int p = blockIdx.y, c = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    float4* ring = reinterpret_cast<float4*>(sm) + (size_t)warp * D * 64;
    const int r0 = c * per_cta, n = max(0, min(per_cta, SEL - r0));
    const int* rl = rows + (size_t)p * SEL + r0;
    const float4* kb = reinterpret_cast<const float4*>(K + (size_t)p * S * DH);
    const float4* vb = reinterpret_cast<const float4*>(V + (size_t)p * S * DH);
    const uint64_t pol = evict_first();
    if (tid == 0) ctr = NW * CB;  // the first batch of each warp is static
    __syncthreads();
    int q_base = warp * CB, q_pos = 0;  // current batch [q_base, q_base + CB)
    int n_valid = 0;
    bool dry = false;
    auto next_row = [&]() -> int {
        if (q_pos == CB) {
            int b = 0;
            if (lane == 0) b = atomicAdd(&ctr, CB);
            q_base = __shfl_sync(FULL, b, 0);
            q_pos = 0;
        }
        const int i = q_base + q_pos++;
        return i < n ? rl[i] : -1;
    };
    auto issue = [&](int s) {
        if (!dry) {
            const int row = next_row();
            if (row >= 0) {
                cp16(ring + s * 64 + lane, kb + (long long)row * 32 + lane, pol);
                cp16(ring + s * 64 + 32 + lane, vb + (long long)row * 32 + lane, pol);
                ++n_valid;
            } else {
                dry = true;
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
#pragma unroll
    for (int s = 0; s < D; ++s) issue(s);
    float4 q[G];
#pragma unroll
    for (int r = 0; r < G; ++r) {
        float4 v = reinterpret_cast<const float4*>(Q + ((size_t)p * G + r) * DH)[lane];
        q[r] = make_float4(v.x * scale_log2, v.y * scale_log2, v.z * scale_log2, v.w * scale_log2);
    }
    const bool b4 = lane & 16, b3 = lane & 8;
    float m_own = -INFINITY, l_own = 0.f;
    float4 acc[G];
#pragma unroll
    for (int r = 0; r < G; ++r) acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int it = 0; it < n_valid; ++it) {
        const int s = it % D;
        asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
        const float4 k = ring[s * 64 + lane], v = ring[s * 64 + 32 + lane];
        issue(s);
        float d[G];
        const float2 kxy = make_float2(k.x, k.y), kzw = make_float2(k.z, k.w);
#pragma unroll
        for (int r = 0; r < G; ++r) {
            const float2 t = __ffma2_rn(make_float2(q[r].z, q[r].w), kzw, __fmul2_rn(make_float2(q[r].x, q[r].y), kxy));
            d[r] = t.x + t.y;
        }
        float a0 = b4 ? d[2] : d[0], a1 = b4 ? d[3] : d[1];
        const float s0 = b4 ? d[0] : d[2], s1 = b4 ? d[1] : d[3];
        a0 += __shfl_xor_sync(FULL, s0, 16);
        a1 += __shfl_xor_sync(FULL, s1, 16);
        float x = b3 ? a1 : a0;
        x += __shfl_xor_sync(FULL, b3 ? a0 : a1, 8);
        x += __shfl_xor_sync(FULL, x, 4);
        x += __shfl_xor_sync(FULL, x, 2);
        x += __shfl_xor_sync(FULL, x, 1);
        float alpha = 1.f;
        if (x > m_own) {
            alpha = safe_scale(m_own, x);
            l_own *= alpha;
            m_own = x;
        }
        const float pw = exp2f(x - m_own);
        l_own += pw;
        const bool grew = __any_sync(FULL, alpha != 1.f);
#pragma unroll
        for (int r = 0; r < G; ++r) {
            const float pr = __shfl_sync(FULL, pw, 8 * r);
            float2 axy = make_float2(acc[r].x, acc[r].y), azw = make_float2(acc[r].z, acc[r].w);
            if (grew) {
                const float ar = __shfl_sync(FULL, alpha, 8 * r);
                axy = __fmul2_rn(axy, make_float2(ar, ar));
                azw = __fmul2_rn(azw, make_float2(ar, ar));
            }
            axy = __ffma2_rn(make_float2(pr, pr), make_float2(v.x, v.y), axy);
            azw = __ffma2_rn(make_float2(pr, pr), make_float2(v.z, v.w), azw);
            acc[r] = make_float4(axy.x, axy.y, azw.x, azw.y);
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    float* o = part + ((((size_t)p * gridDim.x + c) * NW + warp) * G) * (DH + 2);
#pragma unroll
    for (int r = 0; r < G; ++r) {
        const float mr = __shfl_sync(FULL, m_own, 8 * r), lr = __shfl_sync(FULL, l_own, 8 * r);
        float* orow = o + r * (DH + 2);
        if (lane == 0) { orow[0] = mr; orow[1] = lr; }
        orow[2 + 4 * lane + 0] = acc[r].x;
        orow[2 + 4 * lane + 1] = acc[r].y;
        orow[2 + 4 * lane + 2] = acc[r].z;
        orow[2 + 4 * lane + 3] = acc[r].w;
    }
}

__global__ void merge(const float* part, int n_parts, float* out) {
    const int p = blockIdx.x / G, r = blockIdx.x % G, d = threadIdx.x;
    float M = -INFINITY;
    for (int i = 0; i < n_parts; ++i) M = fmaxf(M, part[(((size_t)p * n_parts + i) * G + r) * (DH + 2)]);
    float L = 0.f, O = 0.f;
    for (int i = 0; i < n_parts; ++i) {
        const float* pr = part + (((size_t)p * n_parts + i) * G + r) * (DH + 2);
        const float f = safe_scale(pr[0], M);
        L += pr[1] * f;
        O += pr[2 + d] * f;
    }
    out[((size_t)p * G + r) * DH + d] = O / L;
}

int main() {
    size_t kv = (size_t)P * S * DH;
    float *K, *V, *Q, *part, *out;
    CK(cudaMalloc(&K, kv * 4)); CK(cudaMalloc(&V, kv * 4));
    std::vector<float> h(kv);
    std::mt19937 rng(5);
    std::normal_distribution<float> nd;
    for (auto& x : h) x = nd(rng);
    CK(cudaMemcpy(K, h.data(), kv * 4, cudaMemcpyHostToDevice));
    for (auto& x : h) x = nd(rng);
    CK(cudaMemcpy(V, h.data(), kv * 4, cudaMemcpyHostToDevice));
    std::vector<float> hq(P * G * DH);
    for (auto& x : hq) x = nd(rng);
    CK(cudaMalloc(&Q, hq.size() * 4));
    CK(cudaMemcpy(Q, hq.data(), hq.size() * 4, cudaMemcpyHostToDevice));
    std::vector<int> rows((size_t)P * SEL), all(S);
    for (int p = 0; p < P; ++p) {
        for (int i = 0; i < S; ++i) all[i] = i;
        std::shuffle(all.begin(), all.end(), rng);
        std::sort(all.begin(), all.begin() + SEL);
        std::copy(all.begin(), all.begin() + SEL, rows.begin() + (size_t)p * SEL);
    }
    int* drows;
    CK(cudaMalloc(&drows, rows.size() * 4));
    CK(cudaMemcpy(drows, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&part, (size_t)64 << 20));
    CK(cudaMalloc(&out, P * G * DH * 4));
    const float sl = 1.4426950408889634f / sqrtf(128.f);
    // reference on the host for head 0..1
    std::vector<float> hk(kv), hv(kv);
    CK(cudaMemcpy(hk.data(), K, kv * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hv.data(), V, kv * 4, cudaMemcpyDeviceToHost));
    std::vector<double> ref(2 * G * DH, 0.0);
    for (int p = 0; p < 2; ++p)
        for (int r = 0; r < G; ++r) {
            std::vector<double> sc(SEL);
            double mx = -1e300;
            for (int i = 0; i < SEL; ++i) {
                const float* kr = &hk[((size_t)p * S + rows[(size_t)p * SEL + i]) * DH];
                double a = 0;
                for (int d = 0; d < DH; ++d) a += (double)hq[(p * G + r) * DH + d] * kr[d];
                sc[i] = a / sqrt(128.0);
                mx = std::max(mx, sc[i]);
            }
            double tot = 0;
            for (int i = 0; i < SEL; ++i) { sc[i] = exp(sc[i] - mx); tot += sc[i]; }
            for (int i = 0; i < SEL; ++i) {
                const float* vr = &hv[((size_t)p * S + rows[(size_t)p * SEL + i]) * DH];
                for (int d = 0; d < DH; ++d) ref[(p * G + r) * DH + d] += sc[i] / tot * vr[d];
            }
        }
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const double bytes = (double)P * SEL * DH * 8;
    auto run = [&](const char* name, int n_parts, auto launch) {
        for (int i = 0; i < 3; ++i) launch();
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        for (int i = 0; i < 20; ++i) launch();
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 20;
        merge<<<P * G, DH>>>(part, n_parts, out);
        std::vector<float> ho(2 * G * DH);
        CK(cudaMemcpy(ho.data(), out, ho.size() * 4, cudaMemcpyDeviceToHost));
        double num = 0, den = 0;
        for (size_t i = 0; i < ho.size(); ++i) { num = std::max(num, fabs(ho[i] - ref[i])); den = std::max(den, fabs(ref[i])); }
        printf("%-46s %8.1f us  %7.0f GB/s  rel err %.2e\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9, num / den);
    };
    for (int per : {205, 410}) {
        const int nc = (SEL + per - 1) / per;
        dim3 grid(nc, P);
        char nm[128];
        CK(cudaFuncSetAttribute(gqa_h, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
        snprintf(nm, sizeof nm, "H half-warp cp.async ring4 rows/CTA=%d", per);
        run(nm, nc * 16, [&] { gqa_h<<<grid, 256, 64 * 1024>>>(K, V, drows, per, Q, sl, part); });
        auto runw = [&](auto kern, int D, const char* tag) {
            const int smem = 8 * D * 1024 + 8 * D * 8;
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            snprintf(nm, sizeof nm, "%s D=%d rows/CTA=%d", tag, D, per);
            run(nm, nc * 8, [&] { kern<<<grid, 256, smem>>>(K, V, drows, per, Q, sl, part); });
        };
        runw(gqa_w<4, 4>, 4, "W bulk-copy ring minB4");
        runw(gqa_w<8, 3>, 8, "W bulk-copy ring minB3");
        runw(gqa_w<6, 4>, 6, "W bulk-copy ring minB4");
        runw(gqa_w2<4, 4>, 4, "W2 cp.async minB4");
        runw(gqa_w2p<4, 4>, 4, "W2P packed minB4");
        runw(gqa_w2p<4, 5>, 4, "W2P packed minB5");
    }
    {
        char nm[128];
        auto rund = [&](auto kern, int nw, int per_head, const char* tag, int d = 4) {
            const int per = (SEL + per_head - 1) / per_head;
            const int smem = nw * d * 1024;
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            snprintf(nm, sizeof nm, "%s CTAs/head=%d rows/CTA=%d", tag, per_head, per);
            dim3 grid(per_head, P);
            run(nm, per_head * nw, [&] { kern<<<grid, nw * 32, smem>>>(K, V, drows, per, Q, sl, part); });
        };
        rund(gqa_w2d<4, 32, 2>, 32, 18, "W2D 32 warps CB2");
        rund(gqa_w2d<4, 32, 4>, 32, 18, "W2D 32 warps CB4");
        rund(gqa_w2d<4, 16, 2>, 16, 37, "W2D 16 warps CB2");
        rund(gqa_w2d<4, 8, 2>, 8, 74, "W2D 8 warps CB2");
        rund(gqa_w2d<4, 8, 2>, 8, 64, "W2D 8 warps CB2");
        rund(gqa_w2d<6, 32, 4>, 32, 18, "W2D D6 32 warps CB4", 6);
        rund(gqa_w2d<4, 32, 4>, 32, 16, "W2D 32 warps CB4", 4);
        rund(gqa_w2d<4, 32, 8>, 32, 18, "W2D 32 warps CB8", 4);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
