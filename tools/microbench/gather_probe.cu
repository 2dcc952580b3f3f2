// Microbenchmark: achievable HBM bandwidth for the decode gather pattern on
// B200 -- 20% of 512 B K rows + 512 B V rows per head, row ids sorted -- vs a
// streaming read of the same byte count.  Variants: rows in flight per 8-lane
// group (RPI), K/V separate vs interleaved (one 1 KB row per token), CTAs per
// SM.  Sets the ceiling the attention kernel is measured against.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int H = 32, S = 131072, DH = 128, SEL = 26282;

template <int RPI, bool INTERLEAVED>
__global__ void __launch_bounds__(256) gather(const float* __restrict__ k, const float* __restrict__ v,
                                              const int* __restrict__ rows, int per_cta, float* out) {
    int p = blockIdx.y, c = blockIdx.x;
    int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, grp = lane >> 3, gl = lane & 7;
    const int* r = rows + (size_t)p * SEL + (size_t)c * per_cta;
    int n = min(per_cta, SEL - c * per_cta);
    float acc = 0.f;
    const int slot = warp * 4 + grp, stride = 32 * RPI;
    for (int base = 0; base < n; base += stride) {
        float4 kr[RPI][4], vr[RPI][4];
#pragma unroll
        for (int u = 0; u < RPI; ++u) {
            int ri = base + u * 32 + slot;
            int row = r[ri < n ? ri : 0];
            const float4* kp; const float4* vp;
            if (INTERLEAVED) {
                kp = reinterpret_cast<const float4*>(k + ((size_t)p * S + row) * 2 * DH);
                vp = kp + 32;
            } else {
                kp = reinterpret_cast<const float4*>(k + ((size_t)p * S + row) * DH);
                vp = reinterpret_cast<const float4*>(v + ((size_t)p * S + row) * DH);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) { kr[u][j] = __ldg(kp + j * 8 + gl); vr[u][j] = __ldg(vp + j * 8 + gl); }
        }
#pragma unroll
        for (int u = 0; u < RPI; ++u)
#pragma unroll
            for (int j = 0; j < 4; ++j)
                acc += kr[u][j].x + kr[u][j].y + vr[u][j].z + vr[u][j].w;
    }
    if (acc == 1234.5f) out[0] = acc;
}

__global__ void stream(const float4* __restrict__ a, size_t n, float* out) {
    float acc = 0.f;
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        float4 x = __ldg(a + i);
        acc += x.x + x.w;
    }
    if (acc == 1234.5f) out[0] = acc;
}

int main() {
    size_t kv = (size_t)H * S * DH;
    float *k, *v, *kvi, *out;
    CK(cudaMalloc(&k, kv * 4)); CK(cudaMalloc(&v, kv * 4)); CK(cudaMalloc(&kvi, kv * 8)); CK(cudaMalloc(&out, 64));
    CK(cudaMemset(k, 0, kv * 4)); CK(cudaMemset(v, 0, kv * 4)); CK(cudaMemset(kvi, 0, kv * 8));
    std::vector<int> rows((size_t)H * SEL);
    std::mt19937 rng(1);
    std::vector<int> all(S);
    for (int p = 0; p < H; ++p) {
        for (int i = 0; i < S; ++i) all[i] = i;
        std::shuffle(all.begin(), all.end(), rng);
        std::sort(all.begin(), all.begin() + SEL);
        std::copy(all.begin(), all.begin() + SEL, rows.begin() + (size_t)p * SEL);
    }
    int* drows;
    CK(cudaMalloc(&drows, rows.size() * 4));
    CK(cudaMemcpy(drows, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice));
    double bytes = (double)H * SEL * DH * 4 * 2;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](const char* name, auto launch) {
        for (int i = 0; i < 3; ++i) launch();
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        for (int i = 0; i < 10; ++i) launch();
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 10;
        printf("%-44s %8.1f us  %7.0f GB/s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
    };
    for (int per : {820, 1640, 3280}) {
        dim3 grid((SEL + per - 1) / per, H);
        char nm[128];
        snprintf(nm, sizeof nm, "separate  RPI=1 rows/CTA=%d", per); run(nm, [&] { gather<1, false><<<grid, 256>>>(k, v, drows, per, out); });
        snprintf(nm, sizeof nm, "separate  RPI=2 rows/CTA=%d", per); run(nm, [&] { gather<2, false><<<grid, 256>>>(k, v, drows, per, out); });
        snprintf(nm, sizeof nm, "separate  RPI=4 rows/CTA=%d", per); run(nm, [&] { gather<4, false><<<grid, 256>>>(k, v, drows, per, out); });
        snprintf(nm, sizeof nm, "interleave RPI=1 rows/CTA=%d", per); run(nm, [&] { gather<1, true><<<grid, 256>>>(kvi, nullptr, drows, per, out); });
        snprintf(nm, sizeof nm, "interleave RPI=2 rows/CTA=%d", per); run(nm, [&] { gather<2, true><<<grid, 256>>>(kvi, nullptr, drows, per, out); });
        snprintf(nm, sizeof nm, "interleave RPI=4 rows/CTA=%d", per); run(nm, [&] { gather<4, true><<<grid, 256>>>(kvi, nullptr, drows, per, out); });
    }
    size_t n4 = (size_t)(bytes / 16);
    run("stream same bytes (grid 148x8)", [&] { stream<<<148 * 8, 256>>>(reinterpret_cast<const float4*>(k), n4, out); });
    run("stream same bytes (grid 148x16)", [&] { stream<<<148 * 16, 256>>>(reinterpret_cast<const float4*>(k), n4, out); });
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
