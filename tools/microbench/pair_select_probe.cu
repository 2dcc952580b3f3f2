// Phase timing of pair_select (select_common.cuh) on realistic inputs:
// 32 heads, m2b6 (C=64), 128K middle rows, k=26214, random gaussian queries
// and centroids, multinomial pair histogram.  Each phase boundary records
// clock64() from thread 0.
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>
#include <cuda_runtime.h>
#include "select_common.cuh"
__device__ unsigned long long g_t[64][16];

using namespace pqkv_dev;

template <int NT>
__global__ void probe(const float* q, const float* cen, const uint32_t* thist, const uint16_t* chist, int n_chunks,
                      int k, uint8_t* cls_out) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int p = blockIdx.x, C = 64, C2 = C * C;
    PairScratch ps(smem, C, n_chunks);
    __shared__ uint8_t cls[4096];
    unsigned long long t0 = clock64();
    pair_select<NT, 16>(q + p * 128, 1, 128, cen + (size_t)p * 2 * C * 64, C, thist + (size_t)p * C2,
                        chist + (size_t)p * n_chunks * C2, n_chunks, k, ps.lut, ps.hist, ps.cnt, ps.lst, ps.ceq, ps.wsum, ps.sh,
                        cls, nullptr, ::g_t[p]);
    if (threadIdx.x == 0) {
        ::g_t[p][15] = clock64() - t0;
        cls_out[p] = (uint8_t)ps.sh[3];
    }
}

int main() {
    const int P = 32, C = 64, C2 = C * C, S = 131004, NCH = (S + 4095) / 4096, K = 26214;
    std::mt19937 rng(1);
    std::normal_distribution<float> nd;
    std::vector<float> q(P * 128), cen(P * 2 * C * 64);
    for (auto& x : q) x = nd(rng);
    for (auto& x : cen) x = nd(rng);
    std::vector<uint32_t> th(P * C2, 0);
    std::vector<uint16_t> ch((size_t)P * NCH * C2, 0);
    std::uniform_int_distribution<int> ud(0, C2 - 1);
    for (int p = 0; p < P; ++p)
        for (int i = 0; i < S; ++i) {
            int t = ud(rng) % 600;  // concentrated pairs, like real codes
            th[p * C2 + t]++;
            ch[((size_t)p * NCH + i / 4096) * C2 + t]++;
        }
    float *dq, *dc; uint32_t* dth; uint16_t* dch; uint8_t* dout;
    cudaMalloc(&dq, q.size() * 4); cudaMalloc(&dc, cen.size() * 4); cudaMalloc(&dth, th.size() * 4);
    cudaMalloc(&dch, ch.size() * 2); cudaMalloc(&dout, 64);
    cudaMemcpy(dq, q.data(), q.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dc, cen.data(), cen.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dth, th.data(), th.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dch, ch.data(), ch.size() * 2, cudaMemcpyHostToDevice);
    size_t smem = pair_select_scratch(C, NCH);
    cudaFuncSetAttribute(probe<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(probe<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int nt : {256, 1024}) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            if (nt == 256) probe<256><<<P, 256, smem>>>(dq, dc, dth, dch, NCH, K, dout);
            else probe<1024><<<P, 1024, smem>>>(dq, dc, dth, dch, NCH, K, dout);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            unsigned long long t[64][16];
            cudaMemcpyFromSymbol(t, ::g_t, sizeof(t));
            printf("NT=%d rep %d: kernel %.1f us; head0 phases (cycles):", nt, rep, ms * 1e3);
            for (int ph = 0; ph < 16; ++ph) if (t[0][ph]) printf(" [%d]=%llu", ph, t[0][ph]);
            printf("\n");
        }
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
