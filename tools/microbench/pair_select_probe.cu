// Phase timing of pair_select (select_common.cuh) on inputs dumped from a
// real bench layer (tools/dump_pair_inputs.py): one CTA runs the select;
// per-phase clocks (PQKV_T marks 0..6), per-pass clocks and survivor counts
// (PQKV_PASS_STAMPS).  Usage: pair_select_probe DUMPDIR
#define PQKV_PASS_STAMPS 1
#ifndef PROBE_NT
#define PROBE_NT 256
#endif
#ifndef PROBE_MINB
#define PROBE_MINB 1
#endif
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>
#include <cuda_runtime.h>
#include "select_common.cuh"
__device__ unsigned long long g_t[40];

using namespace pqkv_dev;

__global__ void __launch_bounds__(PROBE_NT, PROBE_MINB) probe(const float* q, int g, const float* cen, const uint32_t* thist, const uint16_t* chist,
                      int n_chunks, int k, uint32_t* res) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int C = 64;
    PairScratch ps(smem, C, n_chunks);
    __shared__ uint8_t cls[4096];
    for (int i = threadIdx.x; i < 40; i += blockDim.x) g_t[i] = 0;
    __syncthreads();
    const unsigned long long t0 = clock64();
    pair_select<PROBE_NT, 4096 / PROBE_NT>(q, g, 128, cen, C, thist, chist, n_chunks, k, ps.lut, ps.hist, ps.cnt, ps.lst, ps.ceq,
                         ps.wsum, ps.sh, cls, nullptr, g_t);
    if (threadIdx.x == 0) {
        g_t[20] = clock64() - t0;
        res[0] = ps.sh[3];
        res[1] = ps.sh[4];
        res[2] = ps.sh[5];
    }
}

template <typename T>
std::vector<T> load(const std::string& path, size_t n) {
    std::vector<T> v(n);
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f || std::fread(v.data(), sizeof(T), n, f) != n) { std::fprintf(stderr, "cannot read %s\n", path.c_str()); std::exit(1); }
    std::fclose(f);
    return v;
}

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : "gpurun_out/pairdump";
    int g = 1, nch = 32, k = 26214;
    FILE* m = std::fopen((dir + "/meta.txt").c_str(), "r");
    if (!m || std::fscanf(m, "%d %d %d", &g, &nch, &k) != 3) return 1;
    std::fclose(m);
    const int C = 64, C2 = C * C;
    auto q = load<float>(dir + "/q.f32", g * 128);
    auto cen = load<float>(dir + "/cen.f32", 2 * C * 64);
    auto th = load<uint32_t>(dir + "/thist.u32", C2);
    auto ch = load<uint16_t>(dir + "/chist.u16", (size_t)nch * C2);
    float *dq, *dc; uint32_t *dth, *dres; uint16_t* dch;
    cudaMalloc(&dq, q.size() * 4); cudaMalloc(&dc, cen.size() * 4); cudaMalloc(&dth, C2 * 4);
    cudaMalloc(&dch, ch.size() * 2); cudaMalloc(&dres, 16);
    cudaMemcpy(dq, q.data(), q.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dc, cen.data(), cen.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dth, th.data(), C2 * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dch, ch.data(), ch.size() * 2, cudaMemcpyHostToDevice);
    const size_t smem = pair_select_scratch(C, nch);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int nnz = 0;
    for (uint32_t v : th) nnz += v != 0;
    for (int rep = 0; rep < 3; ++rep) {
        probe<<<1, PROBE_NT, smem>>>(dq, g, dc, dth, dch, nch, k, dres);
        cudaDeviceSynchronize();
        unsigned long long t[40];
        uint32_t res[4];
        cudaMemcpyFromSymbol(t, g_t, sizeof(t));
        cudaMemcpy(res, dres, 12, cudaMemcpyDeviceToHost);
        const double f = 1.0 / 1965.0;
        std::printf("rep %d nnz %d total %.2f us | lut %.2f keys %.2f radix %.2f classify %.2f chist %.2f cstar %.2f |"
                    " passes:", rep, nnz, t[20] * f, (t[1] - t[0]) * f, (t[3] - t[1]) * f, (t[4] - t[3]) * f,
                    (t[5] - t[4]) * f, (t[6] - t[5]) * f, 0.0);
        for (int p = 0; p < 4 && t[8 + p]; ++p)
            std::printf(" [%d] +%.2f us (hist %.2f digit %.2f) items %llu", p, (t[8 + p] - t[3]) * f,
                        (t[21 + p] - t[8 + p]) * f, (t[25 + p] - t[21 + p]) * f, t[12 + p]);
        std::printf(" | c*=%u take=%u\n", res[0], res[1]);
    }
    std::printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
