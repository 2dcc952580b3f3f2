// dadd_probe -- dependent fp64 add chain latency on one warp (1 or 32 active
// lanes), operands from registers or shared memory.
#include <cstdio>
#include <cuda_runtime.h>

template <int LANES, bool SMEM>
__global__ void chain(const double* in, int n, double* out, long long* cyc) {
    __shared__ double buf[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = in[i];
    __syncthreads();
    if (threadIdx.x >= LANES) return;
    double acc = 0.0, a = in[threadIdx.x], b = in[threadIdx.x + 1];
    long long t0 = clock64();
    if (SMEM) {
        for (int i = 0; i < n; i += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = buf[(i + u) & 1023];
#pragma unroll
            for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, v[u]);
        }
    } else {
        for (int i = 0; i < n; i += 8) {
#pragma unroll
            for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, (u & 1) ? a : b);
        }
    }
    long long t1 = clock64();
    out[threadIdx.x] = acc;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    double *in, *out;
    long long* cyc;
    cudaMalloc(&in, 2048 * 8);
    cudaMalloc(&out, 64 * 8);
    cudaMallocManaged(&cyc, 8);
    cudaMemset(in, 0, 2048 * 8);
    const int n = 1 << 16;
#define RUN(L, S)                                                                     \
    chain<L, S><<<1, 32>>>(in, n, out, cyc);                                          \
    cudaDeviceSynchronize();                                                          \
    chain<L, S><<<1, 32>>>(in, n, out, cyc);                                          \
    cudaDeviceSynchronize();                                                          \
    printf("lanes=%d smem=%d: %.2f cycles/add\n", L, (int)S, (double)*cyc / n);
    RUN(1, false) RUN(32, false) RUN(1, true) RUN(32, true)
    return 0;
}
