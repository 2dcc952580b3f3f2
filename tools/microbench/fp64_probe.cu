// Microbenchmark: FP64 pipe latency/throughput on the target B200 (sm_100a).
// Drives design decisions for the exact-order k-means (serial fp64 chains,
// separate DADD/DMUL without contraction) -- see DESIGN.md "build".
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain_dadd(double* out, double a, int n) {
  double acc = 0.0;
  for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, a * (double)(i & 7));
  out[0] = acc;
}
__global__ void chain_dadd_pure(double* out, const double* a, int n) {
  double acc = 0.0;
  double x = a[0];
#pragma unroll 16
  for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, x);
  out[0] = acc;
}
template <int ILP>
__global__ void tput_dop(double* out, double x, int n) {
  double acc[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) acc[k] = threadIdx.x + k;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
      double d = __dsub_rn(x, acc[k]);
      acc[k] = __dadd_rn(acc[k], __dmul_rn(d, d));
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += acc[k];
  if (s == 1234.5) out[0] = s;
}
template <int ILP>
__global__ void tput_cvt(double* out, const float* xs, int n) {
  float f[ILP];
  double acc[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) { f[k] = xs[threadIdx.x % 32 + k]; acc[k] = 0; }
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) { acc[k] = __dadd_rn(acc[k], (double)f[k]); f[k] += 1.0f; }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += acc[k];
  if (s == 1234.5) out[0] = s;
}
template <int ILP>
__global__ void tput_ffma(float* out, float x, int n) {
  float acc[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) acc[k] = threadIdx.x + k;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) acc[k] = fmaf(acc[k], x, 0.5f);
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += acc[k];
  if (s == 1234.5f) out[0] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("device %s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, clk);
  double* d; float* f; cudaMalloc(&d, 1024); cudaMalloc(&f, 4096);
  cudaMemset(d, 0, 1024); cudaMemset(f, 0, 4096);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  int n = 1 << 20;
  chain_dadd_pure<<<1, 1>>>(d, d, 1000); cudaDeviceSynchronize();
  cudaEventRecord(e0); chain_dadd_pure<<<1, 1>>>(d, d, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("serial DADD chain: %.3f ns/add (%.2f cycles at %.0f MHz)\n", ms * 1e6 / n, ms * 1e-3 / n * clk * 1e3, clk / 1e3);
  int sms = p.multiProcessorCount; int iters = 4096;
  tput_dop<8><<<sms * 4, 256>>>(d, 1.5, 16); cudaDeviceSynchronize();
  cudaEventRecord(e0); tput_dop<8><<<sms * 4, 256>>>(d, 1.5, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double ops = 3.0 * 8 * iters * (double)sms * 4 * 256;
  printf("DSUB+DMUL+DADD throughput: %.2f Tops/s (%.1f ops/clk/SM)\n", ops / ms / 1e9, ops / (ms * 1e-3) / (clk * 1e3) / sms);
  cudaEventRecord(e0); tput_cvt<8><<<sms * 4, 256>>>(d, f, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  ops = 1.0 * 8 * iters * (double)sms * 4 * 256;
  printf("F2F.F64.F32+DADD throughput: %.2f G pairs/s (%.1f pairs/clk/SM)\n", ops / ms / 1e6, ops / (ms * 1e-3) / (clk * 1e3) / sms);
  cudaEventRecord(e0); tput_ffma<8><<<sms * 4, 256>>>(f, 1.0001f, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  ops = 1.0 * 8 * iters * (double)sms * 4 * 256;
  printf("FFMA throughput: %.2f T/s (%.1f /clk/SM)\n", ops / ms / 1e9, ops / (ms * 1e-3) / (clk * 1e3) / sms);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
