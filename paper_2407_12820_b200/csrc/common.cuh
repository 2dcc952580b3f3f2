// common.cuh -- shared helpers for the pqkv sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "pqkv_c.h"

namespace pqkv_dev {

// ---- host-side status plumbing ---------------------------------------------

struct Status {
    int code;
    std::string msg;
};

// Thrown inside the C-ABI implementation, converted to a status at the
// boundary (ctx.cu: pqkv_guard).
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& m) { throw Error(code, m); }

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(PQKV_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define PQKV_CUDA(x) ::pqkv_dev::cuda_check((x), #x)
#define PQKV_LAUNCHED(name) ::pqkv_dev::cuda_check(cudaGetLastError(), name)

inline size_t ceil_div(size_t a, size_t b) { return (a + b - 1) / b; }
inline size_t round_up(size_t a, size_t b) { return ceil_div(a, b) * b; }

// ---- device helpers ---------------------------------------------------------

constexpr unsigned FULL = 0xffffffffu;

// Order-preserving map float -> u32 (larger score -> larger key), with -0.0
// folded onto +0.0 because the reference compares scores with float `!=`
// and `>` (topk.cpp:17-22), under which the two zeros are equal.
__device__ __forceinline__ uint32_t score_key(float f) {
    if (f == 0.0f) f = 0.0f;
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

}  // namespace pqkv_dev
