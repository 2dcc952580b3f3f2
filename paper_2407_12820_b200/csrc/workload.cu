// workload.cu -- device-side synthetic KV workloads.
//
// The reference's gen_workload (workload.cpp:16-117) draws one sequential
// mt19937_64 stream on the host, which takes minutes for 128K x 32-layer
// inputs.  This kernel draws the SAME DISTRIBUTIONS from a counter-based
// generator (every value is a pure function of (seed, head, token, dim)),
// so a layer is generated in HBM at memory speed and any slice can be
// regenerated independently:
//   gaussian mixture (workload.cpp:39-51): n_components means ~ N(0,1)^d per
//     head, token -> uniform component, key = mean + spread * N(0,1);
//     values, queries ~ N(0,1).
//   powerlaw (workload.cpp:53-79): a unit query direction q per head, a
//     uniformly random rank per token (a bijective permutation of [0, s)),
//     key = u + (A*sqrt(d)/(rank+1)^a - u.q) q with u a random unit vector,
//     so the scaled exact score of rank r is A / (r+1)^a (A = 8); values
//     ~ N(0,1); every query row = q.
// Parity with the reference is distributional, not bitwise (the reference
// values themselves come from its host generator via the oracle in tests).
#include <cmath>

#include "internal.cuh"

namespace pqkv_dev {
namespace {

constexpr int WL_THREADS = 256;
constexpr double kTopScore = 8.0;  // kPowerlawTopScore, workload.cpp:16

__device__ __forceinline__ uint64_t mix64(uint64_t z) {  // splitmix64 finaliser
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// Stream id -> independent 64-bit counter space.
__device__ __forceinline__ uint64_t ctr(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b) {
    return mix64(mix64(mix64(seed ^ (stream * 0xd1b54a32d192ed03ull)) + a) + b);
}

__device__ __forceinline__ double uniform01(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }

// Standard normal from one counter (Box-Muller on two derived uniforms).
__device__ __forceinline__ double normal(uint64_t c) {
    const double u1 = uniform01(mix64(c)) + 0x1.0p-54;  // (0, 1]
    const double u2 = uniform01(mix64(c ^ 0x5851f42d4c957f2dull));
    return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}

// Bijective permutation of [0, n): a 4-round Feistel network on the
// enclosing power-of-two domain, cycle-walking out-of-range values.
__device__ uint32_t permute(uint32_t i, uint32_t n, uint64_t key) {
    int bits = 2;
    while ((1u << bits) < n) ++bits;
    bits += bits & 1;
    const int half = bits / 2;
    const uint32_t mask = (1u << half) - 1u;
    uint32_t x = i;
    do {
        uint32_t l = x >> half, r = x & mask;
        for (int rd = 0; rd < 4; ++rd) {
            const uint32_t f = (uint32_t)mix64(key + ((uint64_t)rd << 40) + r) & mask;
            const uint32_t t = r;
            r = l ^ f;
            l = t;
        }
        x = (l << half) | r;
    } while (x >= n);
    return x;
}

struct WlArgs {
    int kind, s, d, g, n_comp;
    double spread, zipf;
    uint64_t seed;
    float* keys;     // [h][s][d]
    float* values;   // [h][s][d]
    float* queries;  // [h][g][d]
};

// Head direction q (powerlaw) into shared memory, normalised in fp64.
__device__ void head_direction(const WlArgs& a, int h, double* q, double* red) {
    const int tid = threadIdx.x;
    double part = 0.0;
    for (int j = tid; j < a.d; j += WL_THREADS) {
        q[j] = normal(ctr(a.seed, 1, h, j));
        part += q[j] * q[j];
    }
    red[tid] = part;
    __syncthreads();
    if (tid == 0) {
        double n2 = 0.0;
        for (int t = 0; t < WL_THREADS; ++t) n2 += red[t];
        red[0] = 1.0 / sqrt(n2 > 0.0 ? n2 : 1.0);
    }
    __syncthreads();
    const double inv = red[0];
    __syncthreads();
    for (int j = tid; j < a.d; j += WL_THREADS) q[j] *= inv;
    __syncthreads();
}

// grid: (token blocks, heads); one warp per token row.
__global__ void __launch_bounds__(WL_THREADS) workload_kernel(WlArgs a) {
    extern __shared__ double wl_smem[];
    double* q = wl_smem;                 // [d] (powerlaw)
    double* red = wl_smem + a.d;         // [WL_THREADS]
    const int h = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long hs = (long long)h * a.s * a.d;
    if (a.kind == PQKV_WORKLOAD_POWERLAW) head_direction(a, h, q, red);
    const int rows_per_block = WL_THREADS / 32;
    for (int i = blockIdx.x * rows_per_block + warp; i < a.s; i += gridDim.x * rows_per_block) {
        float* krow = a.keys + hs + (long long)i * a.d;
        float* vrow = a.values + hs + (long long)i * a.d;
        if (a.kind == PQKV_WORKLOAD_GAUSSIAN) {
            const int comp = (int)(uniform01(ctr(a.seed, 2, h, i)) * a.n_comp);
            for (int j = lane; j < a.d; j += 32) {
                const double mean = normal(ctr(a.seed, 3, (uint64_t)h * a.n_comp + comp, j));
                krow[j] = (float)(mean + a.spread * normal(ctr(a.seed, 4, (uint64_t)h * a.s + i, j)));
            }
        } else {
            // u = random unit vector; key = u + (target - u.q) q
            double n2 = 0.0, along = 0.0;
            for (int j = lane; j < a.d; j += 32) {
                const double u = normal(ctr(a.seed, 5, (uint64_t)h * a.s + i, j));
                n2 += u * u;
                along += u * q[j];
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                n2 += __shfl_xor_sync(FULL, n2, o);
                along += __shfl_xor_sync(FULL, along, o);
            }
            const double inv = 1.0 / sqrt(n2 > 0.0 ? n2 : 1.0);
            along *= inv;
            const uint32_t rank = permute((uint32_t)i, (uint32_t)a.s, a.seed * 0x2545f4914f6cdd1dull + h);
            const double target = kTopScore * sqrt((double)a.d) / pow((double)rank + 1.0, a.zipf);
            for (int j = lane; j < a.d; j += 32) {
                const double u = normal(ctr(a.seed, 5, (uint64_t)h * a.s + i, j)) * inv;
                krow[j] = (float)(u + (target - along) * q[j]);
            }
        }
        for (int j = lane; j < a.d; j += 32) vrow[j] = (float)normal(ctr(a.seed, 6, (uint64_t)h * a.s + i, j));
    }
    if (blockIdx.x == 0) {
        for (int e = tid; e < a.g * a.d; e += WL_THREADS) {
            const int j = e % a.d;
            a.queries[(long long)h * a.g * a.d + e] =
                a.kind == PQKV_WORKLOAD_POWERLAW ? (float)q[j] : (float)normal(ctr(a.seed, 7, h, e));
        }
    }
}

}  // namespace

void launch_workload(pqkv_ctx* ctx, int kind, size_t s, size_t d, size_t h, size_t g, size_t n_comp,
                     double spread, double zipf, uint64_t seed, float* keys, float* values, float* queries,
                     cudaStream_t st) {
    bind_device(ctx);
    if (s == 0 || d == 0 || h == 0 || g == 0) fail(PQKV_EINVAL, "workload: s, d_h, h_kv, g must all be >= 1");
    if (kind != PQKV_WORKLOAD_GAUSSIAN && kind != PQKV_WORKLOAD_POWERLAW) fail(PQKV_EINVAL, "workload: unknown kind");
    if (kind == PQKV_WORKLOAD_GAUSSIAN && n_comp < 1) fail(PQKV_EINVAL, "workload: n_components must be >= 1");
    if (spread < 0.0) fail(PQKV_EINVAL, "workload: spread must be >= 0");
    if (!(zipf > 0.0)) fail(PQKV_EINVAL, "workload: zipf_exponent must be > 0");
    if (s > 0x7fffffff || d > 4096) fail(PQKV_EINVAL, "workload: shape too large");
    WlArgs a{};
    a.kind = kind;
    a.s = (int)s;
    a.d = (int)d;
    a.g = (int)g;
    a.n_comp = (int)n_comp;
    a.spread = spread;
    a.zipf = zipf;
    a.seed = seed;
    a.keys = keys;
    a.values = values;
    a.queries = queries;
    const unsigned bx = (unsigned)std::min<size_t>(ceil_div(s, WL_THREADS / 32),
                                                   std::max<size_t>(1, 8 * (size_t)ctx->sm_count / h + 1));
    const size_t smem = (d + WL_THREADS) * sizeof(double);
    workload_kernel<<<dim3(bx, (unsigned)h), WL_THREADS, smem, st>>>(a);
    PQKV_LAUNCHED("workload_kernel");
}

}  // namespace pqkv_dev
