// Internal helpers shared by the libtsb translation units (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <functional>
#include <string>

#include "../../include/tsb.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "libtsb is written for sm_100a (B200) only"
#endif

namespace tsb {

constexpr uint64_t kGold = 0x9E3779B97F4A7C15ull;  // rng.py:22
constexpr uint64_t kM1 = 0xBF58476D1CE4E5B9ull;    // rng.py:37
constexpr uint64_t kM2 = 0x94D049BB133111EBull;    // rng.py:38
constexpr uint64_t kBaseXor = 0x6A09E667F3BCC909ull;  // rng.py:83, 144
constexpr uint64_t kCapacity = 1ull << 48;            // rng.py:23

// splitmix64 finaliser (rng.py:34-39, _kernels.py:23-27).
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * kM1;
    z = (z ^ (z >> 27)) * kM2;
    return z ^ (z >> 31);
}

// Per-family base key (rng.py:83).
__host__ __device__ __forceinline__ uint64_t family_base(uint64_t seed) {
    return mix64(seed ^ kBaseXor);
}

// Global-coin stream key: site (0,0), TAG_GLOBAL (rng.py:151-156).
__host__ __device__ __forceinline__ uint64_t global_key(uint64_t base) {
    return mix64(base + ((1ull << 48) + 1ull) * kGold);
}

// Draw of stream `key` at `step` (rng.py:53-54 with _splitmix_at(key, step)).
__host__ __device__ __forceinline__ uint64_t draw(uint64_t key, uint64_t step) {
    return mix64(key + (step + 1ull) * kGold);
}

// u < p  <=>  (x >> 11) < ceil(p * 2^53), exactly (rng.py:62-63).
inline uint64_t threshold_of(double p) {
    double x = p * 9007199254740992.0;  // exact power-of-two scaling
    if (!(x > 0.0)) return 0;           // p <= 0 or NaN: never accept
    if (x >= 9007199254740992.0) return 1ull << 53;
    double c = __builtin_ceil(x);
    return (uint64_t)c;
}

// Block-wide reduction (all threads get the result); sh holds one slot per warp.
template <typename T, typename Op>
__device__ T block_reduce(T v, Op op, T *sh) {
    for (int o = 16; o; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    v = sh[0];
    for (int i = 1; i < nw; ++i) v = op(v, sh[i]);
    return v;
}

// Block-wide exclusive prefix sum of one int per thread (sh: one slot per warp).
__device__ __forceinline__ int block_exclusive_sum(int v, int *sh) {
    int incl = v;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    __syncthreads();
    if (lane == 31) sh[wid] = incl;
    __syncthreads();
    int base = 0;
    for (int i = 0; i < wid; ++i) base += sh[i];
    return base + incl - v;
}

// host <-> device copies of caller grids through pinned staging (hostio.cu);
// d2h returns with the copy complete
int staged_h2d(void *dev, const void *src, size_t bytes, cudaStream_t stream);
int staged_d2h(void *dst, const void *dev, size_t bytes, cudaStream_t stream);
// fn(i) for i in [0, n) on the staging engine's host threads
void host_parallel_for(int n, const std::function<void(int)> &fn);

void set_error(const char *fmt, ...);
int fail(int code, const char *fmt, ...);
int cuda_fail(cudaError_t e, const char *what);
int ensure_device(int device);

}  // namespace tsb

#define TSB_CUDA(call)                                         \
    do {                                                       \
        cudaError_t _e = (call);                               \
        if (_e != cudaSuccess) return tsb::cuda_fail(_e, #call); \
    } while (0)
