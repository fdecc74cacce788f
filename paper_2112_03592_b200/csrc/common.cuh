// Device helpers shared by the kernels.
#pragma once

#include <cstdint>

#include "internal.cuh"

namespace aprgpu {

constexpr unsigned kFull = 0xffffffffu;

// reflect_index (reconstruct.hpp:17-25)
__device__ __forceinline__ int reflect_dev(int i, int n) {
    while (i < 0 || i >= n) i = (i < 0) ? (-i - 1) : (2 * n - 1 - i);
    return i;
}

// first position in y[b, e) with y >= key
__device__ __forceinline__ uint32_t lower_bound_u16(const uint16_t* __restrict__ y, uint32_t b, uint32_t e, int key) {
    uint32_t n = e - b;
    while (n > 0) {
        const uint32_t half = n >> 1;
        const uint32_t m = b + half;
        if (static_cast<int>(__ldg(y + m)) < key) {
            b = m + 1;
            n -= half + 1;
        } else {
            n = half;
        }
    }
    return b;
}

__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

__device__ __forceinline__ int warp_min(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(kFull, v, o));
    return v;
}

__device__ __forceinline__ int warp_max(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(kFull, v, o));
    return v;
}

// inclusive warp scan
__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(kFull, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

__host__ __device__ __forceinline__ int grid_dim_dev(int n, int l_max, int l) {
    const int s = 1 << (l_max - l);
    return (n + s - 1) / s;
}

}  // namespace aprgpu
