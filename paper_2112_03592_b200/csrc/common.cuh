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

// Both lower bounds (of k0 <= k1) in the sorted y[b, e) with 8-ary rounds:
// each round issues up to 7 independent loads per key and shrinks the
// interval 8x, so a row of n particles costs ~log8(n) + 1 dependent load
// latencies instead of log2(n) (the tile kernels are latency-bound here).
__device__ __forceinline__ void lower_bound2_kary(const uint16_t* __restrict__ y, uint32_t b, uint32_t e, int k0,
                                                  int k1, uint32_t& s0, uint32_t& s1) {
    uint32_t l0 = b, r0 = e, l1 = b, r1 = e;
    while (r0 - l0 > 8 || r1 - l1 > 8) {
        const uint32_t st0 = (r0 - l0 + 7) >> 3, st1 = (r1 - l1 + 7) >> 3;
        const bool a0 = r0 - l0 > 8, a1 = r1 - l1 > 8;
        int j0 = 0, j1 = 0;
#pragma unroll
        for (int k = 1; k < 8; ++k) {
            const uint32_t p0 = l0 + k * st0, p1 = l1 + k * st1;
            const int v0 = (a0 && p0 < r0) ? static_cast<int>(__ldg(y + p0)) : 0x10000;
            const int v1 = (a1 && p1 < r1) ? static_cast<int>(__ldg(y + p1)) : 0x10000;
            j0 += v0 < k0;
            j1 += v1 < k1;
        }
        if (a0) {
            const uint32_t nl = j0 ? l0 + j0 * st0 + 1 : l0;
            r0 = min(l0 + (j0 + 1) * st0, r0);
            l0 = nl;
        }
        if (a1) {
            const uint32_t nl = j1 ? l1 + j1 * st1 + 1 : l1;
            r1 = min(l1 + (j1 + 1) * st1, r1);
            l1 = nl;
        }
    }
    uint32_t c0 = 0, c1 = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        c0 += (l0 + k < r0 && static_cast<int>(__ldg(y + l0 + k)) < k0);
        c1 += (l1 + k < r1 && static_cast<int>(__ldg(y + l1 + k)) < k1);
    }
    s0 = l0 + c0;
    s1 = l1 + c1;
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

// deconv.hpp:98-99: float(u / std::max<double>(blurred, eps)), blurred a float.
// When the denominator is the float itself, the fp64 quotient of two floats
// rounded to float equals their correctly rounded float quotient (double
// rounding is innocuous: 53 >= 2 * 24 + 2 bits), so the IEEE float division
// gives the reference's bits; the eps branch keeps the fp64 division.
__device__ __forceinline__ float rl_ratio(float u, float blurred, double eps) {
    const double bd = static_cast<double>(blurred);
    if (bd < eps) return __double2float_rn(__ddiv_rn(static_cast<double>(u), eps));
    return __fdiv_rn(u, blurred);
}

// ---- async copies (sm_90+ bulk copy with an mbarrier; sm_80+ cp.async) ----
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// one bulk global -> shared copy completing on bar (16-byte aligned, size a multiple of 16)
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// the same with an L2 eviction-priority policy (createpolicy: evict_first for
// data read once, evict_last for data neighbours re-read)
__device__ __forceinline__ void bulk_copy_hint(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                               uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t l2_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
            smem_u32(bar)),
        "r"(parity)
        : "memory");
}
}  // namespace aprgpu
