// Microbenchmark: gathering a tile's source runs into shared memory with
// (a) one 4-byte cp.async per element (the r01 map kernel's gather) vs
// (b) one cp.async.bulk per run (16-byte aligned superset), on B200.
// Each CTA stages NRUN runs of LEN floats from a 64M-float array; runs are
// consecutive-ish (like a tile's source rows) within a random window.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>
#include <random>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

template <int NRUN, int LEN>
__global__ void __launch_bounds__(128, 8) k_ldgsts(const float* __restrict__ src, const uint32_t* __restrict__ run_begin, float* out) {
    __shared__ __align__(16) float F[NRUN * (LEN + 8)];
    const uint32_t* rb = run_begin + blockIdx.x * NRUN;
    for (int q = threadIdx.x; q < NRUN * LEN; q += 128) {
        const int r = q / LEN, e = q - r * LEN;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(F + q)), "l"(src + __ldg(rb + r) + e) : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    float s = 0;
    for (int q = threadIdx.x; q < NRUN * LEN; q += 128) s += F[q];
    if (s == 12345.0f) out[blockIdx.x] = s;
}

template <int NRUN, int LEN>
__global__ void __launch_bounds__(128, 8) k_bulk(const float* __restrict__ src, const uint32_t* __restrict__ run_begin, float* out) {
    __shared__ __align__(16) float F[NRUN * (LEN + 8)];
    __shared__ __align__(8) uint64_t bar;
    const uint32_t* rb = run_begin + blockIdx.x * NRUN;
    constexpr int SLOT = ((LEN + 3 + 3) / 4) * 4;  // aligned superset slot (floats)
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t bytes_total = 0;
    for (int r = threadIdx.x; r < NRUN; r += 128) {
        const uint32_t b = __ldg(rb + r);
        const uint32_t a0 = b & ~3u, a1 = (b + LEN + 3) & ~3u;
        const uint32_t nb = (a1 - a0) * 4;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(F + r * SLOT)), "l"(src + a0), "r"(nb), "r"(smem_u32(&bar)) : "memory");
        bytes_total += nb;
    }
    // expect_tx: total bytes (sum over threads)
    for (int o = 16; o > 0; o >>= 1) bytes_total += __shfl_xor_sync(~0u, bytes_total, o);
    __shared__ uint32_t wsum[4];
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = bytes_total;
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t tot = wsum[0] + wsum[1] + wsum[2] + wsum[3];
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(tot) : "memory");
    }
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(smem_u32(&bar)), "r"(0) : "memory");
    float s = 0;
    for (int q = threadIdx.x; q < NRUN * SLOT; q += 128) s += F[q];
    if (s == 12345.0f) out[blockIdx.x] = s;
}

template <int NRUN, int LEN>
void run(const float* src, size_t n, int ctas) {
    std::vector<uint32_t> h(static_cast<size_t>(ctas) * NRUN);
    std::mt19937 g(1);
    for (int c = 0; c < ctas; ++c) {
        uint32_t base = g() % (n - 100000);
        for (int r = 0; r < NRUN; ++r) { base += LEN + (g() % 200); h[c * NRUN + r] = base % (n - 64); }
    }
    uint32_t* d; float* out;
    cudaMalloc(&d, 4 * h.size()); cudaMalloc(&out, 4 * ctas);
    cudaMemcpy(d, h.data(), 4 * h.size(), cudaMemcpyHostToDevice);
    float* flush; cudaMalloc(&flush, 256 << 20);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int mode = 0; mode < 2; ++mode) {
        float best = 1e9;
        for (int it = 0; it < 6; ++it) {
            cudaMemsetAsync(flush, it, 256 << 20);
            cudaEventRecord(e0);
            if (mode == 0) k_ldgsts<NRUN, LEN><<<ctas, 128>>>(src, d, out); else k_bulk<NRUN, LEN><<<ctas, 128>>>(src, d, out);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); if (it) best = ms < best ? ms : best;
        }
        const double bytes = double(ctas) * NRUN * LEN * 4;
        printf("NRUN=%d LEN=%d %s: %.1f us  (%.0f GB/s useful, %.1f M copies/s/SM)\n", NRUN, LEN, mode ? "bulk" : "ldgsts", best * 1e3,
               bytes / best / 1e6, double(ctas) * NRUN / (best * 1e-3) / 148 / 1e6);
    }
    cudaFree(d); cudaFree(out); cudaFree(flush);
}

int main() {
    const size_t n = 64u << 20;
    float* src; cudaMalloc(&src, 4 * n); cudaMemset(src, 0, 4 * n);
    run<150, 12>(src, n, 34700);
    run<150, 8>(src, n, 34700);
    run<100, 20>(src, n, 34700);
    run<60, 32>(src, n, 34700);
    cudaError_t e = cudaGetLastError();
    printf("err: %s\n", cudaGetErrorString(e));
}
