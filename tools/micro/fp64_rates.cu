// Microbenchmark: per-SM throughput of DFMA, F2F.F64.F32 (float -> double)
// and an integer float->double bit conversion on B200.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters) {
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double b = 1.0000001, c = 1e-9;
    for (int i = 0; i < iters; ++i) {
        a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
        a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void k_f2f(double* out, int iters) {
    float f[8];
    for (int k = 0; k < 8; ++k) f[k] = threadIdx.x + k;
    double s0 = 0, s1 = 0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            double d = static_cast<double>(f[k]);
            f[k] = __uint_as_float(__float_as_uint(f[k]) ^ 1u);  // keep it live, int op
            if (k & 1) s1 += d; else s0 += d;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1;
}
__global__ void k_f2f_only(double* out, int iters) {
    float f[8];
    for (int k = 0; k < 8; ++k) f[k] = threadIdx.x + k;
    unsigned long long x = 0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            double d = static_cast<double>(f[k]);
            x ^= __double_as_longlong(d);
            f[k] = __uint_as_float(__float_as_uint(f[k]) + 1u);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = __longlong_as_double(x);
}
int main() {
    double* out; cudaMalloc(&out, 148 * 8 * 256 * 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 20000, blocks = 148 * 8, threads = 256;
    auto t = [&](auto kern, const char* name, double ops_per_iter) {
        kern<<<blocks, threads>>>(out, 10);
        cudaEventRecord(e0);
        kern<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double ops = double(blocks) * threads * iters * ops_per_iter;
        printf("%-12s %.3f ms  %.1f ops/clk/SM (at 1.965 GHz)\n", name, ms, ops / (ms * 1e-3) / 148 / 1.965e9);
    };
    t(k_dfma, "dfma", 8);
    t(k_f2f, "f2f+dadd", 8);
    t(k_f2f_only, "f2f+xor", 8);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
