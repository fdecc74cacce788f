// How fast is cudaHostRegister / Unregister of a pageable buffer (the C++
// drop-in's std::vector arguments) compared with pageable and pinned copies?
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>
int main() {
    const size_t n = 68446312 / 4 * 4;  // C3 values
    std::vector<float> h(n / 4, 1.0f), o(n / 4);
    float* d; cudaMalloc(&d, n);
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    for (int it = 0; it < 3; ++it) {
        auto t0 = now();
        cudaMemcpy(d, h.data(), n, cudaMemcpyHostToDevice);
        auto t1 = now();
        cudaHostRegister(h.data(), n, cudaHostRegisterDefault);
        auto t2 = now();
        cudaMemcpy(d, h.data(), n, cudaMemcpyHostToDevice);
        auto t3 = now();
        cudaHostUnregister(h.data());
        auto t4 = now();
        cudaHostRegister(o.data(), n, cudaHostRegisterDefault);
        cudaMemcpy(o.data(), d, n, cudaMemcpyDeviceToHost);
        cudaHostUnregister(o.data());
        auto t5 = now();
        printf("pageable H2D %.2f ms | register %.2f ms | pinned H2D %.2f ms | unregister %.2f ms | reg+D2H+unreg %.2f ms\n",
               ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4), ms(t4, t5));
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
