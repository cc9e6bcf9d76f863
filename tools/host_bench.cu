// Host cost per C-ABI call vs its CUDA runtime building blocks (dev tool).
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/host_bench.cu -Iinclude \
//        -Lpaper_1711_09791_b200 -lsepconv_b200 -Xlinker -rpath,'$ORIGIN/../paper_1711_09791_b200' -o tools/_host_bench
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
#include "sepconv_b200.h"

__global__ void empty_kernel(int* p) { if (p && threadIdx.x == 1024) *p = 0; }

__global__ void spin_kernel(long long cycles) {
    const long long t0 = clock64();
    while (clock64() - t0 < cycles) {}
}

static cudaStream_t g_s;

// host time per call with the stream blocked behind a spinning kernel, so the
// GPU's own execution time never throttles the enqueue rate
template <class F>
static double per_call_us(F f, int n = 400) {
    for (int i = 0; i < 50; ++i) f();
    cudaDeviceSynchronize();
    spin_kernel<<<1, 1, 0, g_s>>>(200000000LL);
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < n; ++i) f();
    auto t1 = std::chrono::steady_clock::now();
    cudaDeviceSynchronize();
    return std::chrono::duration<double, std::micro>(t1 - t0).count() / n;
}

int main() {
    const int R = 64, C = 1024;
    float *x, *y;
    cudaMalloc(&x, 3 * R * C * 4);
    cudaMalloc(&y, 3 * R * C * 4);
    float w[5] = {1.f / 16, 4.f / 16, 6.f / 16, 4.f / 16, 1.f / 16};
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    g_s = s;
    cudaPointerAttributes a;
    int dev;
    printf("{\"sc_two_pass_fused_f32\": %.2f", per_call_us([&] {
        sc_two_pass_fused_f32(x, y, 3, R, C, R * C, R * C, C, C, w, 5, 0, s);
    }));
    printf(", \"cudaLaunchKernel_empty\": %.2f", per_call_us([&] { empty_kernel<<<592, 160, 0, s>>>(nullptr); }));
    printf(", \"cudaPointerGetAttributes\": %.2f", per_call_us([&] { cudaPointerGetAttributes(&a, x); }));
    printf(", \"cudaGetDevice\": %.2f", per_call_us([&] { cudaGetDevice(&dev); }));
    printf(", \"cudaSetDevice\": %.2f}\n", per_call_us([&] { cudaSetDevice(0); }));
    return 0;
}
