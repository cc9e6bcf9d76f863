// fp32_burn.cu -- a sustained FP32-pipe load with the single pass's instruction
// mix (FMUL2 product + FFMA2 x*one+acc add, i.e. mul then add, never fused), to
// measure the FP32 rate the B200 holds under its power cap (dev tool; driven by
// tools/fp32_sustained.py). Build:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC \
//        tools/fp32_burn.cu -o tools/_fp32_burn.so
#include <cuda_runtime.h>

constexpr int NCH = 8;

__global__ void __launch_bounds__(256) burn_kernel(float* out, float a0, float b0, int iters) {
    unsigned long long x[NCH], acc[NCH];
    unsigned long long bb, one;
    asm volatile("mov.b64 %0, {%1, %2};" : "=l"(bb) : "f"(b0), "f"(b0 * 0.5f));
    asm volatile("mov.b64 %0, {%1, %1};" : "=l"(one) : "f"(a0 * 0.0f + 1.0f));
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
        const float v = a0 + i + threadIdx.x;
        asm volatile("mov.b64 %0, {%1, %1};" : "=l"(x[i]) : "f"(v));
        acc[i] = x[i];
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
            unsigned long long p;
            asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(p) : "l"(x[i]), "l"(bb));
            asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[i]) : "l"(p), "l"(one));
            x[i] = p;
        }
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
        float lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[i]));
        s += lo + hi;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// lane-ops per launch = blocks * 256 threads * iters * NCH * 2 instructions * 2 lanes
extern "C" int fp32_burn(float* out, int blocks, int iters, void* stream) {
    burn_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(out, 1.0f, 0.9999999f, iters);
    return (int)cudaGetLastError();
}
