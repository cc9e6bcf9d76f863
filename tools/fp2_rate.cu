// fp2_rate.cu -- issue rate of the packed-FP32 instructions the single pass is
// made of (FMUL2, FADD2, FFMA2 with a register "one" -- the kernels' add -- and
// scalar FFMA / FADD / FMUL), measured as warp-instructions per cycle per SM.
// Each thread runs NCH independent chains so latency is hidden.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/fp2_rate.cu -o tools/_fp2_rate
#include <cuda_runtime.h>

#include <cstdio>

constexpr int NCH = 8;
constexpr int ITERS = 4096;

template <int OP>
__global__ void rate_kernel(float* out, float a0, float b0, long long* cycles) {
    unsigned long long x[NCH], y[NCH];
    float s[NCH];
    const float2 b2 = make_float2(b0, b0 * 0.5f);
    unsigned long long bb;
    asm volatile("mov.b64 %0, {%1, %2};" : "=l"(bb) : "f"(b2.x), "f"(b2.y));
    unsigned long long one;
    asm volatile("mov.b64 %0, {%1, %1};" : "=l"(one) : "f"(a0 * 0.0f + 1.0f));
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
        const float v = a0 + i + threadIdx.x;
        asm volatile("mov.b64 %0, {%1, %1};" : "=l"(x[i]) : "f"(v));
        y[i] = x[i];
        s[i] = v;
    }
    const long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
            if (OP == 0) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(x[i]) : "l"(bb));
            if (OP == 1) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(x[i]) : "l"(bb));
            if (OP == 2) asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(x[i]) : "l"(y[i]), "l"(one));
            if (OP == 3) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(s[i]) : "f"(b0), "f"(a0));
            if (OP == 4) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(s[i]) : "f"(b0));
            if (OP == 5) asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(s[i]) : "f"(b0));
            if (OP == 6) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(bb), "l"(y[i]));
        }
    }
    const long long t1 = clock64();
    float acc = 0;
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
        float lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x[i]));
        acc += lo + hi + s[i];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int OP>
static void run(const char* name, int warps_per_sm) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int threads = 32 * warps_per_sm;
    float* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(float) * sms * threads);
    cudaMalloc(&cyc, sizeof(long long) * sms);
    rate_kernel<OP><<<sms, threads>>>(out, 1.0f, 0.999f, cyc);
    cudaDeviceSynchronize();
    rate_kernel<OP><<<sms, threads>>>(out, 1.0f, 0.999f, cyc);
    cudaDeviceSynchronize();
    long long c = 0;
    cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    const double instr = (double)warps_per_sm * ITERS * NCH;  // warp-instructions per SM
    std::printf("%-32s warps/SM %2d: %.3f warp-instr/cycle/SM (%.2f cycles per instr per SMSP)\n", name,
                warps_per_sm, instr / c, 4.0 * c / instr);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    for (int w : {16, 32}) {
        run<0>("mul.rn.f32x2 (FMUL2)", w);
        run<1>("add.rn.f32x2 (FADD2?)", w);
        run<2>("fma.rn.f32x2 x,one,acc (FFMA2)", w);
        run<6>("fma.rn.f32x2 x,w,y (FFMA2)", w);
        run<3>("fma.rn.f32 (FFMA 3-reg)", w);
        run<4>("add.rn.f32 (FADD)", w);
        run<5>("mul.rn.f32 (FMUL)", w);
    }
    return 0;
}
