// Auxiliary kernels: region copy (copy_back) and the synthetic-input generator.
#include "kernels.cuh"
#include "launch.h"

namespace sc {

// ---------------------------------------------------------------------------
// Auxiliary kernels

// copy_back, S/conv.py:424-449: dst[region] := src[region], per plane.
static __global__ void copy_region_kernel(const float* __restrict__ src, float* __restrict__ dst, long long sps,
                                   long long dps, long long srs, long long drs, int nplanes, int row_lo, int nrows,
                                   int col_lo, int ncols) {
    const long long total = (long long)nplanes * nrows * ncols;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(i % ncols);
        const long long t = i / ncols;
        const int r = (int)(t % nrows);
        const int pl = (int)(t / nrows);
        const int y = row_lo + r, x = col_lo + c;
        dst[pl * dps + (long long)y * drs + x] = src[pl * sps + (long long)y * srs + x];
    }
}

// splitmix64 stream (S/image.py:131-141) mapped to float32 samples; counter-based.
static __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static __global__ void fill_synthetic_kernel(float* __restrict__ dst, long long count, uint64_t seed, uint64_t offset,
                                      int kind) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x) {
        const uint64_t top = mix64(seed + (offset + (uint64_t)i + 1ULL) * 0x9E3779B97F4A7C15ULL) >> 40;
        float v;
        if (kind == 0)
            v = __fmul_rn(__uint2float_rn((unsigned)top), 1.0f / 65536.0f);
        else if (kind == 1)
            v = __fmul_rn(__uint2float_rn((unsigned)top), 1.0f / 16777216.0f);
        else
            v = __fmul_rn(__uint2float_rn((unsigned)(top * 255ULL)), 1.0f / 16777216.0f);
        dst[i] = v;
    }
}


static int grid_for(long long total, int threads) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    long long blocks = (total + threads - 1) / threads;
    long long cap = (long long)sms * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    return (int)blocks;
}

cudaError_t launch_copy_region(const float* src, float* dst, long long sps, long long dps, long long srs,
                               long long drs, int nplanes, int row_lo, int nrows, int col_lo, int ncols,
                               cudaStream_t s) {
    const long long total = (long long)nplanes * nrows * ncols;
    if (total <= 0) return cudaSuccess;
    copy_region_kernel<<<grid_for(total, 256), 256, 0, s>>>(src, dst, sps, dps, srs, drs, nplanes, row_lo, nrows,
                                                             col_lo, ncols);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_fill_synthetic(float* dst, long long count, uint64_t seed, uint64_t offset, int kind,
                                  cudaStream_t s) {
    if (count <= 0) return cudaSuccess;
    fill_synthetic_kernel<<<grid_for(count, 256), 256, 0, s>>>(dst, count, seed, offset, kind);
    count_launch();
    return cudaGetLastError();
}

}  // namespace sc
