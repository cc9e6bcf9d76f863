// Auxiliary kernels: region copy (copy_back) and the synthetic-input generator.
#include "kernels.cuh"
#include "launch.h"

namespace sc {

// ---------------------------------------------------------------------------
// Auxiliary kernels

// copy_back, S/conv.py:424-449: dst[region] := src[region], per plane.
// One warp per region row (grid-stride over rows). The body moves float4s when
// source and destination rows share their 16-B phase (always, for equal
// strides and aligned bases), four loads in flight per lane before the stores;
// the <= 3 columns before the first aligned destination float and the tail are
// scalar. Rows of mismatched phase fall back to coalesced scalar copies.
static __global__ void __launch_bounds__(256) copy_region_kernel(const float* __restrict__ src, float* __restrict__ dst,
                                                                 long long sps, long long dps, long long srs,
                                                                 long long drs, int nplanes, int row_lo, int nrows,
                                                                 int col_lo, int ncols) {
    const int lane = threadIdx.x & 31;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    const long long rows = (long long)nplanes * nrows;
    for (long long rr = warp; rr < rows; rr += nwarps) {
        const long long pl = rr / nrows;
        const int y = row_lo + (int)(rr - pl * nrows);
        const float* s = src + pl * sps + (long long)y * srs + col_lo;
        float* d = dst + pl * dps + (long long)y * drs + col_lo;
        int head = (int)(((16u - (unsigned)(reinterpret_cast<uintptr_t>(d) & 15u)) & 15u) >> 2);
        if (head > ncols) head = ncols;
        if ((reinterpret_cast<uintptr_t>(s + head) & 15u) != 0) {
            for (int c = lane; c < ncols; c += 32) d[c] = s[c];
            continue;
        }
        if (lane < head) d[lane] = s[lane];
        const int nv = (ncols - head) >> 2;
        const float4* s4 = reinterpret_cast<const float4*>(s + head);
        float4* d4 = reinterpret_cast<float4*>(d + head);
        int i = lane;
        for (; i + 96 < nv; i += 128) {
            const float4 a = s4[i], b = s4[i + 32], c = s4[i + 64], e = s4[i + 96];
            d4[i] = a;
            d4[i + 32] = b;
            d4[i + 64] = c;
            d4[i + 96] = e;
        }
        for (; i < nv; i += 32) d4[i] = s4[i];
        const int t0 = head + 4 * nv;
        if (t0 + lane < ncols) d[t0 + lane] = s[t0 + lane];
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
    // one warp per row: up to 8 warps x 8 CTAs per SM
    copy_region_kernel<<<grid_for((long long)nplanes * nrows * 32, 256), 256, 0, s>>>(
        src, dst, sps, dps, srs, drs, nplanes, row_lo, nrows, col_lo, ncols);
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
