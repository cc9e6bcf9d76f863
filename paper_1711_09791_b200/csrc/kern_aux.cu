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


// Split-fused halo snapshot (S/conv.py:392-421 run in place needs the samples
// other items read before their owners overwrite them): for every band boundary
// b >= 1 the 2r image rows around it (one warp per row, float4 lanes, four
// loads in flight), for every strip boundary s >= 1 the 8 columns around it in
// every row (one thread per row: two float4s). Aligned rows only.
static __global__ void __launch_bounds__(256) split_snapshot_kernel(const SnapJob j) {
    const int lane = threadIdx.x & 31;
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nthreads = (long long)gridDim.x * blockDim.x;
    const int c4 = j.C / 4, r2 = 2 * j.rad;
    const long long ntask = (long long)j.nplanes * j.nb * r2;
    for (long long task = tid >> 5; task < ntask; task += nthreads >> 5) {
        const int t = (int)(task % r2);
        const long long q = task / r2;
        const int b = (int)(q % j.nb);
        const int pl = (int)(q / j.nb);
        if (b == 0) continue;
        const int lo = b < j.nb1 ? j.lo1 + b * j.bh1 : j.lo2 + (b - j.nb1) * j.bh2;
        const int y = lo - j.rad + t;
        if (y < 0 || y >= j.R) continue;
        const float4* src = reinterpret_cast<const float4*>(j.img + pl * j.ps + (long long)y * j.rs);
        float4* dst = reinterpret_cast<float4*>(j.side_rows + (((long long)pl * j.nb + b) * r2 + t) * j.C);
        int i = lane;
        for (; i + 96 < c4; i += 128) {
            const float4 v0 = src[i], v1 = src[i + 32], v2 = src[i + 64], v3 = src[i + 96];
            dst[i] = v0;
            dst[i + 32] = v1;
            dst[i + 64] = v2;
            dst[i + 96] = v3;
        }
        for (; i < c4; i += 32) dst[i] = src[i];
    }
    const int nsb = j.nstrips - 1;
    const long long ncol = (long long)j.nplanes * nsb * j.R;
    for (long long i = tid; i < ncol; i += nthreads) {
        const int y = (int)(i % j.R);
        const long long q = i / j.R;
        const int s = (int)(q % nsb) + 1;
        const int pl = (int)(q / nsb);
        const float4* src = reinterpret_cast<const float4*>(j.img + pl * j.ps + (long long)y * j.rs + s * j.tw - 4);
        float4* dst = reinterpret_cast<float4*>(j.side_cols + i * 8);  // i == ((pl * nsb + s - 1) * R + y)
        const float4 a = src[0], c = src[1];
        dst[0] = a;
        dst[1] = c;
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

cudaError_t launch_split_snapshot(const SnapJob& j, cudaStream_t s) {
    const long long work = (long long)j.nplanes * j.nb * 2 * j.rad * 32 + (long long)j.nplanes * (j.nstrips - 1) * j.R;
    if (work <= 0) return cudaSuccess;
    split_snapshot_kernel<<<grid_for(work, 256), 256, 0, s>>>(j);
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

// Stream-ordered wait for the neighbouring bands' signal words (a caller about to
// overwrite its band's input rows waits until both neighbours are done reading
// them, S/executors.py:142-151's launch barrier on the device).
// word 0: the neighbours' launch of epoch `value` started (ready >= value);
// word 1: it finished reading THIS band's rows -- the band above counts its
// below-reading items in [3] (target [5] per launch), the band below its
// above-reading items in [2] (target [4]).
__global__ void signal_wait_kernel(const unsigned long long* a, const unsigned long long* b, int word,
                                   unsigned long long value, unsigned int* err, long long timeout_ns) {
    if (threadIdx.x != 0) return;
    const unsigned long long* sides[2] = {a, b};
    for (int s = 0; s < 2; ++s) {
        const unsigned long long* w = sides[s];
        if (!w) continue;
        wait_signal(w, value, err, timeout_ns);  // the launch of that epoch has started: targets current
        if (word == 1) {
            const int cnt = s == 0 ? 3 : 2;
            const unsigned long long target = value * ld_acquire_sys(w + cnt + 2);
            wait_signal(w + cnt, target, err, timeout_ns);
        }
    }
}

cudaError_t launch_signal_wait(const unsigned long long* a, const unsigned long long* b, int word,
                               unsigned long long value, unsigned int* err, long long timeout_ns, cudaStream_t s) {
    signal_wait_kernel<<<1, 32, 0, s>>>(a, b, word, value, err, timeout_ns);
    count_launch();
    return cudaGetLastError();
}

// Halo pack of the NCCL band step: rows [row_a, row_a + r) and [row_b, row_b + r)
// of every plane into two contiguous (P, r, C) buffers, in one launch (either
// destination may be null).
__global__ void pack_rows_kernel(const float* src, long long sps, long long srs, int P, int r, int C, int row_a,
                                 float* out_a, int row_b, float* out_b) {
    const long long per = (long long)P * r * C;
    const long long total = 2 * per;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const bool second = i >= per;
        float* out = second ? out_b : out_a;
        if (!out) continue;
        const long long k = second ? i - per : i;
        const int p = (int)(k / ((long long)r * C));
        const long long rem = k - (long long)p * r * C;
        const int y = (int)(rem / C), x = (int)(rem - (long long)y * C);
        out[k] = src[p * sps + (long long)((second ? row_b : row_a) + y) * srs + x];
    }
}

cudaError_t launch_pack_rows(const float* src, long long sps, long long srs, int P, int r, int C, int row_a,
                             float* out_a, int row_b, float* out_b, cudaStream_t s) {
    const long long total = 2LL * P * r * C;
    pack_rows_kernel<<<grid_for(total, 256), 256, 0, s>>>(src, sps, srs, P, r, C, row_a, out_a, row_b, out_b);
    count_launch();
    return cudaGetLastError();
}

}  // namespace sc
