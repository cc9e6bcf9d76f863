// kern_wide.cu -- kernel widths above 9 (radius > 4): the reference accepts any
// odd width on its generic and two-pass bodies (S/kernels.py:17-20,
// S/conv.py:86-143, :215-318). The tuned row-streaming kernels keep a 4-column
// smem halo and a 12-sample register window, i.e. r <= 4; wider kernels run
// here: one thread per output sample, taps in global memory, the same float32
// products and sums in the reference's order (bit-identical), no tuning. Up to
// MAX_W_WIDE taps.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstring>
#include <string>

#include "../../include/sepconv_b200.h"
#include "kernels.cuh"
#include "launch.h"

namespace sc {

struct WideParams {
    const float* src;
    float* dst;
    long long sps, srs, dps, drs;
    int nplanes, R, C, rad;
    int src_row0, dst_row0;
    int out_lo, out_hi, out_lo2, out_hi2;  // output rows (global), second segment optional
    int hrow_lo, hrow_hi;                  // rows where the row pass is live
    int flags;
    const float* taps;  // device: 2r+1 floats, or (2r+1)^2 (single pass)
};

__device__ __forceinline__ int wide_row(const WideParams& p, long long i, int& x, int& plane) {
    // i -> (plane, output row of the one or two segments, column)
    const long long n1 = (long long)(p.out_hi - p.out_lo) * p.C;
    const long long n2 = (long long)(p.out_hi2 - p.out_lo2) * p.C;
    plane = (int)(i / (n1 + n2));
    long long k = i - (long long)plane * (n1 + n2);
    if (k < n1) {
        x = (int)(k % p.C);
        return p.out_lo + (int)(k / p.C);
    }
    k -= n1;
    x = (int)(k % p.C);
    return p.out_lo2 + (int)(k / p.C);
}

// horizontal_rows_vec (S/conv.py:215-240) with the HPASS policies: live rows get
// H on the valid columns; with F_ZERO_FILL the ring columns and dead rows get 0.
__global__ void wide_hpass_kernel(const WideParams p) {
    const int W = 2 * p.rad + 1;
    const long long total = (long long)p.nplanes * ((p.out_hi - p.out_lo) + (p.out_hi2 - p.out_lo2)) * p.C;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        int x, pl;
        const int y = wide_row(p, i, x, pl);
        const bool live = y >= p.hrow_lo && y < p.hrow_hi;
        const bool valid = x >= p.rad && x < p.C - p.rad;
        float* d = p.dst + pl * p.dps + (long long)(y - p.dst_row0) * p.drs + x;
        if (live && valid) {
            const float* s = p.src + pl * p.sps + (long long)(y - p.src_row0) * p.srs + (x - p.rad);
            float acc = __fmul_rn(s[0], p.taps[0]);
            for (int m = 1; m < W; ++m) acc = __fadd_rn(acc, __fmul_rn(s[m], p.taps[m]));
            *d = acc;
        } else if (p.flags & F_ZERO_FILL) {
            *d = 0.0f;
        }
    }
}

// vertical_rows_vec (S/conv.py:269-293) over valid rows, valid columns; for the
// fused two-pass (FUSED: src = H0 rows, ring = the input image) the ring samples
// are copied from the input unless F_NO_RING.
__global__ void wide_vpass_kernel(const WideParams p, const float* ring_src, long long ring_ps, long long ring_rs,
                                  int ring_row0, int fused) {
    const int W = 2 * p.rad + 1;
    const long long total = (long long)p.nplanes * ((p.out_hi - p.out_lo) + (p.out_hi2 - p.out_lo2)) * p.C;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        int x, pl;
        const int y = wide_row(p, i, x, pl);
        const bool valid = x >= p.rad && x < p.C - p.rad && y >= p.rad && y < p.R - p.rad;
        float* d = p.dst + pl * p.dps + (long long)(y - p.dst_row0) * p.drs + x;
        if (valid) {
            const float* s = p.src + pl * p.sps + (long long)(y - p.rad - p.src_row0) * p.srs + x;
            float acc = __fmul_rn(s[0], p.taps[0]);
            for (int m = 1; m < W; ++m) acc = __fadd_rn(acc, __fmul_rn(s[m * p.srs], p.taps[m]));
            *d = acc;
        } else if (fused && !(p.flags & F_NO_RING)) {
            *d = ring_src[pl * ring_ps + (long long)(y - ring_row0) * ring_rs + x];
        }
    }
}

// single_pass_rows_vec (S/conv.py:86-114): row-major fold from the first product.
__global__ void wide_single_kernel(const WideParams p) {
    const int W = 2 * p.rad + 1;
    const long long total = (long long)p.nplanes * ((p.out_hi - p.out_lo) + (p.out_hi2 - p.out_lo2)) * p.C;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        int x, pl;
        const int y = wide_row(p, i, x, pl);
        if (x < p.rad || x >= p.C - p.rad || y < p.rad || y >= p.R - p.rad) continue;
        const float* s = p.src + pl * p.sps + (long long)(y - p.rad - p.src_row0) * p.srs + (x - p.rad);
        float acc = __fmul_rn(s[0], p.taps[0]);
        for (int a = 0; a < W; ++a)
            for (int b = (a == 0 ? 1 : 0); b < W; ++b)
                acc = __fadd_rn(acc, __fmul_rn(s[(long long)a * p.srs + b], p.taps[a * W + b]));
        p.dst[pl * p.dps + (long long)(y - p.dst_row0) * p.drs + x] = acc;
    }
}

static int wide_grid(long long total) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    long long b = (total + 255) / 256;
    if (b > (long long)sms * 16) b = (long long)sms * 16;
    return b < 1 ? 1 : (int)b;
}

int launch_wide(const RowsJob& j, cudaStream_t s) {
    if (j.above || j.below) {
        set_error("kernel widths above 9 are not supported for peer-memory row bands");
        return SC_UNSUPPORTED_WIDTH;
    }
    if (j.width > MAX_W_WIDE) {
        set_error("kernel width " + std::to_string(j.width) + " > " + std::to_string(MAX_W_WIDE) + " not supported");
        return SC_UNSUPPORTED_WIDTH;
    }
    const int rad = j.width / 2;
    const bool single = j.mode == MODE_SINGLE;
    const int ntaps = single ? j.width * j.width : j.width;
    const float* host_taps = single ? j.dense : j.taps;
    const long long outs = (long long)j.nplanes * ((j.out_hi - j.out_lo) + (j.out_hi2 - j.out_lo2)) * j.C;
    if (outs <= 0) return SC_OK;
    float* taps = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&taps), sizeof(float) * ntaps, s);
    if (e != cudaSuccess) {
        cudaGetLastError();
        set_error(std::string("wide taps allocation: ") + cudaGetErrorString(e));
        return SC_CUDA_ERROR;
    }
    e = cudaMemcpyAsync(taps, host_taps, sizeof(float) * ntaps, cudaMemcpyHostToDevice, s);
    WideParams p;
    std::memset(&p, 0, sizeof(p));
    p.src = j.src;
    p.dst = j.dst;
    p.sps = j.sps;
    p.srs = j.srs;
    p.dps = j.dps;
    p.drs = j.drs;
    p.nplanes = j.nplanes;
    p.R = j.R;
    p.C = j.C;
    p.rad = rad;
    p.src_row0 = j.src_row0;
    p.dst_row0 = j.dst_row0;
    p.out_lo = j.out_lo;
    p.out_hi = j.out_hi;
    p.out_lo2 = j.out_hi2 > j.out_lo2 ? j.out_lo2 : 0;
    p.out_hi2 = j.out_hi2 > j.out_lo2 ? j.out_hi2 : 0;
    p.hrow_lo = j.hrow_lo;
    p.hrow_hi = j.hrow_hi;
    p.flags = j.flags;
    p.taps = taps;
    float* h0 = nullptr;
    if (e == cudaSuccess) {
        switch (j.mode) {
            case MODE_HPASS:
                wide_hpass_kernel<<<wide_grid(outs), 256, 0, s>>>(p);
                count_launch();
                break;
            case MODE_VPASS:
                wide_vpass_kernel<<<wide_grid(outs), 256, 0, s>>>(p, nullptr, 0, 0, 0, 0);
                count_launch();
                break;
            case MODE_SINGLE:
                wide_single_kernel<<<wide_grid(outs), 256, 0, s>>>(p);
                count_launch();
                break;
            case MODE_FUSED: {
                // H0 (zero outside the live rows and on the column ring) for the rows
                // the outputs need, then the column pass with the ring from the input
                const int lo_all = p.out_hi2 > p.out_lo2 ? (p.out_lo < p.out_lo2 ? p.out_lo : p.out_lo2) : p.out_lo;
                const int hi_all = p.out_hi2 > p.out_lo2 ? (p.out_hi > p.out_hi2 ? p.out_hi : p.out_hi2) : p.out_hi;
                const int h_lo = lo_all - rad > j.src_row0 ? lo_all - rad : j.src_row0;
                const int h_hi = hi_all + rad < j.src_row0 + j.src_rows ? hi_all + rad : j.src_row0 + j.src_rows;
                const long long hplane = (long long)(h_hi - h_lo) * j.C;
                e = cudaMallocAsync(reinterpret_cast<void**>(&h0), sizeof(float) * hplane * j.nplanes, s);
                if (e != cudaSuccess) break;
                WideParams ph = p;
                ph.dst = h0;
                ph.dps = hplane;
                ph.drs = j.C;
                ph.dst_row0 = h_lo;
                ph.out_lo = h_lo;
                ph.out_hi = h_hi;
                ph.out_lo2 = ph.out_hi2 = 0;
                ph.flags = F_ZERO_FILL;
                wide_hpass_kernel<<<wide_grid(hplane * j.nplanes), 256, 0, s>>>(ph);
                WideParams pv = p;
                pv.src = h0;
                pv.sps = hplane;
                pv.srs = j.C;
                pv.src_row0 = h_lo;
                wide_vpass_kernel<<<wide_grid(outs), 256, 0, s>>>(pv, j.src, j.sps, j.srs, j.src_row0, 1);
                count_launch(2);
                break;
            }
            default:
                set_error("no wide kernel for this mode");
                cudaFreeAsync(taps, s);
                return SC_UNSUPPORTED_WIDTH;
        }
    }
    if (e == cudaSuccess) e = cudaGetLastError();
    if (h0) cudaFreeAsync(h0, s);
    cudaFreeAsync(taps, s);
    if (e != cudaSuccess) {
        set_error(std::string("wide kernel: ") + cudaGetErrorString(e));
        return SC_CUDA_ERROR;
    }
    return SC_OK;
}

}  // namespace sc
