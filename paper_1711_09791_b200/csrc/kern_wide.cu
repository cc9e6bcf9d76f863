// kern_wide.cu -- kernel widths above 9 (radius > 4): the reference accepts any
// odd width on its generic and two-pass bodies (S/kernels.py:17-20,
// S/conv.py:86-143, :215-318). The tuned row-streaming kernels keep a 4-column
// smem halo and a 12-sample register window, i.e. r <= 4; wider kernels run
// here: one thread per output sample, the same float32 products and sums in the
// reference's order (bit-identical), no tuning. Up to MAX_W_WIDE taps. The taps
// travel BY VALUE in the kernel parameters (a __grid_constant__ struct, read
// through the constant cache): no per-launch allocation or host copy, so these
// launches are stream-ordered like any other and capture into CUDA graphs. The
// dense single-pass matrix fits up to width 89 (89^2 floats < the 32 KB
// parameter limit); wider dense matrices are copied to a stream-ordered device
// buffer per launch.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstring>
#include <string>

#include "../../include/sepconv_b200.h"
#include "kernels.cuh"
#include "launch.h"

namespace sc {

constexpr int kWideSepTaps = MAX_W_WIDE + 1;  // separable taps (2r+1 <= 255)
constexpr int kWideDenseTaps = 89 * 89;        // dense matrix by value up to width 89

template <int NT>
struct WideParamsT {
    const float* src;
    float* dst;
    long long sps, srs, dps, drs;
    int nplanes, R, C, rad;
    int src_row0, dst_row0;
    int out_lo, out_hi, out_lo2, out_hi2;  // output rows (global), second segment optional
    int hrow_lo, hrow_hi;                  // rows where the row pass is live
    int flags;
    const float* taps_dev;  // dense matrices wider than 89: device copy (else null)
    float taps[NT];         // 2r+1 floats, or (2r+1)^2 (single pass)
};
using WideParams = WideParamsT<kWideSepTaps>;

template <class P>
__device__ __forceinline__ int wide_row(const P& p, long long i, int& x, int& plane) {
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
__global__ void wide_hpass_kernel(const __grid_constant__ WideParams p) {
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
__global__ void wide_vpass_kernel(const __grid_constant__ WideParams p, const float* ring_src, long long ring_ps, long long ring_rs,
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
template <int NT>
__global__ void wide_single_kernel(const __grid_constant__ WideParamsT<NT> p) {
    const int W = 2 * p.rad + 1;
    const float* k = p.taps_dev ? p.taps_dev : p.taps;
    const long long total = (long long)p.nplanes * ((p.out_hi - p.out_lo) + (p.out_hi2 - p.out_lo2)) * p.C;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        int x, pl;
        const int y = wide_row(p, i, x, pl);
        if (x < p.rad || x >= p.C - p.rad || y < p.rad || y >= p.R - p.rad) continue;
        const float* s = p.src + pl * p.sps + (long long)(y - p.rad - p.src_row0) * p.srs + (x - p.rad);
        float acc = __fmul_rn(s[0], k[0]);
        for (int a = 0; a < W; ++a)
            for (int b = (a == 0 ? 1 : 0); b < W; ++b)
                acc = __fadd_rn(acc, __fmul_rn(s[(long long)a * p.srs + b], k[a * W + b]));
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

template <class P>
static void fill_common(P& p, const RowsJob& j, int rad) {
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
    p.taps_dev = nullptr;
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
    const long long outs = (long long)j.nplanes * ((j.out_hi - j.out_lo) + (j.out_hi2 - j.out_lo2)) * j.C;
    if (outs <= 0) return SC_OK;
    cudaError_t e = cudaSuccess;
    if (j.mode == MODE_SINGLE) {
        const int ntaps = j.width * j.width;
        if (ntaps <= kWideDenseTaps) {
            static thread_local WideParamsT<kWideDenseTaps> pd;  // 32 KB: not on the stack
            fill_common(pd, j, rad);
            std::memcpy(pd.taps, j.dense, sizeof(float) * ntaps);
            wide_single_kernel<kWideDenseTaps><<<wide_grid(outs), 256, 0, s>>>(pd);
        } else {
            // dense matrices wider than 89: a stream-ordered device copy from a
            // pinned staging buffer (freed after the kernel, in stream order)
            WideParamsT<1> pd;
            fill_common(pd, j, rad);
            float* dev = nullptr;
            float* pinned = nullptr;
            e = cudaMallocAsync(reinterpret_cast<void**>(&dev), sizeof(float) * ntaps, s);
            if (e == cudaSuccess) e = cudaMallocHost(reinterpret_cast<void**>(&pinned), sizeof(float) * ntaps);
            if (e == cudaSuccess) {
                std::memcpy(pinned, j.dense, sizeof(float) * ntaps);
                e = cudaMemcpyAsync(dev, pinned, sizeof(float) * ntaps, cudaMemcpyHostToDevice, s);
            }
            if (e == cudaSuccess) {
                pd.taps_dev = dev;
                wide_single_kernel<1><<<wide_grid(outs), 256, 0, s>>>(pd);
                e = cudaStreamSynchronize(s);  // the pinned staging buffer is released below
            }
            if (dev) cudaFreeAsync(dev, s);
            if (pinned) cudaFreeHost(pinned);
        }
        if (e == cudaSuccess) e = cudaGetLastError();
        if (e != cudaSuccess) {
            cudaGetLastError();
            set_error(std::string("wide kernel: ") + cudaGetErrorString(e));
            return SC_CUDA_ERROR;
        }
        count_launch();
        return SC_OK;
    }
    WideParams p;
    fill_common(p, j, rad);
    for (int i = 0; i < j.width; ++i) p.taps[i] = j.taps[i];
    float* h0 = nullptr;
    switch (j.mode) {
        case MODE_HPASS:
            wide_hpass_kernel<<<wide_grid(outs), 256, 0, s>>>(p);
            count_launch();
            break;
        case MODE_VPASS:
            wide_vpass_kernel<<<wide_grid(outs), 256, 0, s>>>(p, nullptr, 0, 0, 0, 0);
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
            return SC_UNSUPPORTED_WIDTH;
    }
    if (e == cudaSuccess) e = cudaGetLastError();
    if (h0) cudaFreeAsync(h0, s);
    if (e != cudaSuccess) {
        cudaGetLastError();
        set_error(std::string("wide kernel: ") + cudaGetErrorString(e));
        return SC_CUDA_ERROR;
    }
    return SC_OK;
}

}  // namespace sc
