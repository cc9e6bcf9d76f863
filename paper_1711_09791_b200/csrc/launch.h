// launch.h -- internal (C++) interface between the C ABI layer and the kernel TUs.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace sc {

struct Params;

// Kernel entry for (mode, radius, aligned); nullptr if unsupported.
const void* kernel_fused(int rad, bool aligned, bool symw = false, bool sig = false);
const void* kernel_hpass(int rad, bool aligned);
const void* kernel_vpass(int rad, bool aligned);
const void* kernel_single(int rad, bool aligned, int sym = 0);  // sym: 0, 1 rows mirror, 2 rows+cols
const void* kernel_splitf(int rad, bool symw = false);
const void* kernel_single_cb(int rad, int sym);
const void* kernel_fused_direct(int rad);
const void* kernel_hpass_direct(int rad);
const void* kernel_vpass_direct(int rad);
const void* kernel_single_direct(int rad);
// widths 11..31 (r = 5..10 / 11..15), any row alignment (kern_lanes_wide*.cu); nullptr otherwise
const void* kernel_lanes_wide(int mode, int rad, bool symw, bool aligned);
const void* kernel_lanes_wide2(int mode, int rad, bool symw);
const void* kernel_lanes_wide_single(int rad);

// gen: any row geometry (cols % 16 != 0, rows or buffers not 16-B aligned)
const void* kernel_u8(int rad, bool symw = false, bool occ3 = false, bool gen = false);
// whether the 3-CTA (128-register) u8 build holds this radius without spilling
bool u8_occ3_fits(int rad, bool symw);
cudaError_t launch_hwc_to_planes(const uint8_t* src, float* dst, long long srs, long long dps, long long drs, int R,
                                 int C, cudaStream_t s);
cudaError_t launch_planes_to_hwc(const float* src, uint8_t* dst, long long sps, long long srs, long long drs, int R,
                                 int C, cudaStream_t s);

cudaError_t launch_copy_region(const float* src, float* dst, long long sps, long long dps, long long srs,
                               long long drs, int nplanes, int row_lo, int nrows, int col_lo, int ncols,
                               cudaStream_t s);
// Halo snapshot of the split-fused kernel (layout: Params::side_rows / side_cols).
struct SnapJob {
    const float* img;
    long long ps, rs;
    int nplanes, R, C, rad;
    int tw, nstrips;
    int lo1, bh1, nb1, lo2, bh2, nb;  // band b's first row: b < nb1 ? lo1 + b*bh1 : lo2 + (b-nb1)*bh2
    float* side_rows;
    float* side_cols;
};
cudaError_t launch_split_snapshot(const SnapJob& j, cudaStream_t s);
cudaError_t launch_fill_synthetic(float* dst, long long count, uint64_t seed, uint64_t offset, int kind,
                                  cudaStream_t s);

// Geometry of one row-streaming launch (global row indices).
struct RowsJob {
    int mode;
    const float* src;
    float* dst;
    long long sps, dps, srs, drs;
    int nplanes, R, C;
    int src_row0, src_rows, dst_row0;
    int out_lo, out_hi, hrow_lo, hrow_hi;
    int out_lo2 = 0, out_hi2 = 0;  // optional second output segment
    int flags;
    int width;
    const float* taps;   // width floats (host)
    const float* dense;  // width*width floats (host), SINGLE only
    // optional neighbouring bands (peer memory) holding the halo rows just above /
    // below [src_row0, src_row0 + src_rows); rows 0 = global rows above_row0 / below_row0
    const float* above = nullptr;
    const float* below = nullptr;
    long long above_ps = 0, above_rs = 0, below_ps = 0, below_rs = 0;
    int above_row0 = 0, above_rows = 0, below_row0 = 0, below_rows = 0;
    // MODE_SPLITF: scratch planes (H0); MODE_SINGLECB: the image (copy-back); same rows
    float* scr = nullptr;
    long long scr_ps = 0, scr_rs = 0;
    // row-band readiness signalling between ranks (Params::sig_*; epoch 0 = off)
    unsigned long long* sig_self = nullptr;
    const unsigned long long* sig_above = nullptr;
    const unsigned long long* sig_below = nullptr;
    unsigned long long epoch = 0;
    unsigned int* sig_err = nullptr;
};

// NCCL band step: both halo packs in one launch (kern_aux.cu)
cudaError_t launch_pack_rows(const float* src, long long sps, long long srs, int P, int r, int C, int row_a,
                             float* out_a, int row_b, float* out_b, cudaStream_t s);

// one-thread kernel: wait until the neighbours' signal word `word` (0 ready,
// 1 done) reaches `value` (kern_aux.cu)
cudaError_t launch_signal_wait(const unsigned long long* a, const unsigned long long* b, int word,
                               unsigned long long value, unsigned int* err, long long timeout_ns, cudaStream_t s);

// Plans and launches one row-streaming kernel; returns an SC_* status and sets
// the thread's last error on failure.
int launch_rows(const RowsJob& job, cudaStream_t s);
// widths above MAX_W (kern_wide.cu); called by launch_rows
int launch_wide(const RowsJob& job, cudaStream_t s);

void set_error(const std::string& msg);
int fail_arg(const std::string& msg);                   // SC_INVALID_ARGUMENT with a message
int fail_cuda(cudaError_t e, const std::string& what);  // SC_CUDA_ERROR with the CUDA error string
void count_launch(uint64_t n = 1);

}  // namespace sc
