// kernels.cuh -- sm_100a kernels for the separable (2r+1)-tap convolution path.
//
// One row-streaming kernel template covers the four hot-path operations of the
// reference (S/ = /root/reference/pkg/src/sepconv_lab/):
//
//   MODE_FUSED  conv_two_pass / convolve_image TWO_PASS   S/conv.py:392-421, S/executors.py:308-326
//               single read + single write: H row computed on-chip, V folded
//               through a register shift-register, ring copied from the input.
//   MODE_HPASS  horizontal_rows_vec                       S/conv.py:215-240
//   MODE_VPASS  vertical_rows_vec                         S/conv.py:269-293
//   MODE_SINGLE single_pass_rows_vec / unrolled5_rows_vec S/conv.py:86-114, :146-175
//
// Work decomposition: an "item" is (plane, column strip of TW = 4*NT output
// columns, row band). A persistent grid walks items round-robin. Per CTA:
//   warp 0      producer: streams input rows [x0-4, x0+TW+4) of the strip into a
//               ring of NR shared-memory row slots with the bulk-copy TMA engine
//               (cp.async.bulk + mbarrier complete_tx); generic (unaligned) mode
//               uses plain loads by the 32 producer lanes instead.
//   warps 1..   consumers: thread t owns 4 adjacent output columns. Per input
//               row it reads 12 samples (3 x LDS.128), computes the row pass for
//               its 4 columns and pushes them through a shift register of 2r
//               partial column sums, emitting output row y-r as soon as input
//               row y arrived. Results go straight to HBM with STG.128.
//
// Bit-exactness: every product/sum is __fmul_rn/__fadd_rn (never contracted to
// FMA) in the reference's fold order: left-to-right from the first product,
// kernel rows outer, kernel columns inner (S/conv.py:1-15). The shift register
// preserves that order because input rows arrive in increasing order, which is
// exactly the order of the terms of each output's fold.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace sc {

enum Mode : int { MODE_FUSED = 0, MODE_HPASS = 1, MODE_VPASS = 2, MODE_SINGLE = 3 };

// flags (mirrors include/sepconv_b200.h)
constexpr int F_EXTENDED = 0x1;
constexpr int F_NO_RING = 0x2;
constexpr int F_ZERO_FILL = 0x4;

constexpr int HALO = 4;       // smem columns kept either side of a strip (supports r <= 4)
constexpr int MAX_RAD = 4;
constexpr int MAX_W = 2 * MAX_RAD + 1;
constexpr int MAX_THREADS = 32 + 256;

struct Params {
    const float* src;
    float* dst;
    long long src_plane_stride, dst_plane_stride;  // elements
    long long src_row_stride, dst_row_stride;      // elements
    int nplanes;
    int R, C;                // global image rows / cols
    int src_row0, src_rows;  // src holds global rows [src_row0, src_row0 + src_rows)
    int dst_row0;            // dst row 0 is global row dst_row0
    int out_lo, out_hi;      // output rows produced (global)
    int hrow_lo, hrow_hi;    // rows where the row pass is live (else H0 = 0 / zero fill)
    int flags;
    int tw;                  // strip width = 4 * consumer threads
    int nstrips, band_h, nitems;
    int nr;                  // ring slots (rows)
    float w[MAX_W];
    float k[MAX_W * MAX_W];
};

// ---------------------------------------------------------------------------
// PTX helpers (mbarrier + bulk copy)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(tx)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "SC_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra SC_WAIT;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(sdst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// ---------------------------------------------------------------------------
// Strict float32 arithmetic (never contracted)

__device__ __forceinline__ float fm(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fa(float a, float b) { return __fadd_rn(a, b); }

struct F4 {
    float v[4];
};

__device__ __forceinline__ F4 ld4(const float* p) {
    float4 t = *reinterpret_cast<const float4*>(p);
    F4 r;
    r.v[0] = t.x; r.v[1] = t.y; r.v[2] = t.z; r.v[3] = t.w;
    return r;
}

__device__ __forceinline__ void st4(float* p, const F4& a) {
    *reinterpret_cast<float4*>(p) = make_float4(a.v[0], a.v[1], a.v[2], a.v[3]);
}

// ---------------------------------------------------------------------------
// Item geometry

struct Item {
    int plane, x0, ylo, yhi, in_lo, in_hi;
};

template <int MODE, int RAD>
__device__ __forceinline__ Item decode_item(const Params& p, int item) {
    const int units = p.nplanes * p.nstrips;
    const int band = item / units;
    const int rem = item - band * units;
    Item it;
    it.plane = rem / p.nstrips;
    const int strip = rem - it.plane * p.nstrips;
    it.x0 = strip * p.tw;
    it.ylo = p.out_lo + band * p.band_h;
    it.yhi = min(it.ylo + p.band_h, p.out_hi);
    if (MODE == MODE_HPASS) {
        it.in_lo = it.ylo;
        it.in_hi = it.yhi;
    } else {
        it.in_lo = max(max(it.ylo - RAD, 0), p.src_row0);
        it.in_hi = min(min(it.yhi + RAD, p.R), p.src_row0 + p.src_rows);
    }
    return it;
}

// ---------------------------------------------------------------------------
// Producer: one warp streams rows of the strip into the smem ring.

template <int MODE, int RAD, bool ALIGNED>
__device__ __forceinline__ void producer(const Params& p, float* ring, uint64_t* full, uint64_t* empty) {
    const int lane = threadIdx.x & 31;
    if (ALIGNED && lane != 0) return;
    const int SW = p.tw + 2 * HALO;
    const int NR = p.nr;
    uint64_t pol = 0;
    if (ALIGNED) pol = policy_evict_first();
    int slot = 0;
    uint32_t phase = 0;
    long long g = 0;
    for (int item = blockIdx.x; item < p.nitems; item += gridDim.x) {
        const Item it = decode_item<MODE, RAD>(p, item);
        const int cx0 = max(it.x0 - HALO, 0);
        const int cx1 = min(it.x0 + p.tw + HALO, p.C);
        const int n = cx1 - cx0;
        const float* gbase = p.src + (long long)it.plane * p.src_plane_stride + cx0;
        for (int yi = it.in_lo; yi < it.in_hi; ++yi, ++g) {
            if (g >= NR) mbar_wait(&empty[slot], phase ^ 1u);
            const float* gsrc = gbase + (long long)(yi - p.src_row0) * p.src_row_stride;
            float* sdst = ring + slot * SW + (cx0 - (it.x0 - HALO));
            if (ALIGNED) {
                const uint32_t bytes = (uint32_t)n * 4u;
                mbar_arrive_expect_tx(&full[slot], bytes);
                bulk_g2s(sdst, gsrc, bytes, &full[slot], pol);
            } else {
                for (int c = lane; c < n; c += 32) sdst[c] = __ldg(gsrc + c);
                mbar_arrive(&full[slot]);
            }
            if (++slot == NR) { slot = 0; phase ^= 1u; }
        }
    }
}

// ---------------------------------------------------------------------------
// Consumer helpers

// Row pass for 4 adjacent output columns: win holds columns x4-4 .. x4+7.
template <int RAD>
__device__ __forceinline__ F4 row_pass(const float (&win)[12], const float* w) {
    F4 h;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        float acc = fm(win[HALO - RAD + c], w[0]);
#pragma unroll
        for (int m = 1; m <= 2 * RAD; ++m) acc = fa(acc, fm(win[HALO - RAD + c + m], w[m]));
        h.v[c] = acc;
    }
    return h;
}

// Store one output row segment of 4 columns with the column-ring policy.
//   ring_mode 0: keep   -- only columns in [RAD, C-RAD) are written
//   ring_mode 1: copy   -- ring columns take `ringv` (input samples)
//   ring_mode 2: zero   -- ring columns take 0
template <bool ALIGNED>
__device__ __forceinline__ void store_row(float* drow, int x4, int C, int RAD_, const F4& val, const F4& ringv,
                                          int ring_mode) {
    const bool interior = (x4 >= RAD_) && (x4 + 4 <= C - RAD_);
    if (ALIGNED && interior) {
        st4(drow + x4, val);
        return;
    }
    if (x4 >= C) return;
    F4 o;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int col = x4 + c;
        const bool valid = col >= RAD_ && col < C - RAD_;
        o.v[c] = valid ? val.v[c] : (ring_mode == 1 ? ringv.v[c] : 0.0f);
    }
    if (ALIGNED && ring_mode != 0) {  // x4 + 4 <= C when C % 4 == 0
        st4(drow + x4, o);
        return;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int col = x4 + c;
        if (col >= C) break;
        const bool valid = col >= RAD_ && col < C - RAD_;
        if (valid || ring_mode != 0) drow[col] = o.v[c];
    }
}

// ---------------------------------------------------------------------------
// The kernel

template <int MODE, int RAD, bool ALIGNED>
__global__ void __launch_bounds__(MAX_THREADS, 1) sepconv_rows_kernel(const __grid_constant__ Params p) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int NR = p.nr;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t* empty = full + NR;
    float* ring = reinterpret_cast<float*>(smem_raw + ((2 * NR * 8 + 127) / 128) * 128);
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int ncw = (blockDim.x >> 5) - 1;

    if (threadIdx.x == 0) {
        for (int i = 0; i < NR; ++i) {
            mbar_init(&full[i], ALIGNED ? 1u : 32u);
            mbar_init(&empty[i], (uint32_t)ncw);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (warp == 0) {
        producer<MODE, RAD, ALIGNED>(p, ring, full, empty);
        return;
    }

    constexpr int NACC = (2 * RAD > 0) ? 2 * RAD : 1;
    constexpr int LAG = RAD;  // rows kept after use (FUSED reads row y-r for ring columns)
    const int SW = p.tw + 2 * HALO;
    const int ct = threadIdx.x - 32;
    const int R = p.R, C = p.C;
    const bool ring_copy = (MODE == MODE_FUSED) && !(p.flags & F_NO_RING);
    const bool zero_fill = (MODE == MODE_HPASS) && (p.flags & F_ZERO_FILL);

    int slot = 0;
    uint32_t phase = 0;
    long long g = 0;

    for (int item = blockIdx.x; item < p.nitems; item += gridDim.x) {
        const Item it = decode_item<MODE, RAD>(p, item);
        const int x4 = it.x0 + 4 * ct;
        float* dplane = p.dst + (long long)it.plane * p.dst_plane_stride;
        const int v_lo = max(it.ylo, RAD);
        const int v_hi = min(it.yhi, R - RAD);

        F4 acc[NACC];
#pragma unroll
        for (int j = 0; j < NACC; ++j)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[j].v[c] = 0.0f;

        for (int yi = it.in_lo; yi < it.in_hi; ++yi, ++g) {
            mbar_wait(&full[slot], phase);
            const float* srow = ring + slot * SW + 4 * ct;  // smem col 0 of this thread = x4 - 4
            float win[12];
            {
                const F4 a = ld4(srow), b = ld4(srow + 4), c = ld4(srow + 8);
#pragma unroll
                for (int i = 0; i < 4; ++i) { win[i] = a.v[i]; win[4 + i] = b.v[i]; win[8 + i] = c.v[i]; }
            }
            F4 own;
#pragma unroll
            for (int i = 0; i < 4; ++i) own.v[i] = win[4 + i];

            if (MODE == MODE_HPASS) {
                float* drow = dplane + (long long)(yi - p.dst_row0) * p.dst_row_stride;
                if (yi >= p.hrow_lo && yi < p.hrow_hi) {
                    const F4 h = row_pass<RAD>(win, p.w);
                    store_row<ALIGNED>(drow, x4, C, RAD, h, own, zero_fill ? 2 : 0);
                } else if (zero_fill) {
                    F4 z;
#pragma unroll
                    for (int i = 0; i < 4; ++i) z.v[i] = 0.0f;
                    store_row<ALIGNED>(drow, x4, C, 0, z, z, 2);
                }
            } else {
                // value entering the vertical fold for this input row
                F4 v;
                F4 outv;
                if (MODE == MODE_SINGLE) {
                    // dense fold, row-major: kernel row i of output (yi + RAD - i)
                    if (RAD == 0) {
#pragma unroll
                        for (int c = 0; c < 4; ++c) outv.v[c] = fm(win[HALO + c], p.k[0]);
                    } else {
                        constexpr int W = 2 * RAD + 1;
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            float t = acc[NACC - 1].v[c];
#pragma unroll
                            for (int j = 0; j < W; ++j) t = fa(t, fm(win[HALO - RAD + c + j], p.k[(W - 1) * W + j]));
                            outv.v[c] = t;
                        }
#pragma unroll
                        for (int i = NACC - 1; i >= 1; --i) {
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                float t = acc[i - 1].v[c];
#pragma unroll
                                for (int j = 0; j < W; ++j) t = fa(t, fm(win[HALO - RAD + c + j], p.k[i * W + j]));
                                acc[i].v[c] = t;
                            }
                        }
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            float t = fm(win[HALO - RAD + c], p.k[0]);
#pragma unroll
                            for (int j = 1; j < W; ++j) t = fa(t, fm(win[HALO - RAD + c + j], p.k[j]));
                            acc[0].v[c] = t;
                        }
                    }
                } else {
                    if (MODE == MODE_FUSED) {
                        if (yi >= p.hrow_lo && yi < p.hrow_hi) {
                            v = row_pass<RAD>(win, p.w);
                        } else {
#pragma unroll
                            for (int c = 0; c < 4; ++c) v.v[c] = 0.0f;  // faithful: scratch row stays 0
                        }
                    } else {
                        v = own;  // VPASS: src already holds the row-pass result
                    }
                    if (RAD == 0) {
#pragma unroll
                        for (int c = 0; c < 4; ++c) outv.v[c] = fm(v.v[c], p.w[0]);
                    } else {
#pragma unroll
                        for (int c = 0; c < 4; ++c) outv.v[c] = fa(acc[NACC - 1].v[c], fm(v.v[c], p.w[2 * RAD]));
#pragma unroll
                        for (int j = NACC - 1; j >= 1; --j)
#pragma unroll
                            for (int c = 0; c < 4; ++c) acc[j].v[c] = fa(acc[j - 1].v[c], fm(v.v[c], p.w[j]));
#pragma unroll
                        for (int c = 0; c < 4; ++c) acc[0].v[c] = fm(v.v[c], p.w[0]);
                    }
                }

                const int yo = yi - RAD;
                if (yo >= v_lo && yo < v_hi && yo >= it.in_lo + RAD) {
                    float* drow = dplane + (long long)(yo - p.dst_row0) * p.dst_row_stride;
                    F4 ringv;
                    if (ring_copy) {
                        int s2 = slot - LAG;
                        if (s2 < 0) s2 += NR;
                        ringv = ld4(ring + s2 * SW + 4 * ct + 4);
                    } else {
#pragma unroll
                        for (int c = 0; c < 4; ++c) ringv.v[c] = 0.0f;
                    }
                    store_row<ALIGNED>(drow, x4, C, RAD, outv, ringv, ring_copy ? 1 : 0);
                }
                if (ring_copy && yi >= it.ylo && yi < it.yhi && (yi < RAD || yi >= R - RAD)) {
                    float* drow = dplane + (long long)(yi - p.dst_row0) * p.dst_row_stride;
                    if (x4 < C) store_row<ALIGNED>(drow, x4, C, 0, own, own, 1);
                }
            }

            // release the row LAG rows back (it is no longer read by anyone)
            if (g >= LAG) {
                int s2 = slot - LAG;
                if (s2 < 0) s2 += NR;
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s2]);
            }
            if (++slot == NR) { slot = 0; phase ^= 1u; }
        }
    }
}

}  // namespace sc
