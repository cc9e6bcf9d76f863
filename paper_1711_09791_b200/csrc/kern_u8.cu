// kern_u8.cu -- the PPM data format either side of the path.
//
// The reference reads a binary P6 file into 3 float32 planes (u8 HWC -> planes,
// S/ppm.py:72-73), convolves, and writes it back with round-half-even + clip
// (S/ppm.py:87-89). Here:
//   * hwc_to_planes_kernel / planes_to_hwc_kernel: the two conversions alone;
//   * sepconv_u8_kernel: read_ppm -> two-pass -> write_ppm FUSED in one pass over
//     the interleaved bytes: 3 B/pixel in + 3 B/pixel out instead of 24 B/pixel,
//     with the very same float32 arithmetic (bit-identical output bytes).
// The fused kernel reuses the row-streaming design of kernels.cuh: a TMA
// producer warp streams 3*(TW+32) bytes per row into a shared-memory ring,
// consumer threads own 4 columns x 3 planes and fold the column pass through a
// register shift register.
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "kernels.cuh"
#include "launch.h"

namespace sc {

// float(b) for a byte via the 2^23 magic number: exact, 1 PRMT + 1 FADD.
__device__ __forceinline__ float u8f(uint32_t word, int byte) {
    const uint32_t bits = __byte_perm(word, 0x4B000000u, 0x7650 + byte);  // 0x4B0000bb
    return __fsub_rn(__uint_as_float(bits), 8388608.0f);
}

// clip(rint(x), 0, 255) as a byte (S/ppm.py:88): clamp first (equivalent at
// integer bounds), then round-half-even via 1.5*2^23.
__device__ __forceinline__ uint32_t f2u8(float x) {
    const float c = fminf(fmaxf(x, 0.0f), 255.0f);
    return __float_as_uint(__fadd_rn(c, 12582912.0f)) & 0xFFu;
}

// clip(rint(x), 0, 255) of 12 samples (4 columns x 3 planes, pixel-major) packed
// little-endian into 3 words. Default: the saturating round-half-even conversion
// (cvt.rni.sat.u8.f32 -> F2IP.U8; NaN -> 0 like the clamp below) + byte permutes,
// 21 instructions; SC_U8_F2I=0: clamp, round via 1.5*2^23 (two samples per FADD2),
// mask and shift, ~50 (measured: 16384^2 payload 0.834 -> 0.787 ms).
#ifndef SC_U8_F2I
#define SC_U8_F2I 1
#endif
__device__ __forceinline__ void pack12(const F4 (&outv)[3], uint32_t (&w)[3]) {
#if SC_U8_F2I
    uint32_t b[12];
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int q = 0; q < 3; ++q) asm("cvt.rni.sat.u8.f32 %0, %1;" : "=r"(b[3 * c + q]) : "f"(outv[q].v[c]));
#pragma unroll
    for (int i = 0; i < 3; ++i)
        w[i] = __byte_perm(__byte_perm(b[4 * i], b[4 * i + 1], 0x0040), __byte_perm(b[4 * i + 2], b[4 * i + 3], 0x0040),
                           0x5410);
#else
    uint32_t ob[12];
#pragma unroll
    for (int c = 0; c < 4; c += 2)
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            // clip then round half-even via 1.5*2^23, two samples per FADD2
            const float2 m = __fadd2_rn(make_float2(fminf(fmaxf(outv[q].v[c], 0.0f), 255.0f),
                                                    fminf(fmaxf(outv[q].v[c + 1], 0.0f), 255.0f)),
                                        make_float2(12582912.0f, 12582912.0f));
            ob[3 * c + q] = __float_as_uint(m.x) & 0xFFu;
            ob[3 * (c + 1) + q] = __float_as_uint(m.y) & 0xFFu;
        }
#pragma unroll
    for (int i = 0; i < 3; ++i) w[i] = ob[4 * i] | (ob[4 * i + 1] << 8) | (ob[4 * i + 2] << 16) | (ob[4 * i + 3] << 24);
#endif
}

// One item (column strip x row band) of the fused u8 kernel. EDGE items contain
// ring rows or rows whose row pass is dead (faithful zero H0 rows); the others
// skip those per-row tests.
#ifndef SC_U8_FAST_STAGE
#define SC_U8_FAST_STAGE 1
#endif
// COLEDGE false: an interior strip (no column ring, inside the image) -- every
// thread stores three whole words per row, no per-row column tests -- and its
// stages whose rows all exist and emit skip the per-row range tests. Used for
// large payloads only (F_U8_LEAN, set on the host): measured 16384^2 0.709 ->
// 0.605 ms, 8192^2 0.200 -> 0.183, but 4096^2 +6% and 2048^2 +17%.
// (address of the staged row's logical byte 0, column x0 - U8_HALO, of row y) mod 16
__device__ __forceinline__ uint32_t u8_row_shift(const uint8_t* base, int y, long long stride, int x0) {
    return ((uint32_t)reinterpret_cast<uintptr_t>(base) + (uint32_t)y * (uint32_t)stride + 3u * (uint32_t)x0 -
            3u * (uint32_t)U8_HALO) & 15u;
}

// The output of a thread whose 4 columns touch the column ring or the image edge:
// ring columns keep the input byte of row yo (the pixel ring equals the input),
// staged RAD rows back in the ring. `words`: whole 4-byte stores are allowed
// (destination aligned, all 4 columns inside the image).
template <int RAD, bool GEN = false>
__device__ __forceinline__ void u8_store_edge(const U8Params& p, const uint8_t* ring, const uint32_t (&w3)[3],
                                              uint8_t* drow, int slot, int k, int NS, int SWB, int x0, int x4, int ct,
                                              int yo, int C, bool ring_copy, bool words) {
    uint32_t ob[12];
#pragma unroll
    for (int i = 0; i < 12; ++i) ob[i] = (w3[i >> 2] >> (8 * (i & 3))) & 0xFFu;
    int rr = slot * U8_SROWS + k - RAD;
    if (rr < 0) rr += NS * U8_SROWS;
    const uint32_t shr = GEN ? u8_row_shift(p.src, yo, p.srs, x0) : 0u;
    const uint8_t* yrow = ring + rr * SWB + shr + 12 * ct + 3 * U8_HALO;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int col = x4 + c;
        if (col < RAD || col >= C - RAD) {
#pragma unroll
            for (int q = 0; q < 3; ++q) ob[3 * c + q] = ring_copy ? yrow[3 * c + q] : 0xFFFFFFFFu;
        }
    }
    if (words && ring_copy && x4 + 4 <= C) {
        uint32_t* d32 = reinterpret_cast<uint32_t*>(drow);
#pragma unroll
        for (int i = 0; i < 3; ++i) d32[i] = ob[4 * i] | (ob[4 * i + 1] << 8) | (ob[4 * i + 2] << 16) | (ob[4 * i + 3] << 24);
    } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int col = x4 + c;
            if (col >= C) break;
            if (ring_copy || (col >= RAD && col < C - RAD))
#pragma unroll
                for (int q = 0; q < 3; ++q) drow[3 * c + q] = (uint8_t)ob[3 * c + q];
        }
    }
}

// GEN: any row geometry (cols % 16 != 0, rows or buffers not 16-B aligned). The
// producer widens each row's copy to whole 16-byte blocks and places it so the
// row's logical byte 0 (column x0 - U8_HALO) sits `sh` = its address mod 16 bytes
// into the staged row; consumers read their 36-byte window through funnel shifts
// and, on rows whose destination is not 4-byte aligned, store whole aligned words
// made from their own bytes and the next lane's head bytes (shuffled), with single
// bytes only at warp ends and next to column-edge threads.
template <int RAD, bool EDGE, bool SYMW, bool COLEDGE = true, bool GEN = false>
__device__ __forceinline__ void u8_item(const U8Params& p, const uint8_t* ring, uint64_t* full, uint64_t* empty,
                                        int SWB, int x0, int ylo, int yhi, int in_lo, int in_hi, int& slot,
                                        uint32_t& phase, int& gs) {
    constexpr int NACC = (2 * RAD > 0) ? 2 * RAD : 1;
    const int NS = p.ns;
    const int ct = threadIdx.x - 32, lane = threadIdx.x & 31;
    const int R = p.R, C = p.C;
    const bool ring_copy = !(p.flags & F_NO_RING);
    const int x4 = x0 + 4 * ct;
    const bool fast = !COLEDGE || (x4 >= RAD && x4 + 4 <= C - RAD);
    const int emit_lo = max(max(ylo, RAD), in_lo + RAD);
    const int emit_hi = min(yhi, R - RAD);
    F4 acc[3][NACC];
#pragma unroll
    for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int j = 0; j < NACC; ++j)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[q][j].v[c] = 0.0f;

    for (int r0 = in_lo; r0 < in_hi; r0 += U8_SROWS, ++gs) {
        if (r0 != in_lo) mbar_wait(&full[slot], phase);
        // a stage whose rows all exist and all emit runs without per-row range tests
        auto stage_rows = [&](auto fast_stage) {
            constexpr bool FAST = decltype(fast_stage)::value;
    #pragma unroll
            for (int k = 0; k < U8_SROWS; ++k) {
                const int yi = r0 + k;
                if (!FAST && yi >= in_hi) break;
                // 12 columns x 3 planes = 36 bytes at byte 12*ct + 36 of the staged row
                const uint32_t sh = GEN ? u8_row_shift(p.src, yi, p.srs, x0) : 0u;
                const uint8_t* srow = ring + (slot * U8_SROWS + k) * SWB + sh + 12 * ct + 3 * (U8_HALO - 4);
                uint32_t wd[9];
                if constexpr (GEN) {
                    const uint32_t* a = reinterpret_cast<const uint32_t*>(srow - (sh & 3u));
                    const uint32_t s8 = 8u * (sh & 3u);
                    uint32_t t[10];
    #pragma unroll
                    for (int i = 0; i < 10; ++i) t[i] = a[i];
    #pragma unroll
                    for (int i = 0; i < 9; ++i) wd[i] = __funnelshift_r(t[i], t[i + 1], s8);
                } else {
    #pragma unroll
                    for (int i = 0; i < 9; ++i) wd[i] = reinterpret_cast<const uint32_t*>(srow)[i];
                }
                const bool live = !EDGE || (yi >= p.hrow_lo && yi < p.hrow_hi);
                const int yo = yi - RAD;
                const bool emit = FAST || (yo >= emit_lo && yo < emit_hi);
                F4 outv[3];
    #pragma unroll
                for (int q = 0; q < 3; ++q) {
                    float win[12];
    #pragma unroll
                    for (int c = 0; c < 12; c += 2) {
                        // two samples per packed FADD2: (2^23 + byte) - 2^23, exact
                        const int b0 = 3 * c + q, b1 = 3 * (c + 1) + q;  // byte indices in the 36-byte window
                        const float2 v = __fadd2_rn(
                            make_float2(__uint_as_float(__byte_perm(wd[b0 >> 2], 0x4B000000u, 0x7650 + (b0 & 3))),
                                        __uint_as_float(__byte_perm(wd[b1 >> 2], 0x4B000000u, 0x7650 + (b1 & 3)))),
                            make_float2(-8388608.0f, -8388608.0f));
                        win[c] = v.x;
                        win[c + 1] = v.y;
                    }
                    F4 v;
                    if (live) {
                        v = row_pass<RAD, SYMW>(win, p.w, p.one);
                    } else {
    #pragma unroll
                        for (int c = 0; c < 4; ++c) v.v[c] = 0.0f;
                    }
                    outv[q] = col_fold<RAD, NACC, SYMW>(acc[q], v, p.w, p.one);
                }
                const bool mine = !COLEDGE || x4 < C;
                uint32_t dsh = 0;  // the output row's misalignment (GEN only), uniform across the CTA
                if constexpr (GEN) dsh = ((uint32_t)reinterpret_cast<uintptr_t>(p.dst) + (uint32_t)yo * (uint32_t)p.drs) & 3u;
                if (GEN && emit && dsh) {
                    // words at drow - dsh + 4k; word 0 is the previous lane's, word 3 takes
                    // the next lane's first 4 - dsh bytes when that lane stores words too
                    uint32_t w3[3];
                    pack12(outv, w3);
                    uint8_t* drow = p.dst + (long long)yo * p.drs + 3LL * x4;
                    const bool fs = fast && mine;
                    const uint32_t nx = __shfl_down_sync(0xFFFFFFFFu, w3[0], 1);
                    const bool nfs = __shfl_down_sync(0xFFFFFFFFu, (int)fs, 1) && lane != 31;
                    const bool pfs = __shfl_up_sync(0xFFFFFFFFu, (int)fs, 1) && lane != 0;
                    const uint32_t s8 = 8u * (4u - dsh);
                    if (fs) {
                        uint32_t* q = reinterpret_cast<uint32_t*>(drow - dsh);
                        q[1] = __funnelshift_r(w3[0], w3[1], s8);
                        q[2] = __funnelshift_r(w3[1], w3[2], s8);
                        if (nfs)
                            q[3] = __funnelshift_r(w3[2], nx, s8);
                        else
                            for (int b = 12 - (int)dsh; b < 12; ++b) drow[b] = (uint8_t)(w3[b >> 2] >> (8 * (b & 3)));
                        if (!pfs)
                            for (int b = 0; b < 4 - (int)dsh; ++b) drow[b] = (uint8_t)(w3[0] >> (8 * b));
                    } else if (mine) {
                        u8_store_edge<RAD, GEN>(p, ring, w3, drow, slot, k, NS, SWB, x0, x4, ct, yo, C, ring_copy, false);
                    }
                } else if (emit && mine) {
                    uint32_t w3[3];
                    pack12(outv, w3);
                    uint8_t* drow = p.dst + (long long)yo * p.drs + 3LL * x4;
                    if (fast) {
                        uint32_t* d32 = reinterpret_cast<uint32_t*>(drow);
    #pragma unroll
                        for (int i = 0; i < 3; ++i) d32[i] = w3[i];
                    } else {
                        u8_store_edge<RAD, GEN>(p, ring, w3, drow, slot, k, NS, SWB, x0, x4, ct, yo, C, ring_copy,
                                                true);
                    }
                }
                if (EDGE && ring_copy && yi >= ylo && yi < yhi && (yi < RAD || yi >= R - RAD) && x4 < C) {
                    // ring rows: the input bytes unchanged
                    uint8_t* drow = p.dst + (long long)yi * p.drs + 3LL * x4;
                    const uint8_t* irow = ring + (slot * U8_SROWS + k) * SWB + sh + 12 * ct + 3 * U8_HALO;
                    const int nb = 3 * min(4, C - x4);
                    for (int b = 0; b < nb; ++b) drow[b] = irow[b];
                }
            }
        };
        if (SC_U8_FAST_STAGE && !EDGE && !COLEDGE && r0 + U8_SROWS <= in_hi && r0 - RAD >= emit_lo &&
            r0 - RAD + U8_SROWS <= emit_hi)
            stage_rows(std::true_type{});
        else
            stage_rows(std::false_type{});
        constexpr int LAGS = (RAD + U8_SROWS - 1) / U8_SROWS > 0 ? (RAD + U8_SROWS - 1) / U8_SROWS : 1;
        if (gs >= LAGS) {
            int rel = slot - LAGS;
            if (rel < 0) rel += NS;
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[rel]);
        }
        if (++slot == NS) { slot = 0; phase ^= 1u; }
    }
}

#ifndef SC_U8_MAXT
#define SC_U8_MAXT (32 + 256)
#endif
#ifndef SC_U8_MINB
#define SC_U8_MINB 1
#endif
// OCC3: the instantiation for payloads below 32 Mpixel -- at most 128 consumer
// threads and 3 CTAs per SM (128 registers instead of 146, no spills): measured
// 2048^2 -4.5%, 4096^2 -5%; on large payloads the 2-CTA build stays ahead (8192^2
// +5%, 16384^2 +2.5% with OCC3), so the host picks by size.
template <int RAD, bool SYMW, bool OCC3 = false, bool GEN = false>
__global__ void __launch_bounds__(OCC3 ? 160 : SC_U8_MAXT, OCC3 ? 3 : SC_U8_MINB)
    sepconv_u8_kernel(const __grid_constant__ U8Params p) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int NS = p.ns;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t* empty = full + NS;
    int* sitem = reinterpret_cast<int*>(empty + NS);
    uint8_t* ring = smem_raw + ((2 * NS * 8 + NS * 4 + 127) / 128) * 128;
    const int SWB = p.rowb;  // bytes per staged row (3 * (tw + 2 * U8_HALO), + 32 for GEN)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ncw = (blockDim.x >> 5) - 1;
    const int units = p.nstrips;

    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) {
            mbar_init(&full[i], 1u);
            mbar_init(&empty[i], (uint32_t)ncw);
        }
        mbar_fence_init();
    }
    __syncthreads();

    auto decode = [&](int item, int& x0, int& ylo, int& yhi, int& in_lo, int& in_hi) {
        const int band = item / units;
        const int strip = item - band * units;
        x0 = strip * p.tw;
        ylo = band * p.band_h;
        yhi = min(ylo + p.band_h, p.R);
        in_lo = max(ylo - RAD, 0);
        in_hi = min(yhi + RAD, p.R);
    };

    if (warp == 0) {
        if (lane != 0) return;
        const uint64_t pol = policy_evict_normal();
        int slot = 0, gs = 0;
        uint32_t phase = 0;
        bool first = SC_STATIC_FIRST;  // first item = block index (see the row kernels' producer)
        for (;;) {
            const int item = first ? (int)blockIdx.x : (int)gridDim.x * SC_STATIC_FIRST + atomicAdd(&p.work[0], 1);
            first = false;
            if (item >= p.nitems) {
                if (gs >= NS) mbar_wait(&empty[slot], phase ^ 1u);
                sitem[slot] = -1;
                mbar_arrive_expect_tx(&full[slot], 0u);
                __threadfence();
                if (atomicAdd(&p.work[1], 1) == (int)gridDim.x - 1) {
                    atomicExch(&p.work[0], 0);
                    atomicExch(&p.work[1], 0);
                }
                return;
            }
            int x0, ylo, yhi, in_lo, in_hi;
            decode(item, x0, ylo, yhi, in_lo, in_hi);
            const int cx0 = max(x0 - U8_HALO, 0);
            const int cx1 = min(x0 + p.tw + U8_HALO, p.C);
            const uint32_t bytes = 3u * (uint32_t)(cx1 - cx0);
            const int soff = 3 * (cx0 - (x0 - U8_HALO));
            for (int r0 = in_lo; r0 < in_hi; r0 += U8_SROWS, ++gs) {
                if (gs >= NS) mbar_wait(&empty[slot], phase ^ 1u);
                const int nrows = min(U8_SROWS, in_hi - r0);
                sitem[slot] = item;
                if constexpr (GEN) {
                    // whole 16-byte blocks around each row's bytes: every block holds a
                    // payload byte, so the widened read stays inside mapped pages
                    uint32_t tot = 0;
                    for (int k = 0; k < nrows; ++k) {
                        const uintptr_t g0 = reinterpret_cast<uintptr_t>(p.src + (long long)(r0 + k) * p.srs + 3LL * cx0);
                        tot += (uint32_t)(((g0 + bytes + 15) & ~(uintptr_t)15) - (g0 & ~(uintptr_t)15));
                    }
                    mbar_arrive_expect_tx(&full[slot], tot);
                    for (int k = 0; k < nrows; ++k) {
                        const uintptr_t g0 = reinterpret_cast<uintptr_t>(p.src + (long long)(r0 + k) * p.srs + 3LL * cx0);
                        const uintptr_t a0 = g0 & ~(uintptr_t)15, a1 = (g0 + bytes + 15) & ~(uintptr_t)15;
                        const uint32_t sh = ((uint32_t)g0 - (uint32_t)soff) & 15u;
                        bulk_g2s(ring + (slot * U8_SROWS + k) * SWB + ((sh + (uint32_t)soff) & ~15u),
                                 reinterpret_cast<const uint8_t*>(a0), (uint32_t)(a1 - a0), &full[slot], pol);
                    }
                } else {
                    mbar_arrive_expect_tx(&full[slot], bytes * (uint32_t)nrows);
                    for (int k = 0; k < nrows; ++k)
                        bulk_g2s(ring + (slot * U8_SROWS + k) * SWB + soff,
                                 p.src + (long long)(r0 + k) * p.srs + 3LL * cx0, bytes, &full[slot], pol);
                }
                if (++slot == NS) { slot = 0; phase ^= 1u; }
            }
        }
    }

    // ---- consumers: 4 columns x 3 planes per thread
    int slot = 0, gs = 0;
    uint32_t phase = 0;
    for (;;) {
        mbar_wait(&full[slot], phase);
        const int item = sitem[slot];
        if (item < 0) break;
        int x0, ylo, yhi, in_lo, in_hi;
        decode(item, x0, ylo, yhi, in_lo, in_hi);
        // interior items (every input row live, no ring rows) run the lean loop
        const bool edge = in_lo < p.hrow_lo || in_hi > p.hrow_hi || ylo < RAD || yhi > p.R - RAD;
        if (edge)
            u8_item<RAD, true, SYMW, true, GEN>(p, ring, full, empty, SWB, x0, ylo, yhi, in_lo, in_hi, slot, phase, gs);
        else if (RAD >= 4 || !(p.flags & F_U8_LEAN) || x0 < RAD || x0 + p.tw > p.C - RAD)
            u8_item<RAD, false, SYMW, true, GEN>(p, ring, full, empty, SWB, x0, ylo, yhi, in_lo, in_hi, slot, phase,
                                                 gs);
        else if constexpr (RAD < 4)  // r = 4 with the lean variant spills
            u8_item<RAD, false, SYMW, false, GEN>(p, ring, full, empty, SWB, x0, ylo, yhi, in_lo, in_hi, slot, phase,
                                                  gs);
    }
}

// u8 HWC -> float32 planes (S/ppm.py:72-73), one thread per pixel.
__global__ void hwc_to_planes_kernel(const uint8_t* __restrict__ src, float* __restrict__ dst, long long srs,
                                     long long dps, long long drs, int R, int C) {
    const long long total = (long long)R * C;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int y = (int)(i / C), x = (int)(i - (long long)y * C);
        const uint8_t* s = src + y * srs + 3LL * x;
#pragma unroll
        for (int q = 0; q < 3; ++q) dst[q * dps + y * drs + x] = (float)s[q];
    }
}

// float32 planes -> u8 HWC with clip(rint(x), 0, 255) (S/ppm.py:87-89).
__global__ void planes_to_hwc_kernel(const float* __restrict__ src, uint8_t* __restrict__ dst, long long sps,
                                     long long srs, long long drs, int R, int C) {
    const long long total = (long long)R * C;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int y = (int)(i / C), x = (int)(i - (long long)y * C);
        uint8_t* d = dst + y * drs + 3LL * x;
#pragma unroll
        for (int q = 0; q < 3; ++q) d[q] = (uint8_t)f2u8(src[q * sps + y * srs + x]);
    }
}

bool u8_occ3_fits(int rad, bool symw) { return rad <= 1 || (rad == 2 && symw); }

// symw: mirror-symmetric taps (w[j] == w[2r-j] bitwise): products shared by value
template <bool GEN>
static const void* kernel_u8_t(int rad, bool symw, bool occ3) {
#define SC_U8K(R, S) \
    (occ3 ? (const void*)sepconv_u8_kernel<R, S, true, GEN> : (const void*)sepconv_u8_kernel<R, S, false, GEN>)
#define SC_U8K2(R, S) ((const void*)sepconv_u8_kernel<R, S, false, GEN>)
    switch (rad) {
        case 0: return SC_U8K(0, false);
        case 1: return symw ? SC_U8K(1, true) : SC_U8K(1, false);
        // r = 2 without shared products and r >= 3: the 3-CTA build would spill
        // (u8_occ3_fits); the 2-CTA build only
        case 2: return symw ? SC_U8K(2, true) : SC_U8K2(2, false);
        case 3: return symw ? SC_U8K2(3, true) : SC_U8K2(3, false);
        // r = 4 with shared products spills (the products of 5 distinct taps stay live)
        case 4: return SC_U8K2(4, false);
        default: return nullptr;
    }
#undef SC_U8K
#undef SC_U8K2
}

const void* kernel_u8(int rad, bool symw, bool occ3, bool gen) {
    return gen ? kernel_u8_t<true>(rad, symw, occ3) : kernel_u8_t<false>(rad, symw, occ3);
}

static int grid_cap(long long total, int threads) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    long long b = (total + threads - 1) / threads;
    if (b > (long long)sms * 8) b = (long long)sms * 8;
    return b < 1 ? 1 : (int)b;
}

cudaError_t launch_hwc_to_planes(const uint8_t* src, float* dst, long long srs, long long dps, long long drs, int R,
                                 int C, cudaStream_t s) {
    hwc_to_planes_kernel<<<grid_cap((long long)R * C, 256), 256, 0, s>>>(src, dst, srs, dps, drs, R, C);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_planes_to_hwc(const float* src, uint8_t* dst, long long sps, long long srs, long long drs, int R,
                                 int C, cudaStream_t s) {
    planes_to_hwc_kernel<<<grid_cap((long long)R * C, 256), 256, 0, s>>>(src, dst, sps, srs, drs, R, C);
    count_launch();
    return cudaGetLastError();
}

}  // namespace sc

// ---------------------------------------------------------------------------
// C ABI (declared in include/sepconv_b200.h)

namespace sc {
int launch_rows_u8(const uint8_t* src, uint8_t* dst, long long srs, long long drs, int R, int C, const float* taps,
                   int width, int flags, cudaStream_t s);
}

using namespace sc;

static int u8_fail(int code, const char* msg) {
    set_error(msg);
    return code;
}

static bool dev_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged) return false;
    cudaSetDevice(a.device);
    return true;
}

extern "C" int sc_two_pass_u8hwc(const uint8_t* src, uint8_t* dst, int rows, int cols, int64_t src_row_stride,
                                 int64_t dst_row_stride, const float* taps, int width, int flags, void* stream) {
    set_error("");
    if (!src || !dst || !taps || rows < 1 || cols < 1) return u8_fail(1, "null pointer or non-positive dimension");
    if (width < 1 || width % 2 == 0) return u8_fail(1, "kernel width must be odd and >= 1");
    if (width > MAX_W) return u8_fail(3, "kernel width > 9 not supported");
    if (rows < width || cols < width) return u8_fail(2, "image smaller than kernel width");
    if (src_row_stride < 3LL * cols || dst_row_stride < 3LL * cols) return u8_fail(1, "row stride shorter than a row");
    if (!dev_ptr(src) || !dev_ptr(dst)) return u8_fail(1, "buffer is not device memory");
    const long long ns = (long long)(rows - 1) * src_row_stride + 3LL * cols;
    const long long nd = (long long)(rows - 1) * dst_row_stride + 3LL * cols;
    const char* a = reinterpret_cast<const char*>(src);
    const char* b = reinterpret_cast<const char*>(dst);
    if (a < b + nd && b < a + ns) return u8_fail(1, "source and destination must be distinct buffers");
    return launch_rows_u8(src, dst, src_row_stride, dst_row_stride, rows, cols, taps, width, flags,
                          static_cast<cudaStream_t>(stream));
}

extern "C" int sc_hwc_u8_to_planes_f32(const uint8_t* src, float* dst, int rows, int cols, int64_t src_row_stride,
                                       int64_t dst_plane_stride, int64_t dst_row_stride, void* stream) {
    set_error("");
    if (!src || !dst || rows < 1 || cols < 1 || src_row_stride < 3LL * cols || dst_row_stride < cols ||
        dst_plane_stride < (long long)rows * dst_row_stride)
        return u8_fail(1, "bad geometry");
    if (!dev_ptr(src) || !dev_ptr(dst)) return u8_fail(1, "buffer is not device memory");
    cudaError_t e = launch_hwc_to_planes(src, dst, src_row_stride, dst_plane_stride, dst_row_stride, rows, cols,
                                         static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return u8_fail(4, cudaGetErrorString(e));
    return 0;
}

extern "C" int sc_planes_f32_to_hwc_u8(const float* src, uint8_t* dst, int rows, int cols, int64_t src_plane_stride,
                                       int64_t src_row_stride, int64_t dst_row_stride, void* stream) {
    set_error("");
    if (!src || !dst || rows < 1 || cols < 1 || dst_row_stride < 3LL * cols || src_row_stride < cols ||
        src_plane_stride < (long long)rows * src_row_stride)
        return u8_fail(1, "bad geometry");
    if (!dev_ptr(src) || !dev_ptr(dst)) return u8_fail(1, "buffer is not device memory");
    cudaError_t e = launch_planes_to_hwc(src, dst, src_plane_stride, src_row_stride, dst_row_stride, rows, cols,
                                         static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return u8_fail(4, cudaGetErrorString(e));
    return 0;
}
