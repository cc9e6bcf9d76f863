// direct.cuh -- register-streaming variant of the row kernels (no shared memory).
//
// One warp owns a 128-column strip of one plane and walks a band of rows:
// each lane loads its own 4 columns per row with LDG.128 (lane 0 / lane 31 also
// load the float4 just left / right of the strip), gets its neighbours' halo
// columns with warp shuffles, and runs the same per-row arithmetic as the TMA
// kernel (row_pass / col_fold / dense_fold: identical bits). Rows are loaded
// U at a time, one batch ahead of the batch being computed, so every warp keeps
// 2U row loads in flight; warps claim (plane, strip, band) items from an atomic
// ticket, so no SM idles at the tail.
#pragma once

#include <type_traits>

#include "kernels.cuh"

namespace sc {

#ifndef SC_DU
#define SC_DU 2
#endif
#ifndef SC_DMINB
#define SC_DMINB 2
#endif
constexpr int DU = SC_DU;    // rows per load batch
constexpr int DWARPS = 8;    // warps per CTA (independent workers)

template <int RAD>
struct RowRegs {
    float4 own[DU];
    // lane 0: the columns just left of the strip; lane 31: just right of it
    // (2 columns suffice for r <= 2, 4 for r <= 4)
    typename std::conditional<(RAD <= 2), float2, float4>::type ext[DU];
};

__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

template <int MODE, int RAD>
__device__ __forceinline__ void direct_load(RowRegs<RAD>& rr, const float* rowp, int yi, int in_hi, long long srs,
                                            int x4, int C, int lane, bool left_ok, bool right_ok) {
#pragma unroll
    for (int k = 0; k < DU; ++k) {
        const float* q = rowp + (long long)k * srs;
        const bool live = (yi + k) < in_hi;
        rr.own[k] = (live && x4 < C) ? ldg4(q + x4) : make_float4(0.f, 0.f, 0.f, 0.f);
        if (MODE != MODE_VPASS && RAD > 0) {
            const bool e = live && ((lane == 0 && left_ok) || (lane == 31 && right_ok));
            if constexpr (RAD <= 2) {
                const float* a = q + (lane == 0 ? x4 - 2 : x4 + 4);
                rr.ext[k] = e ? __ldg(reinterpret_cast<const float2*>(a)) : make_float2(0.f, 0.f);
            } else {
                rr.ext[k] = e ? ldg4(q + (lane == 0 ? x4 - 4 : x4 + 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
    }
}

// Build the 12-sample window (columns x4-4 .. x4+7) of row k from registers + shuffles.
template <int MODE, int RAD>
__device__ __forceinline__ void direct_window(float (&win)[12], const RowRegs<RAD>& rr, int k, int lane) {
    const float4 o = rr.own[k];
    win[4] = o.x; win[5] = o.y; win[6] = o.z; win[7] = o.w;
    if (MODE == MODE_VPASS || RAD == 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) { win[i] = 0.f; win[8 + i] = 0.f; }
        return;
    }
    float4 l, r;
    l.x = __shfl_up_sync(0xffffffffu, o.x, 1);
    l.y = __shfl_up_sync(0xffffffffu, o.y, 1);
    l.z = __shfl_up_sync(0xffffffffu, o.z, 1);
    l.w = __shfl_up_sync(0xffffffffu, o.w, 1);
    r.x = __shfl_down_sync(0xffffffffu, o.x, 1);
    r.y = __shfl_down_sync(0xffffffffu, o.y, 1);
    r.z = __shfl_down_sync(0xffffffffu, o.z, 1);
    r.w = __shfl_down_sync(0xffffffffu, o.w, 1);
    if constexpr (RAD <= 2) {
        const auto e = rr.ext[k];
        if (lane == 0) { l.z = reinterpret_cast<const float*>(&e)[0]; l.w = reinterpret_cast<const float*>(&e)[1]; }
        if (lane == 31) { r.x = reinterpret_cast<const float*>(&e)[0]; r.y = reinterpret_cast<const float*>(&e)[1]; }
    } else {
        const auto e = rr.ext[k];
        const float* ep = reinterpret_cast<const float*>(&e);
        if (lane == 0) l = make_float4(ep[0], ep[1], ep[2], ep[3]);
        if (lane == 31) r = make_float4(ep[0], ep[1], ep[2], ep[3]);
    }
    win[0] = l.x; win[1] = l.y; win[2] = l.z; win[3] = l.w;
    win[8] = r.x; win[9] = r.y; win[10] = r.z; win[11] = r.w;
}

template <int MODE, int RAD>
__global__ void __launch_bounds__(32 * DWARPS, SC_DMINB) sepconv_direct_kernel(const __grid_constant__ Params p) {
    constexpr int NACC = (2 * RAD > 0) ? 2 * RAD : 1;
    const int lane = threadIdx.x & 31;
    const int R = p.R, C = p.C;
    const bool ring_copy = (MODE == MODE_FUSED) && !(p.flags & F_NO_RING);
    const bool zero_fill = (MODE == MODE_HPASS) && (p.flags & F_ZERO_FILL);
    // launched with programmatic stream serialization (capi.cu): wait for the
    // previous kernel on the stream before touching global memory
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (;;) {
        int item = 0;
        if (lane == 0) item = atomicAdd(&p.work[0], 1);
        item = __shfl_sync(0xffffffffu, item, 0);
        if (item >= p.nitems) break;
        const Item it = decode_item<MODE, RAD>(p, item);
        const int x4 = it.x0 + 4 * lane;
        const bool fast = x4 >= RAD && x4 + 4 <= C - RAD;
        const bool left_ok = it.x0 >= 4;
        const bool right_ok = it.x0 + 128 + 4 <= C;
        const float* splane = p.src + (long long)it.plane * p.src_plane_stride;
        float* dplane = p.dst + (long long)it.plane * p.dst_plane_stride;
        const bool row_edge = item_rows_edge<MODE, RAD>(p, it);
        int emit_lo, emit_hi;
        if (MODE == MODE_HPASS) {
            emit_lo = it.ylo;
            emit_hi = it.yhi;
        } else {
            emit_lo = max(max(it.ylo, RAD), it.in_lo + RAD);
            emit_hi = min(it.yhi, R - RAD);
        }
        float* dcur = dplane + (long long)(emit_lo - p.dst_row0) * p.dst_row_stride;

        F4 acc[NACC];
#pragma unroll
        for (int j = 0; j < NACC; ++j)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[j].v[c] = 0.0f;
        // ring-column values of the last RAD input rows (FUSED edge lanes)
        F4 hist[RAD > 0 ? RAD : 1];
#pragma unroll
        for (int j = 0; j < (RAD > 0 ? RAD : 1); ++j)
#pragma unroll
            for (int c = 0; c < 4; ++c) hist[j].v[c] = 0.0f;

        RowRegs<RAD> A, B;
        const float* rowp = splane + (long long)(it.in_lo - p.src_row0) * p.src_row_stride;
        direct_load<MODE, RAD>(A, rowp, it.in_lo, it.in_hi, p.src_row_stride, x4, C, lane, left_ok, right_ok);

        auto run_batch = [&](const RowRegs<RAD>& rr, int y0) {
#pragma unroll
            for (int k = 0; k < DU; ++k) {
                const int yi = y0 + k;
                if (yi >= it.in_hi) break;
                float win[12];
                direct_window<MODE, RAD>(win, rr, k, lane);
                F4 own;
#pragma unroll
                for (int i = 0; i < 4; ++i) own.v[i] = win[4 + i];
                const bool live = !row_edge || (yi >= p.hrow_lo && yi < p.hrow_hi);
                const int yo = (MODE == MODE_HPASS) ? yi : yi - RAD;
                const bool emit = yo >= emit_lo && yo < emit_hi;
                F4 outv;
                if (MODE == MODE_HPASS) {
                    if (live) {
                        outv = row_pass<RAD>(win, p.w, p.one);
                    } else {
#pragma unroll
                        for (int i = 0; i < 4; ++i) outv.v[i] = 0.0f;
                    }
                    if (emit && (live || zero_fill)) {
                        if (fast && live)
                            st4(dcur + x4, outv);
                        else
                            store_edge(dcur, x4, C, live ? RAD : 0, outv, own, zero_fill ? 2 : 0);
                    }
                } else {
                    if (MODE == MODE_SINGLE) {
                        outv = dense_fold<RAD, NACC>(acc, win, p.k, p.one);
                    } else {
                        F4 v;
                        if (MODE == MODE_FUSED) {
                            if (live) {
                                v = row_pass<RAD>(win, p.w, p.one);
                            } else {
#pragma unroll
                                for (int i = 0; i < 4; ++i) v.v[i] = 0.0f;
                            }
                        } else {
                            v = own;
                        }
                        outv = col_fold<RAD, NACC>(acc, v, p.w, p.one);
                    }
                    if (emit) {
                        if (fast) {
                            st4(dcur + x4, outv);
                        } else {
                            F4 ringv = (RAD > 0) ? hist[RAD > 0 ? RAD - 1 : 0] : own;
                            store_edge(dcur, x4, C, RAD, outv, ringv, ring_copy ? 1 : 0);
                        }
                    }
                    if (ring_copy && row_edge && yi >= it.ylo && yi < it.yhi && (yi < RAD || yi >= R - RAD)) {
                        float* drow = dplane + (long long)(yi - p.dst_row0) * p.dst_row_stride;
                        store_edge(drow, x4, C, 0, own, own, 1);
                    }
                    if (MODE == MODE_FUSED && RAD > 0 && !fast) {
#pragma unroll
                        for (int j = (RAD > 0 ? RAD - 1 : 0); j >= 1; --j) hist[j] = hist[j - 1];
                        hist[0] = own;
                    }
                }
                if (emit) dcur += p.dst_row_stride;
            }
        };

        for (int y0 = it.in_lo; y0 < it.in_hi; y0 += 2 * DU) {
            const float* rp1 = rowp + (long long)(y0 + DU - it.in_lo) * p.src_row_stride;
            if (y0 + DU < it.in_hi)
                direct_load<MODE, RAD>(B, rp1, y0 + DU, it.in_hi, p.src_row_stride, x4, C, lane, left_ok, right_ok);
            run_batch(A, y0);
            if (y0 + DU >= it.in_hi) break;
            const float* rp2 = rowp + (long long)(y0 + 2 * DU - it.in_lo) * p.src_row_stride;
            if (y0 + 2 * DU < it.in_hi)
                direct_load<MODE, RAD>(A, rp2, y0 + 2 * DU, it.in_hi, p.src_row_stride, x4, C, lane, left_ok,
                                       right_ok);
            run_batch(B, y0 + DU);
        }
    }
    // the last warp out re-arms the ticket pair
    if (lane == 0) {
        __threadfence();
        const int total = (int)(gridDim.x * (blockDim.x >> 5));
        if (atomicAdd(&p.work[1], 1) == total - 1) {
            atomicExch(&p.work[0], 0);
            atomicExch(&p.work[1], 0);
        }
    }
}

}  // namespace sc
