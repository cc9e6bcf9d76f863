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
//   MODE_SPLITF conv_two_pass with the reference's buffer end state (scratch :=
//               H0, image[valid] := V(H0) in place), fused: one read of the
//               image, one write of scratch, one write of the image. Samples of
//               OTHER items' regions (row and column halos) come from a
//               snapshot taken before the launch (split_snapshot_kernel), since
//               their owners overwrite them in place.
//   MODE_SINGLECB the single pass with copy-back (S/executors.py:330-331) in one
//               pass: the valid region goes to the workspace AND back into the
//               image in place, halos from the same snapshot.
//
// Work decomposition: an "item" is (plane, column strip of TW = 4*GROUPS*NT
// output columns, row band). A persistent grid claims items from an atomic
// ticket (dynamic scheduling); the planner in capi.cu picks TW and the band
// schedule. Launches use programmatic dependent launch (griddepcontrol).
// Per CTA:
//   warp 0      producer (one lane): streams input rows [x0-4, x0+TW+4) of the
//               strip into a ring of NS shared-memory stages x SROWS rows with
//               the bulk-copy TMA engine (cp.async.bulk + mbarrier complete_tx),
//               from this band's buffer or -- for halo rows of a multi-GPU
//               band -- from a neighbouring band's peer-mapped buffer. Unaligned
//               rows are copied from the 16-B boundary below them and their
//               shift is published in shared memory.
//   warps 1..   consumers: thread t owns GROUPS 4-column groups (strip offsets
//               4t + g*TW/GROUPS; one group for the two-pass modes, two for the
//               single pass). Per input row and group it reads a 12-sample
//               window (3 x LDS.128), computes the row pass for its 4 columns
//               and pushes them through a shift register of 2r partial column
//               sums, emitting output row y-r as soon as input row y arrived.
//               Results go straight to HBM with STG.128. Rows of any other
//               alignment (cols % 4 != 0, misaligned views): thread (warp q,
//               lane l) owns columns 128q + l + 32i instead -- conflict-free
//               LDS.32 at any shift, STG.32 with 128 contiguous bytes per warp
//               (consume_item_lanes).
//
// Bit-exactness: every product/sum is __fmul_rn/__fadd_rn (never contracted to
// FMA) in the reference's fold order: left-to-right from the first product,
// kernel rows outer, kernel columns inner (S/conv.py:1-15). The shift register
// preserves that order because input rows arrive in increasing order, which is
// exactly the order of the terms of each output's fold.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

namespace sc {

enum Mode : int { MODE_FUSED = 0, MODE_HPASS = 1, MODE_VPASS = 2, MODE_SINGLE = 3, MODE_SPLITF = 4, MODE_SINGLECB = 5 };
// modes that run the row pass on the staged input and fold it down the columns
__host__ __device__ constexpr bool fused_like(int mode) { return mode == MODE_FUSED || mode == MODE_SPLITF; }
__host__ __device__ constexpr bool single_like(int mode) { return mode == MODE_SINGLE || mode == MODE_SINGLECB; }
// modes that overwrite their own source in place: other items' halos come from the snapshot
__host__ __device__ constexpr bool snap_mode(int mode) { return mode == MODE_SPLITF || mode == MODE_SINGLECB; }

// flags (mirrors include/sepconv_b200.h)
constexpr int F_EXTENDED = 0x1;
constexpr int F_NO_RING = 0x2;
constexpr int F_ZERO_FILL = 0x4;
// tuning flags (set by the planner from SC_* environment variables)
constexpr int SIG_WORDS = 8;  // signal block: [0] ready, [2]/[3] done counts above/below, [4]/[5] per-launch targets
constexpr int F_U8_LEAN = 0x400;  // u8 kernel: interior strips take the lean loops (large payloads)
constexpr int F_L2_EVICT_FIRST = 0x100;  // evict_first hint on the row loads (default: evict_normal,
                                         // which lets neighbouring bands' halo rows hit in L2)

constexpr int HALO = 4;       // smem columns kept either side of a strip (supports r <= 4)
constexpr int MAX_RAD = 4;
constexpr int MAX_W = 2 * MAX_RAD + 1;
constexpr int MAX_W_WIDE = 255;  // widths 33..255 run the plain kernels of kern_wide.cu
// widths 11..31 (r = 5..15): the lane-strided consumer (consume_item_lanes) with a
// wider smem halo and the taps in ParamsW -- its window is streamed from shared
// memory tap by tap, so only the column fold's 2r partial sums live in registers
constexpr int MAX_RAD_LANES = 15;
constexpr int MAX_RAD_ADJ = 10;           // aligned rows, two-pass modes: the adjacent-column consumer up to 21 taps
constexpr int MAX_RAD_LANES_SINGLE = 10;  // the dense fold: up to 21 x 21 (wider ones spill)
constexpr int MAX_W_LANES = 2 * MAX_RAD_LANES + 1;
// smem columns kept either side of a strip: a multiple of 4 (16-B copies) >= r
__host__ __device__ constexpr int halo_of(int rad) { return rad <= 4 ? 4 : ((rad + 3) / 4) * 4; }
constexpr int MAX_THREADS = 32 + 256;  // producer warp + up to 8 consumer warps
#ifndef SC_MAXT
#define SC_MAXT MAX_THREADS
#endif

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
    int out_lo2, out_hi2;    // optional second output segment (empty if lo2 >= hi2)
    int nitems0;             // items of the first segment; the rest belong to the second
    int hrow_lo, hrow_hi;    // rows where the row pass is live (else H0 = 0 / zero fill)
    int flags;
    int tw;                  // strip width = 8 * consumer threads (two 4-column groups each)
    int nstrips, band_h, nitems;
    int band_h2;             // band height of the second segment
    int ns;                  // smem stages (SROWS rows each)
    float one;               // 1.0f, passed at run time (see mad2)
    int* work;               // [next item, finished CTAs]: dynamic scheduling ticket pair (zero at launch)
    unsigned long long* trace;  // SC_TRACE builds only: per-CTA timeline (else null)
    // Input rows the producer may fetch: [avail_lo, avail_hi). Rows of that range
    // outside src's own [src_row0, src_row0 + src_rows) come from the neighbouring
    // bands `above` / `below` (other GPUs' buffers mapped over NVLink, multi.py
    // PeerBandStepper): the halo exchange is the kernel's own TMA reads.
    int avail_lo, avail_hi;
    const float* above;
    const float* below;
    long long above_ps, above_rs, below_ps, below_rs;
    int above_row0, below_row0;  // global row of row 0 of above / below
    // MODE_SPLITF: the scratch planes (global rows, H0 written for every own row);
    // MODE_SINGLECB: the image (second destination of the valid region). Both:
    // rows [snap_lo, snap_hi) are written by some item (outside them the image is
    // never written and is read directly), and the halo snapshot: side_rows[((plane * side_nb + b) * 2r + t) * C + x] =
    // image row lo_b - r + t of band boundary b (b = band ordinal >= 1, lo_b its
    // first row); side_cols[((plane * (nstrips - 1) + s - 1) * R + y) * 8 + i] =
    // image column s * tw - 4 + i of row y (strip boundary s >= 1)
    float* scr;
    long long scr_ps, scr_rs;
    const float* side_rows;
    const float* side_cols;
    int side_nb;
    float w[MAX_W];
    float k[MAX_W * MAX_W];
    // last: inserting fields before w/k shifts the taps' constant-bank offsets,
    // which measurably changes register allocation (fused 76 -> 84, unaligned 96 -> 102)
    int snap_lo, snap_hi;
    // Row-band readiness signalling between ranks (peer transport, epoch > 0):
    // sig_self = this band's signal words in its own device memory (mapped by the
    // neighbours): [0] ready epoch; [2] / [3] running counts of the items that
    // have finished reading the band above / below; [4] / [5] how many items read
    // it per launch (sig_n_above / sig_n_below, fixed by the plan). sig_above /
    // sig_below = the neighbours' words (peer-mapped, may be null). CTA 0
    // publishes ready = epoch when the grid starts (its inputs are in place:
    // stream order; the grid is resident and nothing it waits for depends on
    // it); every CTA waits until both neighbours published ready >= epoch before
    // its first neighbour read or any write (their halo rows are current; and a
    // neighbour that started this step has finished the previous one, so buffers
    // it read then may be overwritten). "Done reading my rows" for epoch e is
    // count >= e * n on the neighbour's side: each neighbour-reading item adds 1
    // once its copies landed. Only those items (one band of strips at each end)
    // count, early and late in the launch -- a per-launch counter that every CTA
    // bumped at its end cost 4 us per step (measured), per-CTA done words 6 us. sig_err (host-mapped) is
    // set if a wait outlives sig_timeout_ns.
    unsigned long long* sig_self;
    const unsigned long long* sig_above;
    const unsigned long long* sig_below;
    unsigned long long epoch;
    unsigned int* sig_err;
    long long sig_timeout_ns;
    unsigned long long sig_n_above, sig_n_below;
};

// Parameters of the widths 11..31 kernels: Params plus their taps (kept out of
// Params so the r <= 4 kernels' parameter block, and their launch cost, stay as they are).
struct ParamsW : Params {
    float wide_w[MAX_W_LANES];
    float wide_k[MAX_W_LANES * MAX_W_LANES];
};

// SC_TRACE (a dev-only build variant): per-CTA timeline of TRACE_SLOTS words.
//   [0] globaltimer at start, [1] clock64 at start, [2..9] clock64 when the
//   producer's claim for item i returned, [10..17] item ids, [20..27] clock64 when
//   the consumers saw item i's first stage, [30..37] clock64 when they finished it,
//   [40] clock64 at consumer exit, [41] globaltimer at exit, [42] items, [43] smid,
//   [48..55] clock64 when stage s (CTA-wide count) was ready, [56..63] when it was done
constexpr int TRACE_SLOTS = 64;
#ifdef SC_TRACE
__device__ __forceinline__ unsigned long long trace_gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define SC_TR(p, idx, val) \
    do { if ((p).trace) (p).trace[(size_t)blockIdx.x * TRACE_SLOTS + (idx)] = (unsigned long long)(val); } while (0)
#else
#define SC_TR(p, idx, val) do { } while (0)
#endif

// Interleaved-u8 (PPM payload) fused path, csrc/kern_u8.cu
constexpr int U8_HALO = 16;   // columns either side of a strip (16*3 bytes keeps TMA 16-B aligned)
constexpr int U8_SROWS = 4;

struct U8Params {
    const uint8_t* src;
    uint8_t* dst;
    long long srs, drs;  // row strides in BYTES
    int R, C;
    int hrow_lo, hrow_hi;
    int flags;
    int tw, nstrips, band_h, nitems, ns;
    int rowb;  // bytes per staged row in the ring
    float w[MAX_W];
    float one;
    int* work;
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

// Transaction count without an arrival: the phase also needs a later mbar_arrive.
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t tx) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(tx) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(tx)
                 : "memory");
}

#ifndef SC_WAIT_HINT
#define SC_WAIT_HINT 0  // ns; > 0: try_wait suspends the thread up to this long per poll
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if SC_WAIT_HINT > 0
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "SC_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra SC_WAIT;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "n"(SC_WAIT_HINT)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "SC_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra SC_WAIT;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
#endif
}

__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(sdst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// System-scope release / acquire on 64-bit signal words (peer memory over NVLink).
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// A system-scope count without a fence: used only after the counted reads have
// COMPLETED (their mbarrier phase was waited, the data is in shared memory), so no
// later write by the reader's neighbour can reach them; a release here stalled the
// counting warp behind every earlier store of its item (+5 us per step, measured).
__device__ __forceinline__ void red_add_relaxed_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Spin until *flag >= value (acquire, system scope); on timeout flag the error word
// and go on (a hung neighbour must not hang this GPU).
static __device__ __noinline__ void wait_signal(const unsigned long long* flag, unsigned long long value,
                                         unsigned int* err, long long timeout_ns) {
    if (!flag) return;
    const unsigned long long t0 = global_ns();
    unsigned ns = 32;
    while (ld_acquire_sys(flag) < value) {
        if ((long long)(global_ns() - t0) > timeout_ns) {
            if (err) atomicExch_system(err, 1u);
            return;
        }
        __nanosleep(ns);
        if (ns < 1024) ns *= 2;
    }
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

// acc + x*w as two IEEE roundings (mul, then add), packed two columns wide.
// ptxas (CUDA 12.9) contracts mul.rn.f32x2 + add.rn.f32x2 into one FFMA2 with a
// single rounding -- which would break parity -- so the add is issued as an
// FFMA2 by a RUN-TIME 1.0: prod*1 is exact and the FFMA2 rounds once, i.e. the
// same bits as add.rn, and ptxas cannot fold what it cannot prove is 1.
__device__ __forceinline__ float2 mad2(float2 acc, float2 x, float2 w, float2 one) {
    return __ffma2_rn(__fmul2_rn(x, w), one, acc);
}

// acc + prod with one rounding (see mad2)
__device__ __forceinline__ float2 add2p(float2 acc, float2 prod, float2 one) {
    return __ffma2_rn(prod, one, acc);  // acc + prod, one rounding (see mad2)
}

// Product of the window pair (win[idx], win[idx+1]) with one tap. A pair that
// starts at an odd index straddles two register pairs, and forming it costs a
// MOV pair; two scalar multiplies writing an aligned product pair use the same
// FMA-pipe slots as one FMUL2 and one instruction less (SC_ODD_SCALAR=0: always
// FMUL2). Bits are identical either way.
#ifndef SC_ODD_SCALAR
#define SC_ODD_SCALAR 1
#endif
// the packed form always (the single pass's dense folds: scalar products there
// raised its registers from 88-94 to 118-157)
__device__ __forceinline__ float2 prod2p(const float (&win)[12], int idx, float kv) {
    return __fmul2_rn(make_float2(win[idx], win[idx + 1]), make_float2(kv, kv));
}
__device__ __forceinline__ float2 prod2(const float (&win)[12], int idx, float kv) {
#if SC_ODD_SCALAR
    if (idx & 1) return make_float2(__fmul_rn(win[idx], kv), __fmul_rn(win[idx + 1], kv));
#endif
    return __fmul2_rn(make_float2(win[idx], win[idx + 1]), make_float2(kv, kv));
}

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
// Geometry
//
// Strip = TW = 4*GROUPS*NT output columns; consumer thread t owns GROUPS
// 4-column groups at strip offsets 4t + g*TW/GROUPS, so each warp-wide STG.128
// writes 512 contiguous bytes. Rows travel in stages of SROWS rows per mbarrier
// pair. GROUPS per mode (measured on B200): the two-pass modes run one group per
// thread (fewer registers -> 4 CTAs/SM; fused 2592^2 -17%, cfg5 -1%), the
// FP32-bound single pass keeps two (more independent FMA chains per thread).

#ifndef SC_GROUPS
#define SC_GROUPS 1
#endif
#ifndef SC_GROUPS_SINGLE
#define SC_GROUPS_SINGLE 2
#endif
#ifndef SC_F2
#define SC_F2 1
#endif
#ifndef SC_SROWS
#define SC_SROWS 4
#endif
constexpr int SROWS = SC_SROWS;
// stages a consumer holds back after finishing one (see consume_item)
__host__ __device__ constexpr int stage_lags(int mode, int rad) {
    return mode == MODE_FUSED ? ((rad + SROWS - 1) / SROWS > 0 ? (rad + SROWS - 1) / SROWS : 1) : 0;
}
__host__ __device__ constexpr int groups_of(int mode, int rad = 0) {
    return single_like(mode) && rad <= MAX_RAD ? SC_GROUPS_SINGLE : SC_GROUPS;
}
// lane-strided consumer: column pairs per thread and group. The column / dense fold
// keeps 2r partial sums per column in registers: one pair (2 columns) per thread
// holds them without spilling for the dense fold from r = 6 (two pairs: 40..1470
// bytes of spills at r = 6..10) and for the two-pass modes from r = 11
#ifndef SC_TWO_PAIRS_MAX_RAD
#define SC_TWO_PAIRS_MAX_RAD 10
#endif
__host__ __device__ constexpr int pairs_of(int mode, int rad) {
    return (single_like(mode) ? rad > 5 : rad > SC_TWO_PAIRS_MAX_RAD) ? 1 : 2;
}
// lane-strided consumer, dense fold of 7 x 7 and wider matrices: rolled row loop, one
// body. The unrolled bodies (4 rows x FAST / edge variants) of a 9 x 9 fold are 83 KB
// of FP instructions and run out of the instruction cache: measured at 3 x 8192^2,
// general matrix, W = 7: 1.01 -> 0.71 ms, W = 9: 1.97 -> 1.18 ms (tools/_w79.py)
#ifndef SC_LEAN_MIN_RAD
#define SC_LEAN_MIN_RAD 3
#endif
__host__ __device__ constexpr bool lean_of(int mode, int rad) { return single_like(mode) && rad >= SC_LEAN_MIN_RAD; }
// output columns per consumer thread (aligned: the adjacent-column consumers)
__host__ __device__ constexpr int cols_per_thread(int mode, int rad, bool aligned = false) {
    return rad <= MAX_RAD || aligned ? 4 * groups_of(mode, rad) : 2 * pairs_of(mode, rad) * groups_of(mode, rad);
}

// Shared-memory row width (floats): the segment [x0-4, x0+TW+4), plus room for
// the 16-B realignment of unaligned rows (up to 3 floats before and after, and
// the 4-float pad the segment starts after).
template <bool ALIGNED, int HL = HALO>
__device__ __forceinline__ int row_width(int tw) {
    return ALIGNED ? tw + 2 * HL : tw + 2 * HL + 16;
}

struct Item {
    int plane, x0, ylo, yhi, in_lo, in_hi;
    int strip, band;  // strip index, band ordinal over both segments
};

template <int MODE, int RAD>
__device__ __forceinline__ Item decode_item(const Params& p, int item) {
    const int units = p.nplanes * p.nstrips;
    int seg_lo = p.out_lo, seg_hi = p.out_hi, bh = p.band_h, band0 = 0;
    if (item >= p.nitems0) {
        item -= p.nitems0;
        seg_lo = p.out_lo2;
        seg_hi = p.out_hi2;
        bh = p.band_h2;
        band0 = p.nitems0 / units;
    }
    const int band = item / units;
    const int rem = item - band * units;
    Item it;
    it.plane = rem / p.nstrips;
    const int strip = rem - it.plane * p.nstrips;
    it.strip = strip;
    it.band = band0 + band;
    it.x0 = strip * p.tw;
    it.ylo = seg_lo + band * bh;
    it.yhi = min(it.ylo + bh, seg_hi);
    if (MODE == MODE_HPASS) {
        it.in_lo = it.ylo;
        it.in_hi = it.yhi;
    } else {
        it.in_lo = max(max(it.ylo - RAD, 0), p.avail_lo);
        it.in_hi = min(min(it.yhi + RAD, p.R), p.avail_hi);
    }
    return it;
}

// Rows needing per-row special cases: ring rows (FUSED copies them), rows where
// the row pass is dead (FUSED's zero H0 rows, HPASS's zero fill).
template <int MODE, int RAD>
__device__ __forceinline__ bool item_rows_edge(const Params& p, const Item& it) {
    if (MODE == MODE_HPASS) return it.ylo < p.hrow_lo || it.yhi > p.hrow_hi;
    if (fused_like(MODE))
        return it.in_lo < p.hrow_lo || it.in_hi > p.hrow_hi || it.ylo < RAD || it.yhi > p.R - RAD;
    return false;
}

// Global input row y of `plane`: from this band's buffer, or from a neighbouring
// band's (peer) buffer for halo rows outside it.
__device__ __forceinline__ const float* src_row(const Params& p, int plane, int y) {
    if (y < p.src_row0)
        return p.above + (long long)plane * p.above_ps + (long long)(y - p.above_row0) * p.above_rs;
    if (y >= p.src_row0 + p.src_rows)
        return p.below + (long long)plane * p.below_ps + (long long)(y - p.below_row0) * p.below_rs;
    return p.src + (long long)plane * p.src_plane_stride + (long long)(y - p.src_row0) * p.src_row_stride;
}

// ---------------------------------------------------------------------------
// Producer: one warp streams the strip's rows into the smem stage ring.

#ifndef SC_STATIC_FIRST
#define SC_STATIC_FIRST 1
#endif

template <int MODE, int RAD, bool ALIGNED, bool SIG = false>
__device__ __forceinline__ void producer(const Params& p, float* ring, uint64_t* full, uint64_t* empty,
                                         int* sitem, int* sshift) {
    // Items are claimed dynamically (atomic ticket), so CTAs that get more
    // bandwidth do more items and no SM idles in a tail. The claimed item id
    // rides in sitem[slot] of its first stage; id -1 tells consumers to stop.
    // ALIGNED: rows start 16-B aligned, so each row segment is one bulk copy
    // straight into place. Otherwise (any width / stride) the copy starts at the
    // 16-B boundary below the segment and the row's shift (0..3 floats) is
    // published in sshift[] for the consumers. Either way one lane issues TMA.
    const int lane = threadIdx.x & 31;
    if (lane != 0) return;
    constexpr int HL = halo_of(RAD);
    const int SW = row_width<ALIGNED, HL>(p.tw);
    const int NS = p.ns;
    uint64_t pol = 0;
    if (ALIGNED) pol = (p.flags & F_L2_EVICT_FIRST) ? policy_evict_first() : policy_evict_normal();
    int slot = 0;
    uint32_t phase = 0;
    int gs = 0;
#ifdef SC_TRACE
    int ntr = 0;
#endif
    // Row-band signalling: the neighbours' rows must be current (and their previous
    // step finished) before this CTA reads a neighbour row or writes anything. The
    // wait is deferred past the first stage's own-row copies: those are issued
    // first with the stage's transaction count (no arrival), the wait overlaps
    // their DRAM latency, and the producer's arrival -- after the wait -- is what
    // releases the stage to the consumers, so no store precedes the wait.
    bool waited = !SIG || p.epoch == 0;  // SIG: the peer-signalled instantiation only
    auto wait_neighbours = [&]() {
        wait_signal(p.sig_above, p.epoch, p.sig_err, p.sig_timeout_ns);
        wait_signal(p.sig_below, p.epoch, p.sig_err, p.sig_timeout_ns);
        asm volatile("fence.proxy.async.global;" ::: "memory");  // TMA reads after the acquire
        waited = true;
    };
    // The first item of every CTA is its own index (no atomic: 600-900 CTAs
    // claiming from one counter at launch serialise on it); later items come
    // from the ticket, offset by the grid size.
    bool first = SC_STATIC_FIRST;
    for (;;) {
        const int item = first ? (int)blockIdx.x : (int)gridDim.x * SC_STATIC_FIRST + atomicAdd(&p.work[0], 1);
        first = false;
#ifdef SC_TRACE
        if (ntr < 8) {
            SC_TR(p, 2 + ntr, clock64());
            SC_TR(p, 10 + ntr, item);
        }
        ++ntr;
#endif
        if (item >= p.nitems) {
            // no more work for this CTA: the next kernel on the stream may start
            // launching (it still waits for this grid to complete before its reads)
            asm volatile("griddepcontrol.launch_dependents;");
            if (gs >= NS) mbar_wait(&empty[slot], phase ^ 1u);
            sitem[slot] = -1;
            mbar_arrive_expect_tx(&full[slot], 0u);
            {
                // the last CTA out re-arms the ticket pair for the next launch
                __threadfence();
                if (atomicAdd(&p.work[1], 1) == (int)gridDim.x - 1) {
                    atomicExch(&p.work[0], 0);
                    atomicExch(&p.work[1], 0);
                }
            }
            return;
        }
        const Item it = decode_item<MODE, RAD>(p, item);
        const int cx0 = max(it.x0 - HL, 0);
        const int cx1 = min(it.x0 + p.tw + HL, p.C);
        const int n = cx1 - cx0;
        const int soff = cx0 - (it.x0 - HL);
        for (int r0 = it.in_lo; r0 < it.in_hi; r0 += SROWS, ++gs) {
            if (gs >= NS) mbar_wait(&empty[slot], phase ^ 1u);
            const int nrows = min(SROWS, it.in_hi - r0);
            float* sbase = ring + slot * SROWS * SW + soff;
            sitem[slot] = item;
            if (snap_mode(MODE)) {
                if (!waited) wait_neighbours();
                // own rows: the item's own columns from the image (nobody else writes
                // them), the 4-column halos from the column snapshot; halo rows (other
                // bands' rows) wholly from the row snapshot
                static_assert(!snap_mode(MODE) || ALIGNED, "in-place modes run aligned rows only");
                const int xr = min(it.x0 + p.tw, p.C);
                const bool lh = it.strip > 0, rh = it.strip + 1 < p.nstrips;
                uint32_t total = 0;
                for (int k = 0; k < nrows; ++k) {
                    const int y = r0 + k;
                    total += (y >= it.ylo && y < it.yhi) ? 4u * (uint32_t)(xr - it.x0) + (lh ? 16u : 0u) + (rh ? 16u : 0u)
                                                         : (uint32_t)n * 4u;  // halo rows: one full-width copy
                }
                mbar_arrive_expect_tx(&full[slot], total);
                for (int k = 0; k < nrows; ++k) {
                    const int y = r0 + k;
                    float* srow = sbase + k * SW;  // column cx0
                    if (y >= it.ylo && y < it.yhi) {
                        float* mid = srow + (it.x0 - cx0);
                        bulk_g2s(mid, src_row(p, it.plane, y) + it.x0, 4u * (uint32_t)(xr - it.x0), &full[slot], pol);
                        const long long cb = ((long long)it.plane * (p.nstrips - 1) - 1) * p.R + y;
                        if (lh) bulk_g2s(mid - 4, p.side_cols + (cb + (long long)it.strip * p.R) * 8, 16u, &full[slot], pol);
                        if (rh)
                            bulk_g2s(mid + (xr - it.x0), p.side_cols + (cb + (long long)(it.strip + 1) * p.R) * 8 + 4,
                                     16u, &full[slot], pol);
                    } else if (y < p.snap_lo || y >= p.snap_hi) {
                        // a row no item writes (the single pass's ring rows): the image itself
                        bulk_g2s(srow, src_row(p, it.plane, y) + cx0, (uint32_t)n * 4u, &full[slot], pol);
                    } else {
                        const int b = y < it.ylo ? it.band : it.band + 1;  // boundary at this band's top / bottom
                        const int t = y < it.ylo ? y - (it.ylo - RAD) : y - (it.yhi - RAD);
                        const float* side =
                            p.side_rows + (((long long)it.plane * p.side_nb + b) * (2 * RAD) + t) * (long long)p.C;
                        bulk_g2s(srow, side + cx0, (uint32_t)n * 4u, &full[slot], pol);
                    }
                }
            } else if (ALIGNED) {
                const uint32_t bytes = (uint32_t)n * 4u;
                if (!waited && r0 >= p.src_row0 && r0 + nrows <= p.src_row0 + p.src_rows) {
                    // first stage, own rows only: copies first, the wait under them
                    mbar_expect_tx(&full[slot], bytes * (uint32_t)nrows);
                    for (int k = 0; k < nrows; ++k)
                        bulk_g2s(sbase + k * SW, src_row(p, it.plane, r0 + k) + cx0, bytes, &full[slot], pol);
                    wait_neighbours();
                    mbar_arrive(&full[slot]);
                } else {
                    if (!waited) wait_neighbours();
                    mbar_arrive_expect_tx(&full[slot], bytes * (uint32_t)nrows);
                    for (int k = 0; k < nrows; ++k)
                        bulk_g2s(sbase + k * SW, src_row(p, it.plane, r0 + k) + cx0, bytes, &full[slot], pol);
                }
            } else {
                if (!waited) wait_neighbours();
                // the segment [g, g+n) lands at the 16-B aligned smem index 4 + soff, preceded
                // by its shift s = (g mod 16 B) / 4 floats: column c sits at c - x0 + HL + 4 + s
                uint32_t total = 0;
                for (int k = 0; k < nrows; ++k) {
                    const uintptr_t a = reinterpret_cast<uintptr_t>(src_row(p, it.plane, r0 + k) + cx0);
                    const uintptr_t e = a + 4u * (uintptr_t)n;
                    total += (uint32_t)(((e + 15) & ~(uintptr_t)15) - (a & ~(uintptr_t)15));
                }
                mbar_arrive_expect_tx(&full[slot], total);
                for (int k = 0; k < nrows; ++k) {
                    const uintptr_t a = reinterpret_cast<uintptr_t>(src_row(p, it.plane, r0 + k) + cx0);
                    const uintptr_t a_dn = a & ~(uintptr_t)15;
                    const uintptr_t e_up = (a + 4u * (uintptr_t)n + 15) & ~(uintptr_t)15;
                    sshift[slot * SROWS + k] = (int)((a - a_dn) >> 2);
                    bulk_g2s(sbase + k * SW + 4, reinterpret_cast<const void*>(a_dn), (uint32_t)(e_up - a_dn),
                             &full[slot], pol);
                }
            }
            if (++slot == NS) { slot = 0; phase ^= 1u; }
        }
    }
}

// Tap index used for the multiply by w[j]: with mirror-symmetric taps (SYMW:
// w[j] == w[2r-j] bitwise, checked on the host) taps j and 2r-j are the same
// value, so writing them with one index makes the products of the same operand
// one expression (the column fold multiplies each row value by r+1 distinct taps
// instead of 2r+1). Same IEEE products, same adds, same order: bit-identical.
template <int RAD, bool SYMW>
__host__ __device__ constexpr int tap_ix(int j) {
    return SYMW && j > RAD ? 2 * RAD - j : j;
}

// ---------------------------------------------------------------------------
// Per-row arithmetic for one 4-column group. win holds columns x4-4 .. x4+7.

template <int RAD, bool SYMW = false>
__device__ __forceinline__ F4 row_pass(const float (&win)[12], const float* w, float one) {
    F4 h;
#if SC_F2
    const float2 one2 = make_float2(one, one);
    // packed f32x2: two adjacent output columns per FMUL2/FADD2, each lane an
    // IEEE fp32 mul/add (same bits as __fmul_rn/__fadd_rn, never fused)
#pragma unroll
    for (int c = 0; c < 4; c += 2) {
        const int o = HALO - RAD + c;
        float2 acc = __fmul2_rn(make_float2(win[o], win[o + 1]), make_float2(w[0], w[0]));
#pragma unroll
        for (int m = 1; m <= 2 * RAD; ++m) acc = add2p(acc, prod2(win, o + m, w[tap_ix<RAD, SYMW>(m)]), one2);
        h.v[c] = acc.x;
        h.v[c + 1] = acc.y;
    }
#else
    (void)one;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        float acc = fm(win[HALO - RAD + c], w[0]);
#pragma unroll
        for (int m = 1; m <= 2 * RAD; ++m) acc = fa(acc, fm(win[HALO - RAD + c + m], w[m]));
        h.v[c] = acc;
    }
#endif
    return h;
}

// Column fold: push row value v into the shift register, return the finished
// output (row y-RAD). acc[j] holds the partial sum of output y-RAD+... started
// j+1 rows ago; every update is acc + v*w[j], exactly the reference's order.
template <int RAD, int NACC, bool SYMW = false>
__device__ __forceinline__ F4 col_fold(F4 (&acc)[NACC], const F4& v, const float* w, float one) {
    F4 out;
    (void)one;
    if (RAD == 0) {
#pragma unroll
        for (int c = 0; c < 4; ++c) out.v[c] = fm(v.v[c], w[0]);
        return out;
    }
#if SC_F2
#pragma unroll
    for (int c = 0; c < 4; c += 2) {
        const float2 one2 = make_float2(one, one);
        const float2 vv = make_float2(v.v[c], v.v[c + 1]);
        constexpr int jl = tap_ix<RAD, SYMW>(2 * RAD);
        float2 t = mad2(make_float2(acc[NACC - 1].v[c], acc[NACC - 1].v[c + 1]), vv, make_float2(w[jl], w[jl]), one2);
        out.v[c] = t.x;
        out.v[c + 1] = t.y;
#pragma unroll
        for (int j = NACC - 1; j >= 1; --j) {
            const int jj = tap_ix<RAD, SYMW>(j);
            t = mad2(make_float2(acc[j - 1].v[c], acc[j - 1].v[c + 1]), vv, make_float2(w[jj], w[jj]), one2);
            acc[j].v[c] = t.x;
            acc[j].v[c + 1] = t.y;
        }
        t = __fmul2_rn(vv, make_float2(w[0], w[0]));
        acc[0].v[c] = t.x;
        acc[0].v[c + 1] = t.y;
    }
#else
#pragma unroll
    for (int c = 0; c < 4; ++c) out.v[c] = fa(acc[NACC - 1].v[c], fm(v.v[c], w[2 * RAD]));
#pragma unroll
    for (int j = NACC - 1; j >= 1; --j)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[j].v[c] = fa(acc[j - 1].v[c], fm(v.v[c], w[j]));
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[0].v[c] = fm(v.v[c], w[0]);
#endif
    return out;
}

// Dense fold (single pass): input row yi carries kernel row i of output yi+RAD-i.
template <int RAD, int NACC>
__device__ __forceinline__ F4 dense_fold(F4 (&acc)[NACC], const float (&win)[12], const float* k, float one) {
    constexpr int W = 2 * RAD + 1;
    F4 out;
    (void)one;
    if (RAD == 0) {
#pragma unroll
        for (int c = 0; c < 4; ++c) out.v[c] = fm(win[HALO + c], k[0]);
        return out;
    }
#if SC_F2
    const float2 one2 = make_float2(one, one);
#pragma unroll
    for (int c = 0; c < 4; c += 2) {
        const int o = HALO - RAD + c;
        float2 t = make_float2(acc[NACC - 1].v[c], acc[NACC - 1].v[c + 1]);
#pragma unroll
        for (int j = 0; j < W; ++j) t = add2p(t, prod2p(win, o + j, k[(W - 1) * W + j]), one2);
        out.v[c] = t.x;
        out.v[c + 1] = t.y;
#pragma unroll
        for (int i = NACC - 1; i >= 1; --i) {
            t = make_float2(acc[i - 1].v[c], acc[i - 1].v[c + 1]);
#pragma unroll
            for (int j = 0; j < W; ++j) t = add2p(t, prod2p(win, o + j, k[i * W + j]), one2);
            acc[i].v[c] = t.x;
            acc[i].v[c + 1] = t.y;
        }
        t = prod2p(win, o, k[0]);
#pragma unroll
        for (int j = 1; j < W; ++j) t = add2p(t, prod2p(win, o + j, k[j]), one2);
        acc[0].v[c] = t.x;
        acc[0].v[c + 1] = t.y;
    }
#else
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        float t = acc[NACC - 1].v[c];
#pragma unroll
        for (int j = 0; j < W; ++j) t = fa(t, fm(win[HALO - RAD + c + j], k[(W - 1) * W + j]));
        out.v[c] = t;
    }
#pragma unroll
    for (int i = NACC - 1; i >= 1; --i) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            float t = acc[i - 1].v[c];
#pragma unroll
            for (int j = 0; j < W; ++j) t = fa(t, fm(win[HALO - RAD + c + j], k[i * W + j]));
            acc[i].v[c] = t;
        }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        float t = fm(win[HALO - RAD + c], k[0]);
#pragma unroll
        for (int j = 1; j < W; ++j) t = fa(t, fm(win[HALO - RAD + c + j], k[j]));
        acc[0].v[c] = t;
    }
#endif
    return out;
}

// Single pass with a mirror-symmetric dense matrix (K[i][j] == K[2r-i][j]
// bitwise, e.g. outer(w, w) of symmetric taps: gaussian5, sigma1 and the sharpen
// taps of the BASELINE configs): the products of kernel rows i and 2r-i are
// identical IEEE results of the same operands, so each is computed once and
// used twice. Fold order and every rounding are unchanged (bit-identical);
// (2r+1)*r fewer multiplies per input row (25 -> 15 at r = 2) in an FP32-bound
// kernel.

// COLSYM: the matrix is also mirror-symmetric in its columns (K[i][j] == K[i][2r-j]:
// outer(w, w) of symmetric taps). The products of column pair c with tap j and
// of pair c+2 with tap j-2 then multiply the same window samples by equal taps
// when j and j-2 mirror each other (j = 3, 1 at r = 2): writing both with the
// same tap index makes them one expression (27 instead of 30 FMUL2 per 4
// columns and row at r = 2).
template <int RAD, int NACC, bool COLSYM = false>
__device__ __forceinline__ F4 dense_fold_sym(F4 (&acc)[NACC], const float (&win)[12], const float* k, float one) {
    static_assert(RAD >= 1, "symmetric fold needs RAD >= 1");
    constexpr int W = 2 * RAD + 1;
    F4 out;
    const float2 one2 = make_float2(one, one);
#pragma unroll
    for (int c = 0; c < 4; c += 2) {
        const int o = HALO - RAD + c;
        float2 pr[RAD + 1][W];  // products of kernel rows 0..RAD (rows 2r..RAD+1 mirror them)
#pragma unroll
        for (int i = 0; i <= RAD; ++i)
#pragma unroll
            for (int j = 0; j < W; ++j)
            {
                const int kj = COLSYM ? (j < W - 1 - j ? j : W - 1 - j) : j;
                pr[i][j] = prod2p(win, o + j, k[i * W + kj]);
            }
        float2 t = make_float2(acc[NACC - 1].v[c], acc[NACC - 1].v[c + 1]);
#pragma unroll
        for (int j = 0; j < W; ++j) t = add2p(t, pr[0][j], one2);  // kernel row W-1 == row 0
        out.v[c] = t.x;
        out.v[c + 1] = t.y;
#pragma unroll
        for (int i = NACC - 1; i >= 1; --i) {
            t = make_float2(acc[i - 1].v[c], acc[i - 1].v[c + 1]);
#pragma unroll
            for (int j = 0; j < W; ++j) t = add2p(t, pr[i <= RAD ? i : W - 1 - i][j], one2);
            acc[i].v[c] = t.x;
            acc[i].v[c + 1] = t.y;
        }
        t = pr[0][0];
#pragma unroll
        for (int j = 1; j < W; ++j) t = add2p(t, pr[0][j], one2);
        acc[0].v[c] = t.x;
        acc[0].v[c + 1] = t.y;
    }
    return out;
}

// Store 4 columns of an output row with the column-ring policy (edge threads).
//   ring_mode 0: keep -- only columns in [rad, C-rad) are written
//   ring_mode 1: copy -- ring columns take `ringv` (the input samples)
//   ring_mode 2: zero -- ring columns take 0
// (aligned rows: x4 + 4 <= C whenever x4 < C)
__device__ __forceinline__ void store_edge(float* drow, int x4, int C, int rad, const F4& val, const F4& ringv,
                                        int ring_mode) {
    if (x4 >= C) return;
    F4 o;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int col = x4 + c;
        const bool valid = col >= rad && col < C - rad;
        o.v[c] = valid ? val.v[c] : (ring_mode == 1 ? ringv.v[c] : 0.0f);
    }
    if (ring_mode != 0) {
        st4(drow + x4, o);
        return;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int col = x4 + c;
        if (col >= C) break;
        const bool valid = col >= rad && col < C - rad;
        if (valid || ring_mode != 0) drow[col] = o.v[c];
    }
}

__device__ __forceinline__ void load_win(float (&win)[12], const float* s) {
    const F4 a = ld4(s), b = ld4(s + 4), c = ld4(s + 8);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        win[i] = a.v[i];
        win[4 + i] = b.v[i];
        win[8 + i] = c.v[i];
    }
}

// ---------------------------------------------------------------------------
// Consumer of 16-B aligned rows: one item (plane, strip, band). ROW_EDGE items
// contain ring rows or rows with a dead row pass; all others run the lean loop.
// (Rows of any other alignment: consume_item_lanes below.)

// COL_EDGE: the item's strip touches the image's column ring or its right edge
// (first and last strips); interior strips (COL_EDGE false) store
// every group with one STG.128 and need no per-row column tests (measured: -2% at
// cfg5 under the bench's sustained power cap, where issue slots are scarce; not
// used by the single pass, whose register allocation it upset: cfg2 +13%).
template <int MODE, int RAD, bool ROW_EDGE, int SYM, bool COL_EDGE = true, bool SIG = false>
__device__ __forceinline__ void consume_item(const Params& p, const Item& it, const float* ring, uint64_t* full,
                                             uint64_t* empty, int& slot, uint32_t& phase, int& gs) {
    constexpr int NACC = (2 * RAD > 0) ? 2 * RAD : 1;
    const int SW = row_width<true>(p.tw);
    const int NS = p.ns;
    const int ct = threadIdx.x - 32;
    const int lane = threadIdx.x & 31;
    constexpr int GROUPS = groups_of(MODE);
    // two-pass modes: SYM != 0 = mirror-symmetric taps, products shared by value
    // (tap_ix); under a sustained power cap the fewer FP instructions measured
    // 1.2% faster at cfg5 (1.0136 vs 1.0254 ms), no change at full clocks
    constexpr bool SYMW = !single_like(MODE) && SYM != 0;
    const int tw2 = p.tw / GROUPS;  // column offset between a thread's groups
    const int R = p.R, C = p.C;
    const bool ring_copy = (MODE == MODE_FUSED) && !(p.flags & F_NO_RING);  // SPLITF: image ring untouched
    const bool zero_fill = (MODE == MODE_HPASS) && (p.flags & F_ZERO_FILL);

    int x4[GROUPS];
    bool fast[GROUPS];
#pragma unroll
    for (int g = 0; g < GROUPS; ++g) {
        x4[g] = it.x0 + 4 * ct + g * tw2;
        fast[g] = !COL_EDGE || (x4[g] >= RAD && x4[g] + 4 <= C - RAD);
    }
    float* dplane = p.dst + (long long)it.plane * p.dst_plane_stride;

    // rows whose output is emitted: HPASS emits row yi, the vertical modes row yi-RAD
    int emit_lo, emit_hi;
    if (MODE == MODE_HPASS) {
        emit_lo = it.ylo;
        emit_hi = it.yhi;
    } else {
        emit_lo = max(max(it.ylo, RAD), it.in_lo + RAD);
        emit_hi = min(it.yhi, R - RAD);
    }
    float* dcur = dplane + (long long)(emit_lo - p.dst_row0) * p.dst_row_stride;

    F4 acc[GROUPS][NACC];
#pragma unroll
    for (int g = 0; g < GROUPS; ++g)
#pragma unroll
        for (int j = 0; j < NACC; ++j)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[g][j].v[c] = 0.0f;

    for (int r0 = it.in_lo; r0 < it.in_hi; r0 += SROWS, ++gs) {
        if (r0 != it.in_lo) mbar_wait(&full[slot], phase);  // the item's first stage was waited by the caller
        if (SIG && p.epoch && threadIdx.x == 32) {
            // done accounting of the row-band signalling: this stage's copies have
            // landed, so an item that read the band above (its first stage) or the
            // band below (its last stage) has finished reading that neighbour
            if (r0 == it.in_lo && it.in_lo < p.src_row0) red_add_relaxed_sys(p.sig_self + 2, 1ULL);
            if (r0 + SROWS >= it.in_hi && it.in_hi > p.src_row0 + p.src_rows) red_add_relaxed_sys(p.sig_self + 3, 1ULL);
        }
#ifdef SC_TRACE
        if (threadIdx.x == 32 && gs < 8) SC_TR(p, 48 + gs, clock64());
#endif
        // stages are contiguous in smem: the ring is one circular buffer of NS*SROWS rows
        const float* sstage = ring + slot * SROWS * SW + 4 * ct;
        // A stage whose rows all exist and all emit (every stage of an interior item
        // but its first and last) runs without per-row range tests.
        auto stage_rows = [&](auto fast_stage) {
            constexpr bool FAST = decltype(fast_stage)::value;
    #pragma unroll
            for (int k = 0; k < SROWS; ++k) {
                const int yi = r0 + k;
                if (FAST || yi < it.in_hi) {
                    const bool live = !ROW_EDGE || (yi >= p.hrow_lo && yi < p.hrow_hi);
                    const int yo = (MODE == MODE_HPASS) ? yi : yi - RAD;
                    const bool emit = FAST || (yo >= emit_lo && yo < emit_hi);
    #pragma unroll
                    for (int g = 0; g < GROUPS; ++g) {
                        // a warp whose group lies wholly right of the image (the padding of a
                        // partial last strip) has nothing to store: skip its arithmetic
                        // (warp-uniform: lane 0's columns)
                        if (COL_EDGE && x4[g] - 4 * lane >= C) continue;
                        float win[12];
                        load_win(win, sstage + k * SW + g * tw2);
                        F4 own;
    #pragma unroll
                        for (int i = 0; i < 4; ++i) own.v[i] = win[4 + i];
                        F4 outv;
                        if (MODE == MODE_HPASS) {
                            if (live) {
                                outv = row_pass<RAD, SYMW>(win, p.w, p.one);
                            } else {
    #pragma unroll
                                for (int i = 0; i < 4; ++i) outv.v[i] = 0.0f;
                            }
                        } else if (single_like(MODE)) {
                            if constexpr (SYM >= 1 && SC_F2 && RAD >= 1)
                                outv = dense_fold_sym<RAD, NACC, (SYM >= 2)>(acc[g], win, p.k, p.one);
                            else
                                outv = dense_fold<RAD, NACC>(acc[g], win, p.k, p.one);
                        } else {
                            F4 v;
                            if (fused_like(MODE)) {
                                if (live) {
    #ifdef SC_NOCOMPUTE
                                    v = own;
    #else
                                    v = row_pass<RAD, SYMW>(win, p.w, p.one);
    #endif
                                } else {
    #pragma unroll
                                    for (int i = 0; i < 4; ++i) v.v[i] = 0.0f;  // faithful: scratch row stays 0
                                }
                            } else {
                                v = own;  // VPASS: src already holds the row-pass result
                            }
                            if constexpr (MODE == MODE_SPLITF) {
                                // the reference's scratch row: H0 on the valid columns, 0 on the
                                // column ring and on dead rows (the workspace is zeroed first,
                                // S/conv.py:414); own rows only. No scratch (null): the
                                // in-place fused two-pass -- image only, 2 traversals
                                if (p.scr && yi >= it.ylo && yi < it.yhi) {
                                    float* hrow = p.scr + (long long)it.plane * p.scr_ps + (long long)yi * p.scr_rs;
                                    if (fast[g]) {
                                        st4(hrow + x4[g], v);
                                    } else {
                                        F4 zero;
    #pragma unroll
                                        for (int i = 0; i < 4; ++i) zero.v[i] = 0.0f;
                                        store_edge(hrow, x4[g], C, RAD, v, zero, 2);
                                    }
                                }
                            }
    #ifdef SC_NOCOMPUTE
                            outv = v;  // dev-only variant: pipeline cost without the arithmetic
    #else
                            outv = col_fold<RAD, NACC, SYMW>(acc[g], v, p.w, p.one);
    #endif
                        }
                        if (MODE == MODE_HPASS) {
                            // dead rows are written only under zero fill
                            if (emit && (live || zero_fill)) {
                                if (fast[g] && live)
                                    st4(dcur + 4 * ct + g * tw2 + (it.x0), outv);
                                else
                                    store_edge(dcur, x4[g], C, live ? RAD : 0, outv, own, zero_fill ? 2 : 0);
                            }
                        } else if (emit) {
                            if constexpr (MODE == MODE_SINGLECB) {
                                // copy-back: the same valid samples into the image, in place
                                float* irow = p.scr + (long long)it.plane * p.scr_ps + (long long)yo * p.scr_rs;
                                if (fast[g]) {
                                    st4(irow + x4[g], outv);
                                } else {
                                    F4 zero;
    #pragma unroll
                                    for (int i = 0; i < 4; ++i) zero.v[i] = 0.0f;
                                    store_edge(irow, x4[g], C, RAD, outv, zero, 0);
                                }
                            }
                            if (fast[g]) {
                                st4(dcur + x4[g], outv);
                            } else {
                                F4 ringv;
                                if (ring_copy) {
                                    int rr = slot * SROWS + k - RAD;  // ring row of input row yo
                                    if (rr < 0) rr += NS * SROWS;
                                    const float* rrow = ring + rr * SW + 4 * ct + g * tw2;
                                    ringv = ld4(rrow + 4);
                                } else {
    #pragma unroll
                                    for (int i = 0; i < 4; ++i) ringv.v[i] = 0.0f;
                                }
                                store_edge(dcur, x4[g], C, RAD, outv, ringv, ring_copy ? 1 : 0);
                            }
                        }
                        if (ROW_EDGE && ring_copy && yi >= it.ylo && yi < it.yhi && (yi < RAD || yi >= R - RAD)) {
                            float* drow = dplane + (long long)(yi - p.dst_row0) * p.dst_row_stride;
                            store_edge(drow, x4[g], C, 0, own, own, 1);
                        }
                    }
                    if (emit) dcur += p.dst_row_stride;
                }
            }
        };
        const int yo0 = (MODE == MODE_HPASS) ? r0 : r0 - RAD;
        if (!ROW_EDGE && !COL_EDGE && r0 + SROWS <= it.in_hi && yo0 >= emit_lo && yo0 + SROWS <= emit_hi)
            stage_rows(std::true_type{});
        else
            stage_rows(std::false_type{});
#ifdef SC_TRACE
        if (threadIdx.x == 32 && gs < 8) SC_TR(p, 56 + gs, clock64());
#endif
        // this stage is done; release the one LAGS stages back: the fused two-pass
        // still reads rows up to RAD back for the ring columns, every other mode
        // hands its stage straight back (one more stage of prefetch from the same
        // ring; ncu on the single pass: 9% of the consumers' samples were waits
        // for a full stage with a 3-stage ring)
        constexpr int LAGS = stage_lags(MODE, RAD);
        if (gs >= LAGS) {
            int rel = slot - LAGS;
            if (rel < 0) rel += NS;
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[rel]);
        }
        if (++slot == NS) { slot = 0; phase ^= 1u; }
    }
}

// ---------------------------------------------------------------------------
// Consumer of 16-B aligned rows at widths 11..21 (r = 5..10), two-pass modes:
// adjacent columns as consume_item, with a window of 4 + 2*halo_of(r) samples per
// row (5-7 x LDS.128 for 4 outputs, where the lane-strided consumer reads 4*(2r+1)
// words one by one: ncu had its shared-memory pipe 67% busy at W = 11, next to an
// FMA pipe at 61%), products of odd-start window pairs as two scalar multiplies
// (no pair-forming moves), the column fold through the same shift register.

template <int RAD, bool SYMW, int HL>
__device__ __forceinline__ F4 row_pass_win(const float (&win)[4 + 2 * HL], const float* w, float one) {
    F4 h;
    const float2 one2 = make_float2(one, one);
    auto pairprod = [&](int idx, float kv) {
        if (idx & 1) return make_float2(__fmul_rn(win[idx], kv), __fmul_rn(win[idx + 1], kv));
        return __fmul2_rn(make_float2(win[idx], win[idx + 1]), make_float2(kv, kv));
    };
#pragma unroll
    for (int c = 0; c < 4; c += 2) {
        const int o = HL - RAD + c;
        float2 acc = pairprod(o, w[0]);
#pragma unroll
        for (int m = 1; m <= 2 * RAD; ++m) acc = add2p(acc, pairprod(o + m, w[tap_ix<RAD, SYMW>(m)]), one2);
        h.v[c] = acc.x;
        h.v[c + 1] = acc.y;
    }
    return h;
}

template <int MODE, int RAD, bool ROW_EDGE, int SYM>
__device__ __forceinline__ void consume_item_adj(const Params& p, const float* w, const Item& it, const float* ring,
                                                 uint64_t* full, uint64_t* empty, int& slot, uint32_t& phase, int& gs) {
    static_assert(MODE == MODE_FUSED || MODE == MODE_HPASS || MODE == MODE_VPASS, "two-pass modes only");
    constexpr int NACC = 2 * RAD;
    constexpr bool SYMW = SYM != 0;
    constexpr int LAGS = stage_lags(MODE, RAD);
    constexpr int HL = halo_of(RAD);
    constexpr int WN = 4 + 2 * HL;
    const int SW = row_width<true, HL>(p.tw);
    const int NS = p.ns;
    const int ct = threadIdx.x - 32;
    const int lane = threadIdx.x & 31;
    const int R = p.R, C = p.C;
    const bool ring_copy = (MODE == MODE_FUSED) && !(p.flags & F_NO_RING);
    const bool zero_fill = (MODE == MODE_HPASS) && (p.flags & F_ZERO_FILL);
    const int x4 = it.x0 + 4 * ct;
    const bool fast = x4 >= RAD && x4 + 4 <= C - RAD;  // all four columns valid
    const bool warp_outside = x4 - 4 * lane >= C;       // the whole warp lies right of the image
    float* dplane = p.dst + (long long)it.plane * p.dst_plane_stride;

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

    for (int r0 = it.in_lo; r0 < it.in_hi; r0 += SROWS, ++gs) {
        if (r0 != it.in_lo) mbar_wait(&full[slot], phase);  // the item's first stage was waited by the caller
        const float* sstage = ring + slot * SROWS * SW + 4 * ct;  // column x4 - HL of the stage's first row
        auto stage_rows = [&](auto fast_stage) {
            constexpr bool FAST = decltype(fast_stage)::value;
#pragma unroll
            for (int k = 0; k < SROWS; ++k) {
                const int yi = r0 + k;
                if (FAST || yi < it.in_hi) {
                    const bool live = !ROW_EDGE || (yi >= p.hrow_lo && yi < p.hrow_hi);
                    const int yo = (MODE == MODE_HPASS) ? yi : yi - RAD;
                    const bool emit = FAST || (yo >= emit_lo && yo < emit_hi);
                    if (!warp_outside) {
                        const float* srow = sstage + k * SW;
                        F4 own, outv;
                        if (MODE == MODE_VPASS) {
                            own = ld4(srow + HL);
                            outv = col_fold<RAD, NACC, SYMW>(acc, own, w, p.one);
                        } else {
                            float win[WN];
#pragma unroll
                            for (int q = 0; q < WN / 4; ++q) {
                                const F4 t = ld4(srow + 4 * q);
#pragma unroll
                                for (int i = 0; i < 4; ++i) win[4 * q + i] = t.v[i];
                            }
#pragma unroll
                            for (int i = 0; i < 4; ++i) own.v[i] = win[HL + i];
                            F4 v;
                            if (live) {
                                v = row_pass_win<RAD, SYMW, HL>(win, w, p.one);
                            } else {
#pragma unroll
                                for (int i = 0; i < 4; ++i) v.v[i] = 0.0f;  // dead row: H0 = 0 / zero fill
                            }
                            outv = MODE == MODE_HPASS ? v : col_fold<RAD, NACC, SYMW>(acc, v, w, p.one);
                        }
                        if (MODE == MODE_HPASS) {
                            if (emit && (live || zero_fill)) {
                                if (fast && live)
                                    st4(dcur + x4, outv);
                                else
                                    store_edge(dcur, x4, C, live ? RAD : 0, outv, own, zero_fill ? 2 : 0);
                            }
                        } else if (emit) {
                            if (fast) {
                                st4(dcur + x4, outv);
                            } else {
                                F4 ringv;
                                if (ring_copy) {
                                    int rr = slot * SROWS + k - RAD;  // ring row of input row yo
                                    if (rr < 0) rr += NS * SROWS;
                                    ringv = ld4(ring + rr * SW + 4 * ct + HL);
                                } else {
#pragma unroll
                                    for (int i = 0; i < 4; ++i) ringv.v[i] = 0.0f;
                                }
                                store_edge(dcur, x4, C, RAD, outv, ringv, ring_copy ? 1 : 0);
                            }
                        }
                        if (ROW_EDGE && ring_copy && yi >= it.ylo && yi < it.yhi && (yi < RAD || yi >= R - RAD)) {
                            float* drow = dplane + (long long)(yi - p.dst_row0) * p.dst_row_stride;
                            store_edge(drow, x4, C, 0, own, own, 1);
                        }
                    }
                    if (emit) dcur += p.dst_row_stride;
                }
            }
        };
        const int yo0 = (MODE == MODE_HPASS) ? r0 : r0 - RAD;
        if (!ROW_EDGE && r0 + SROWS <= it.in_hi && yo0 >= emit_lo && yo0 + SROWS <= emit_hi)
            stage_rows(std::true_type{});
        else
            stage_rows(std::false_type{});
        if (gs >= LAGS) {
            int rel_s = slot - LAGS;
            if (rel_s < 0) rel_s += NS;
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[rel_s]);
        }
        if (++slot == NS) { slot = 0; phase ^= 1u; }
    }
}

// ---------------------------------------------------------------------------
// Consumer for rows of ANY alignment (ALIGNED false: cols % 4 != 0, views whose
// rows do not start on 16-B boundaries, either side): lane-strided columns.
//
// Thread (warp q, lane l) owns columns 128q + l + 32i (i = 0..3) of each of its
// groups instead of 4 adjacent ones. Every shared-memory read is then an LDS.32
// whose 32 lanes hit 32 consecutive words -- conflict-free whatever the row's
// shift -- so the window needs no realignment (the adjacent-column layout pays 26
// selects per row for it), every packed operand pair (columns c, c+32) is formed
// by the loads themselves (no odd-pair moves), and every store is an STG.32 whose
// warp writes 128 contiguous bytes at any destination alignment (no staging rows,
// no shuffles, no per-warp edge columns). Same products, same sums, same order
// per column as everywhere else: bit-identical.
// Measured on B200 (3 x 16384^2 views offset by one float, tools/misalign_probe.py;
// odd sizes, tools/generic_perf.py): see DESIGN.md section 6.

template <int RAD, bool SYMW>
__device__ __forceinline__ float2 row_pass_pair(const float2 (&X)[2 * RAD + 1], const float* w, float2 one2) {
    float2 acc = __fmul2_rn(X[0], make_float2(w[0], w[0]));
#pragma unroll
    for (int m = 1; m <= 2 * RAD; ++m) {
        const int t = tap_ix<RAD, SYMW>(m);
        acc = add2p(acc, __fmul2_rn(X[m], make_float2(w[t], w[t])), one2);
    }
    return acc;
}

template <int RAD, int NACC, bool SYMW>
__device__ __forceinline__ float2 col_fold_pair(float2 (&acc)[NACC], float2 v, const float* w, float2 one2) {
    if (RAD == 0) return __fmul2_rn(v, make_float2(w[0], w[0]));
    constexpr int jl = tap_ix<RAD, SYMW>(2 * RAD);
    const float2 out = mad2(acc[NACC - 1], v, make_float2(w[jl], w[jl]), one2);
#pragma unroll
    for (int j = NACC - 1; j >= 1; --j) {
        const int jj = tap_ix<RAD, SYMW>(j);
        acc[j] = mad2(acc[j - 1], v, make_float2(w[jj], w[jj]), one2);
    }
    acc[0] = __fmul2_rn(v, make_float2(w[0], w[0]));
    return out;
}

// ROWSYM: K[i][j] == K[2r-i][j] bitwise (see dense_fold_sym): rows i and 2r-i share their products
template <int RAD, int NACC, bool ROWSYM>
__device__ __forceinline__ float2 dense_fold_pair(float2 (&acc)[NACC], const float2 (&X)[2 * RAD + 1], const float* k,
                                                  float2 one2) {
    constexpr int W = 2 * RAD + 1;
    if (RAD == 0) return __fmul2_rn(X[0], make_float2(k[0], k[0]));
    auto mul = [&](int i, int j) { return __fmul2_rn(X[j], make_float2(k[i * W + j], k[i * W + j])); };
    float2 out;
    if constexpr (ROWSYM) {
        float2 pr[RAD + 1][W];  // products of kernel rows 0..RAD (rows 2r..r+1 mirror them)
#pragma unroll
        for (int i = 0; i <= RAD; ++i)
#pragma unroll
            for (int j = 0; j < W; ++j) pr[i][j] = mul(i, j);
        float2 t = acc[NACC - 1];
#pragma unroll
        for (int j = 0; j < W; ++j) t = add2p(t, pr[0][j], one2);  // kernel row 2r == row 0
        out = t;
#pragma unroll
        for (int i = NACC - 1; i >= 1; --i) {
            t = acc[i - 1];
#pragma unroll
            for (int j = 0; j < W; ++j) t = add2p(t, pr[i <= RAD ? i : W - 1 - i][j], one2);
            acc[i] = t;
        }
        t = pr[0][0];
#pragma unroll
        for (int j = 1; j < W; ++j) t = add2p(t, pr[0][j], one2);
        acc[0] = t;
    } else {
        float2 t = acc[NACC - 1];
#pragma unroll
        for (int j = 0; j < W; ++j) t = add2p(t, mul(W - 1, j), one2);
        out = t;
#pragma unroll
        for (int i = NACC - 1; i >= 1; --i) {
            t = acc[i - 1];
#pragma unroll
            for (int j = 0; j < W; ++j) t = add2p(t, mul(i, j), one2);
            acc[i] = t;
        }
        t = mul(0, 0);
#pragma unroll
        for (int j = 1; j < W; ++j) t = add2p(t, mul(0, j), one2);
        acc[0] = t;
    }
    return out;
}

// w / k: the taps / dense matrix in the kernel's parameter block (Params::w, ::k;
// ParamsW::wide_w, ::wide_k for r > 4). LEAN (the single pass at r > 4): the rows
// of a stage run in a rolled loop and every item takes the ROW_EDGE path -- the
// unrolled bodies of a 21 x 21 dense fold would not fit the instruction cache --
// and mirror-symmetric matrices share no products (their (r+1)(2r+1) product
// pairs would not fit the register file).
template <int MODE, int RAD, bool ROW_EDGE, int SYM, bool SIG = false>
__device__ __forceinline__ void consume_item_lanes(const Params& p, const float* w, const float* kd, const Item& it,
                                                   const float* ring, uint64_t* full, uint64_t* empty,
                                                   const int* sshift, int& slot, uint32_t& phase, int& gs) {
    static_assert(!snap_mode(MODE), "in-place modes run aligned rows only");
    constexpr int W = 2 * RAD + 1;
    constexpr int NACC = (2 * RAD > 0) ? 2 * RAD : 1;
    constexpr int GROUPS = groups_of(MODE, RAD);
    constexpr int PAIRS = pairs_of(MODE, RAD);  // column pairs (c, c+32) per thread and group
    constexpr int CPT = 2 * PAIRS;
    constexpr unsigned ALLC = (1u << CPT) - 1u;
    constexpr bool LEAN = lean_of(MODE, RAD);
    constexpr int ROW_UNROLL = LEAN ? 1 : SROWS;
    constexpr bool SYMW = !single_like(MODE) && SYM != 0;
    constexpr bool ROWSYM = SYM >= 1 && RAD <= MAX_RAD;
    constexpr int LAGS = stage_lags(MODE, RAD);
    constexpr int HL = halo_of(RAD);
    const int SW = row_width<false, HL>(p.tw);
    const int NS = p.ns;
    const int ct = threadIdx.x - 32;
    const int lane = threadIdx.x & 31;
    const int tw2 = p.tw / GROUPS;  // column offset between a thread's groups
    const int R = p.R, C = p.C;
    const bool ring_copy = (MODE == MODE_FUSED) && !(p.flags & F_NO_RING);
    const bool zero_fill = (MODE == MODE_HPASS) && (p.flags & F_ZERO_FILL);
    const float2 one2 = make_float2(p.one, p.one);

    // column tests do not depend on the row: bit 4g + i of `inside` (column exists)
    // and `valid` (column outside the column ring)
    int rel[GROUPS];
    unsigned inside = 0, valid = 0;
#pragma unroll
    for (int g = 0; g < GROUPS; ++g) {
        rel[g] = g * tw2 + CPT * (ct & ~31) + lane;
#pragma unroll
        for (int i = 0; i < CPT; ++i) {
            const int col = it.x0 + rel[g] + 32 * i;
            if (col < C) inside |= 1u << (CPT * g + i);
            if (col >= RAD && col < C - RAD) valid |= 1u << (CPT * g + i);
        }
    }
    float* dplane = p.dst + (long long)it.plane * p.dst_plane_stride + it.x0;

    int emit_lo, emit_hi;
    if (MODE == MODE_HPASS) {
        emit_lo = it.ylo;
        emit_hi = it.yhi;
    } else {
        emit_lo = max(max(it.ylo, RAD), it.in_lo + RAD);
        emit_hi = min(it.yhi, R - RAD);
    }
    float* dcur = dplane + (long long)(emit_lo - p.dst_row0) * p.dst_row_stride;

    float2 acc[GROUPS][PAIRS][NACC];
#pragma unroll
    for (int g = 0; g < GROUPS; ++g)
#pragma unroll
        for (int q = 0; q < PAIRS; ++q)
#pragma unroll
            for (int j = 0; j < NACC; ++j) acc[g][q][j] = make_float2(0.0f, 0.0f);

    for (int r0 = it.in_lo; r0 < it.in_hi; r0 += SROWS, ++gs) {
        if (r0 != it.in_lo) mbar_wait(&full[slot], phase);  // the item's first stage was waited by the caller
        if (SIG && p.epoch && threadIdx.x == 32) {
            if (r0 == it.in_lo && it.in_lo < p.src_row0) red_add_relaxed_sys(p.sig_self + 2, 1ULL);
            if (r0 + SROWS >= it.in_hi && it.in_hi > p.src_row0 + p.src_rows) red_add_relaxed_sys(p.sig_self + 3, 1ULL);
        }
        // column x0 of ring row rr sits at ring[rr * SW + HL + 4 + sshift[rr]] (producer)
        int sh[SROWS];
        if (!LEAN) {
#pragma unroll
            for (int k = 0; k < SROWS; ++k) sh[k] = sshift[slot * SROWS + k];
        }
        const float* sstage = ring + slot * SROWS * SW + HL + 4;
        auto stage_rows = [&](auto fast_stage) {
            constexpr bool FAST = decltype(fast_stage)::value;
#pragma unroll ROW_UNROLL
            for (int k = 0; k < SROWS; ++k) {
                const int yi = r0 + k;
                if (FAST || yi < it.in_hi) {
                    const bool live = !ROW_EDGE || (yi >= p.hrow_lo && yi < p.hrow_hi);
                    const int yo = (MODE == MODE_HPASS) ? yi : yi - RAD;
                    const bool emit = FAST || (yo >= emit_lo && yo < emit_hi);
                    const float* srow = sstage + k * SW + (LEAN ? sshift[slot * SROWS + k] : sh[k]);
                    const bool ring_row = ROW_EDGE && ring_copy && yi >= it.ylo && yi < it.yhi && (yi < RAD || yi >= R - RAD);
#pragma unroll
                    for (int g = 0; g < GROUPS; ++g) {
                        // a warp whose columns all lie right of the image has nothing to store
                        if (it.x0 + rel[g] - lane >= C) continue;
                        const float* s = srow + rel[g];
                        float2 outv[PAIRS], own[PAIRS];
#pragma unroll
                        for (int q = 0; q < PAIRS; ++q) {
                            float2 X[W];
                            if (MODE == MODE_VPASS) {
                                own[q] = make_float2(s[64 * q], s[64 * q + 32]);
                            } else {
#pragma unroll
                                for (int j = 0; j < W; ++j) X[j] = make_float2(s[64 * q + j - RAD], s[64 * q + 32 + j - RAD]);
                                own[q] = X[RAD];
                            }
                            if (MODE == MODE_HPASS) {
                                outv[q] = live ? row_pass_pair<RAD, SYMW>(X, w, one2) : make_float2(0.0f, 0.0f);
                            } else if (single_like(MODE)) {
                                outv[q] = dense_fold_pair<RAD, NACC, ROWSYM>(acc[g][q], X, kd, one2);
                            } else {
                                float2 v = own[q];  // VPASS: src already holds the row-pass result
                                if (MODE == MODE_FUSED)  // dead rows: the faithful scratch row stays 0
                                    v = live ? row_pass_pair<RAD, SYMW>(X, w, one2) : make_float2(0.0f, 0.0f);
                                outv[q] = col_fold_pair<RAD, NACC, SYMW>(acc[g][q], v, w, one2);
                            }
                        }
                        const unsigned in4 = (inside >> (CPT * g)) & ALLC, va4 = (valid >> (CPT * g)) & ALLC;
                        float o4[CPT], w4[CPT];
#pragma unroll
                        for (int q = 0; q < PAIRS; ++q) {
                            o4[2 * q] = outv[q].x;
                            o4[2 * q + 1] = outv[q].y;
                            w4[2 * q] = own[q].x;
                            w4[2 * q + 1] = own[q].y;
                        }
                        if (MODE == MODE_HPASS) {
                            // dead rows are written (as zeros) only under zero fill; on live
                            // rows the column ring is zeroed under zero fill, else kept
                            if (emit && (live || zero_fill)) {
                                float* d = dcur + rel[g];
                                if (live && va4 == ALLC) {
#pragma unroll
                                    for (int i = 0; i < CPT; ++i) d[32 * i] = o4[i];
                                } else {
#pragma unroll
                                    for (int i = 0; i < CPT; ++i) {
                                        const bool val = live && ((va4 >> i) & 1u);
                                        if (((in4 >> i) & 1u) && (val || zero_fill)) d[32 * i] = val ? o4[i] : 0.0f;
                                    }
                                }
                            }
                        } else if (emit) {
                            float* d = dcur + rel[g];
                            if (va4 == ALLC) {
#pragma unroll
                                for (int i = 0; i < CPT; ++i) d[32 * i] = o4[i];
                            } else {
                                // ring columns of output row yo keep the input sample, staged RAD rows back
                                int rr = slot * SROWS + k - RAD;
                                if (rr < 0) rr += NS * SROWS;
                                const float* rrow = ring + rr * SW + HL + 4 + rel[g];
#pragma unroll
                                for (int i = 0; i < CPT; ++i) {
                                    if ((va4 >> i) & 1u)
                                        d[32 * i] = o4[i];
                                    else if (ring_copy && ((in4 >> i) & 1u))
                                        d[32 * i] = rrow[sshift[rr] + 32 * i];
                                }
                            }
                        }
                        if (ring_row) {  // a ring row of the image: the input row itself
                            float* d = dplane + (long long)(yi - p.dst_row0) * p.dst_row_stride + rel[g];
#pragma unroll
                            for (int i = 0; i < CPT; ++i)
                                if ((in4 >> i) & 1u) d[32 * i] = w4[i];
                        }
                    }
                    if (emit) dcur += p.dst_row_stride;
                }
            }
        };
        const int yo0 = (MODE == MODE_HPASS) ? r0 : r0 - RAD;
        if (!LEAN && !ROW_EDGE && r0 + SROWS <= it.in_hi && yo0 >= emit_lo && yo0 + SROWS <= emit_hi)
            stage_rows(std::true_type{});
        else
            stage_rows(std::false_type{});
        if (gs >= LAGS) {
            int rel_s = slot - LAGS;
            if (rel_s < 0) rel_s += NS;
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[rel_s]);
        }
        if (++slot == NS) { slot = 0; phase ^= 1u; }
    }
}

// ---------------------------------------------------------------------------
// The kernel

// SIG: the row-band readiness signalling (Params::sig_*) is compiled in; only the
// peer-band launches use it, so every other kernel carries none of its code.
#ifndef SC_MINB
#define SC_MINB 1
#endif
// w / kd: the taps and the dense matrix inside the kernel's parameter block
template <int MODE, int RAD, bool ALIGNED, int SYM, bool SIG>
__device__ __forceinline__ void rows_kernel_body(const Params& p, const float* w, const float* kd) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int NS = p.ns;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t* empty = full + NS;
    int* sitem = reinterpret_cast<int*>(empty + NS);
    int* sshift = sitem + NS;  // per ring row (NS * SROWS): float shift of an unaligned row
    float* ring = reinterpret_cast<float*>(smem_raw + ((2 * NS * 8 + NS * 4 + NS * SROWS * 4 + 127) / 128) * 128);
    (void)w;
    (void)kd;
    const int warp = threadIdx.x >> 5;
    const int ncw = (blockDim.x >> 5) - 1;

    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) {
            mbar_init(&full[i], 1u);
            mbar_init(&empty[i], (uint32_t)ncw);
        }
        mbar_fence_init();
    }
    __syncthreads();
    // launched with programmatic stream serialization: the setup above overlapped
    // the previous kernel's tail; no global memory is touched before it completed
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // this band's inputs are in place (the previous grid completed): one CTA says so
    if (SIG && p.epoch && threadIdx.x == 0 && blockIdx.x == 0) {
        // per-epoch counts of the items that read the band above / below (fixed
        // by the plan), ordered before ready by the release
        p.sig_self[4] = p.sig_n_above;
        p.sig_self[5] = p.sig_n_below;
        st_release_sys(p.sig_self, p.epoch);
    }

    if (warp == 0) {
#ifdef SC_TRACE
        if (threadIdx.x == 0) {
            SC_TR(p, 0, trace_gt());
            SC_TR(p, 1, clock64());
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            SC_TR(p, 43, smid);
        }
#endif
        producer<MODE, RAD, ALIGNED, SIG>(p, ring, full, empty, sitem, sshift);
        return;
    }

    int slot = 0;
    uint32_t phase = 0;
    int gs = 0;
#ifdef SC_TRACE
    int ntr = 0;
#endif
    for (;;) {
        mbar_wait(&full[slot], phase);
        const int item = sitem[slot];
        if (item < 0) break;
#ifdef SC_TRACE
        if (threadIdx.x == 32 && ntr < 8) SC_TR(p, 20 + ntr, clock64());
#endif
        const Item it = decode_item<MODE, RAD>(p, item);
        if constexpr (ALIGNED && RAD > MAX_RAD) {  // widths 11..21 on aligned rows
            if (item_rows_edge<MODE, RAD>(p, it))
                consume_item_adj<MODE, RAD, true, SYM>(p, w, it, ring, full, empty, slot, phase, gs);
            else
                consume_item_adj<MODE, RAD, false, SYM>(p, w, it, ring, full, empty, slot, phase, gs);
        } else if constexpr (!ALIGNED && lean_of(MODE, RAD)) {  // one (ROW_EDGE) body
            consume_item_lanes<MODE, RAD, true, SYM, SIG>(p, w, kd, it, ring, full, empty, sshift, slot, phase, gs);
        } else if constexpr (!ALIGNED) {
            if (item_rows_edge<MODE, RAD>(p, it))
                consume_item_lanes<MODE, RAD, true, SYM, SIG>(p, w, kd, it, ring, full, empty, sshift, slot, phase, gs);
            else
                consume_item_lanes<MODE, RAD, false, SYM, SIG>(p, w, kd, it, ring, full, empty, sshift, slot, phase, gs);
        } else if (item_rows_edge<MODE, RAD>(p, it))
            consume_item<MODE, RAD, true, SYM, true, SIG>(p, it, ring, full, empty, slot, phase, gs);
        else if (single_like(MODE) || it.x0 < RAD || it.x0 + p.tw > p.C - RAD)
            consume_item<MODE, RAD, false, SYM, true, SIG>(p, it, ring, full, empty, slot, phase, gs);
        else
            consume_item<MODE, RAD, false, SYM, false, SIG>(p, it, ring, full, empty, slot, phase, gs);
#ifdef SC_TRACE
        if (threadIdx.x == 32 && ntr < 8) SC_TR(p, 30 + ntr, clock64());
        ++ntr;
#endif
    }
#ifdef SC_TRACE
    if (threadIdx.x == 32) {
        SC_TR(p, 40, clock64());
        SC_TR(p, 41, trace_gt());
        SC_TR(p, 42, ntr);
    }
#endif
}

template <int MODE, int RAD, bool ALIGNED, int SYM = 0, bool SIG = false>
__global__ void __launch_bounds__(SC_MAXT, SC_MINB) sepconv_rows_kernel(const __grid_constant__ Params p) {
    static_assert(RAD <= MAX_RAD, "r > 4: sepconv_lanes_wide_kernel");
    rows_kernel_body<MODE, RAD, ALIGNED, SYM, SIG>(p, p.w, p.k);
}

// Widths 11..31 (r = 5..15), rows of any alignment: the generic producer and the
// lane-strided consumer with the taps of ParamsW.
// ALIGNED (two-pass modes, r <= 10): 16-B aligned rows, the adjacent-column consumer.
template <int MODE, int RAD, int SYM = 0, bool ALIGNED = false>
__global__ void __launch_bounds__(SC_MAXT, SC_MINB) sepconv_lanes_wide_kernel(const __grid_constant__ ParamsW p) {
    static_assert(RAD > MAX_RAD && RAD <= MAX_RAD_LANES, "r = 5..15");
    static_assert(!ALIGNED || (RAD <= MAX_RAD_ADJ && !single_like(MODE)), "aligned variant: two-pass modes, r <= 10");
    rows_kernel_body<MODE, RAD, ALIGNED, SYM, false>(p, p.wide_w, p.wide_k);
}

}  // namespace sc
