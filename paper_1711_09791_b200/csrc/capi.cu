// capi.cu -- C ABI of libsepconv_b200.so (declared in include/sepconv_b200.h).
//
// Validation mirrors the reference's checks before any launch:
//   shape/stride/range errors and aliasing -> SC_INVALID_ARGUMENT (S/conv.py:68-75)
//   plane smaller than the kernel          -> SC_INVALID_DIMENSION (S/conv.py:76-79)
//   width not odd in 1..9                  -> SC_UNSUPPORTED_WIDTH
// then plans the launch (strip width, row-band height, persistent grid) for the
// device that owns the buffers.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <vector>
#include <mutex>
#include <string>
#include <tuple>
#include <algorithm>
#include <array>
#include <unistd.h>

#include "../../include/sepconv_b200.h"
#include "direct.cuh"
#include "kernels.cuh"
#include "launch.h"

namespace sc {

static thread_local std::string t_err;
static std::atomic<uint64_t> g_launches{0};

void set_error(const std::string& msg) { t_err = msg; }
void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

static int fail(int code, const std::string& msg) {
    set_error(msg);
    return code;
}

static int cuda_fail(cudaError_t e, const char* what) {
    return fail(SC_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

int fail_arg(const std::string& msg) { return fail(SC_INVALID_ARGUMENT, msg); }
int fail_cuda(cudaError_t e, const std::string& what) {
    cudaGetLastError();
    return fail(SC_CUDA_ERROR, what + ": " + cudaGetErrorString(e));
}

// Tuning knobs (SC_* environment variables, 0 = unset), read in ONE pass over the
// environment per launch so a knob changed between calls still takes effect
// while the common case costs no getenv() per knob.
struct Knobs {
    int force_generic = 0, direct = 0, l2_evict_first = 0, debug_plan = 0;
    int occ = 0, ns = 0, nt = 0, band_h = 0, band_h2 = 0, tail_waves = 0, exact_waves = 0, ipc = 0, no_lanes_wide = 0, no_lean_single = 0, no_wide_adj = 0;
    int no_sym = 0, no_colsym = 0, no_pdl = 0, split_passes = 0, snapshot_fail = 0, peer_timeout_ms = 0;
    int u8_occ2 = 0;
    int u8_gen = 0;
};

static Knobs read_knobs() {
    Knobs k;
    for (char** e = environ; e && *e; ++e) {
        const char* s = *e;
        if (s[0] != 'S' || s[1] != 'C' || s[2] != '_') continue;
        const char* eq = std::strchr(s, '=');
        if (!eq || !eq[1]) continue;
        const std::string name(s + 3, eq - s - 3);
        const int v = std::atoi(eq + 1);
        if (name == "FORCE_GENERIC") k.force_generic = v;
        else if (name == "DIRECT") k.direct = v;
        else if (name == "L2_EVICT_FIRST") k.l2_evict_first = v;
        else if (name == "DEBUG_PLAN") k.debug_plan = v;
        else if (name == "OCC") k.occ = v;
        else if (name == "NS") k.ns = v;
        else if (name == "NT") k.nt = v;
        else if (name == "BAND_H") k.band_h = v;
        else if (name == "BAND_H2") k.band_h2 = v;
        else if (name == "TAIL_WAVES") k.tail_waves = v;
        else if (name == "EXACT_WAVES") k.exact_waves = v;
        else if (name == "IPC") k.ipc = v;
        else if (name == "NO_SYM") k.no_sym = v;
        else if (name == "NO_COLSYM") k.no_colsym = v;
        else if (name == "NO_PDL") k.no_pdl = v;
        else if (name == "SPLIT_PASSES") k.split_passes = v;
        else if (name == "SNAPSHOT_FAIL") k.snapshot_fail = v;
        else if (name == "PEER_TIMEOUT_MS") k.peer_timeout_ms = v;
        else if (name == "U8_OCC2") k.u8_occ2 = v;  // small u8 payloads on the 2-CTA build
        else if (name == "NO_WIDE_ADJ") k.no_wide_adj = v;  // widths 11..21 on aligned rows: the lane-strided consumer
        else if (name == "NO_LEAN_SINGLE") k.no_lean_single = v;  // general 7x7 / 9x9 single pass on the aligned kernel
        else if (name == "NO_LANES_WIDE") k.no_lanes_wide = v;  // widths 11..31 on the plain kernels
        else if (name == "U8_GEN") k.u8_gen = v;    // the general-geometry u8 build on aligned rows too
    }
    return k;
}

// --------------------------------------------------------------------------
// Device of a pointer (the caller's buffers decide where we launch)

static int select_device(const void* ptr) {
    cudaPointerAttributes attr;
    cudaError_t e = cudaPointerGetAttributes(&attr, ptr);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    if (attr.type != cudaMemoryTypeDevice && attr.type != cudaMemoryTypeManaged) return -1;
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess || cur != attr.device) cudaSetDevice(attr.device);
    return attr.device;
}

struct DevInfo {
    int sms = 0;
};

static DevInfo dev_info(int dev) {
    static std::mutex mu;
    static std::map<int, DevInfo> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    DevInfo d;
    cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = d;
    return d;
}

static int occupancy(const void* kern, int threads, size_t smem) {
    static std::mutex mu;
    static std::map<std::tuple<const void*, int, size_t, int>, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple(kern, threads, smem, dev);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    int occ = 0;
    if (smem > 227 * 1024 ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem) != cudaSuccess) {
        cudaGetLastError();
        occ = 0;  // infeasible (e.g. an SC_NS ring larger than shared memory)
    }
    if (occ < 0) occ = 0;
    cache[key] = occ;
    return occ;
}

// [next item, finished CTAs] ticket pairs for the kernels' dynamic item
// scheduling. The last CTA of a launch re-zeroes its pair, so a pair may be
// reused by any launch that is ORDERED after it:
//  * eager launches: one pair per (device, stream), keyed by the stream's
//    unique id (cudaStreamGetId: never reused within a context, unlike the
//    handle). Launches on one stream are ordered -- with programmatic dependent
//    launch too, since tickets are only claimed after griddepcontrol.wait, i.e.
//    after the previous grid completed. Launches on different streams never
//    share a pair, however many are queued.
//  * launches captured into a CUDA graph: a pair of their own, never handed out
//    again (replays of one graph are serialised by CUDA, and each replay's last
//    CTA re-zeroes it for the next).
// Pairs come from zeroed pools of kPoolPairs, allocated on demand with stream
// capture relaxed for this thread and zeroed on a private stream (no device-wide
// synchronisation, legal while the caller's stream is capturing).
static constexpr int kPoolPairs = 4096;

struct TicketPools {
    std::mutex mu;
    std::map<int, std::vector<int*>> pools;            // device -> pools
    std::map<int, long long> used;                     // device -> pairs handed out
    std::map<std::pair<int, unsigned long long>, int*> by_stream;  // (device, stream id) -> pair
};

static TicketPools& tickets() {
    static TicketPools t;
    return t;
}

static int* new_pair_locked(TicketPools& t, int dev) {
    long long& u = t.used[dev];
    std::vector<int*>& pools = t.pools[dev];
    if (u >= (long long)pools.size() * kPoolPairs) {
        cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
        cudaThreadExchangeStreamCaptureMode(&mode);
        int* b = nullptr;
        cudaStream_t zs = nullptr;
        bool ok = cudaMalloc(&b, sizeof(int) * 2 * kPoolPairs) == cudaSuccess &&
                  cudaStreamCreateWithFlags(&zs, cudaStreamNonBlocking) == cudaSuccess &&
                  cudaMemsetAsync(b, 0, sizeof(int) * 2 * kPoolPairs, zs) == cudaSuccess &&
                  cudaStreamSynchronize(zs) == cudaSuccess;
        if (zs) cudaStreamDestroy(zs);
        cudaThreadExchangeStreamCaptureMode(&mode);
        if (!ok) {
            cudaGetLastError();
            if (b) cudaFree(b);
            return nullptr;
        }
        pools.push_back(b);
    }
    int* pair = pools[u / kPoolPairs] + 2 * (u % kPoolPairs);
    ++u;
    return pair;
}

static int* work_slot(int dev, cudaStream_t s) {
    TicketPools& t = tickets();
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cap) != cudaSuccess) {
        cudaGetLastError();
        cap = cudaStreamCaptureStatusNone;
    }
    std::lock_guard<std::mutex> lk(t.mu);
    if (cap == cudaStreamCaptureStatusActive) return new_pair_locked(t, dev);
    unsigned long long id = 0;
    if (cudaStreamGetId(s, &id) != cudaSuccess) {
        cudaGetLastError();
        id = ~0ULL - reinterpret_cast<uintptr_t>(s);
    }
    int*& pair = t.by_stream[{dev, id}];
    if (!pair) pair = new_pair_locked(t, dev);
    return pair;
}

#ifdef SC_TRACE
// dev-only timeline buffer of the last launch (see TRACE_SLOTS in kernels.cuh)
static constexpr int kTraceCtas = 4096;
static unsigned long long* g_trace = nullptr;
static unsigned long long* trace_buffer() {
    if (!g_trace && cudaMalloc(&g_trace, sizeof(unsigned long long) * TRACE_SLOTS * kTraceCtas) != cudaSuccess) {
        cudaGetLastError();
        g_trace = nullptr;
    }
    return g_trace;
}
#endif

// --------------------------------------------------------------------------
// Planner


static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Launch geometry of one job; memoised per (kernel, device, shape, knobs) because
// planning costs more host time than the launch itself for small images.
struct Plan {
    int nt = 0, threads = 0, ns = 0, tw = 0, nstrips = 0, occ = 1, grid = 0;
    size_t smem = 0;
    int lo1 = 0, hi1 = 0, lo2 = 0, hi2 = 0, band_h = 1, band_h2 = 1, nitems = 0, nitems0 = 0;
};

using PlanKey = std::array<long long, 16>;

static int plan_rows(const RowsJob& j, const void* kern, bool aligned, bool direct, int dev, const Knobs& kn,
                     Plan& pl) {
    const int rad = j.width / 2;
    const bool seg2 = j.out_hi2 > j.out_lo2;
    const int COLS_PER_THREAD = cols_per_thread(j.mode, rad, aligned);  // 4-column groups (r > 4: column pairs) per consumer thread
    const int HL = halo_of(rad);
    int nt = 0, threads = 0, ns = 0, tw = 0;
    size_t smem = 0;
    if (direct) {
        nt = 32;
        tw = 128;
        threads = 32 * DWARPS;
    }
    const DevInfo di = dev_info(dev);
    const int occ_cap = kn.occ;
    const int lags = stage_lags(j.mode, rad);
    int ns_req = kn.ns ? kn.ns : 16 / SROWS;
    if (ns_req < lags + 2) ns_req = lags + 2;
    // widths 11..31: the fused kernel holds ceil(r/4) stages back for the ring
    // columns; keep two stages in flight beyond them (measured -2% at W = 11)
    if (rad > MAX_RAD && !kn.ns && ns_req < lags + 3) ns_req = lags + 3;
    if (ns_req > 32) ns_req = 32;
    auto smem_for = [&](int tw_, int ns_) {
        const int sw = aligned ? tw_ + 2 * HL : tw_ + 2 * HL + 16;  // row_width<ALIGNED, HL>
        return (size_t)((2 * ns_ * 8 + ns_ * 4 + ns_ * SROWS * 4 + 127) / 128) * 128 + (size_t)ns_ * SROWS * sw * 4;
    };
    // an SC_NS ring deeper than shared memory holds for the narrowest strip is clamped
    while (ns_req > lags + 2 && smem_for(COLS_PER_THREAD * 64, ns_req) > 227 * 1024) --ns_req;
    auto occ_for = [&](int threads_, size_t smem_) {
        int o = occupancy(kern, threads_, smem_);
        if (occ_cap > 0 && o > occ_cap) o = occ_cap;
        return o;
    };

    // Work split. Items are (plane, strip, row band), claimed from an atomic ticket
    // in order, so load balance only depends on the tail of a launch; every item
    // re-reads a 2r-row halo and every strip an 8-column halo.
    //  * large jobs (>= ~8 waves of 128-row items): 512-column strips (two-pass; the
    //    single pass, 8 columns per thread: 1024), a head of 128-row bands (halo
    //    4/128) and a tail of 32-row bands sized to two waves; mid-size jobs the same
    //    with 64/16-row bands;
    //  * small jobs: the strip width and a uniform band height are chosen together to
    //    give every CTA ~2 items (1 if that makes bands < 16 rows) at the least halo +
    //    padding cost (narrow strips are cheaper than short bands: 8/TW vs 2r/bh);
    //  * explicit two-segment jobs (a band's boundary strips) use short bands.
    int lo1 = j.out_lo, hi1 = j.out_hi, lo2 = seg2 ? j.out_lo2 : 0, hi2 = seg2 ? j.out_hi2 : 0;
    if (hi1 <= lo1) { lo1 = lo2; hi1 = hi2; lo2 = hi2 = 0; }
    const int rows_total = (hi1 - lo1) + (hi2 > lo2 ? hi2 - lo2 : 0);
    // every band re-reads 2r halo rows: radii above 4 take bands twice as tall
    // (measured at 3 x 8192^2: W = 11 -7%, W = 21 -4%)
    const bool tall_bands = rad > MAX_RAD;
    const int bh_tall = kn.band_h > 0 ? kn.band_h : (tall_bands ? 256 : 128);
    const int bh_short = kn.band_h2 > 0 ? kn.band_h2 : (tall_bands ? 64 : 32);
    int occ = 1, h1 = bh_short, h2 = bh_short, nstrips = 0;
    long long G = 1;
    if (direct) {
        occ = occ_for(threads, 0);
        if (occ < 1) return fail(SC_CUDA_ERROR, "direct kernel cannot be resident");
        G = (long long)di.sms * occ * DWARPS;
        nstrips = (j.C + tw - 1) / tw;
        const long long units = (long long)j.nplanes * nstrips;
        h1 = 64;
        while (h1 > 4 && units * ((rows_total + h1 - 1) / h1) < 2 * G) h1 /= 2;
        h2 = h1;
    } else {
        const int forced = kn.nt;
        const int tail_waves = kn.tail_waves > 0 ? kn.tail_waves : 2;
        static const int cand[] = {128, 96, 64, 160, 192, 256};
        double best_cost = 1e30;
        int best_head = 0, best_tall = bh_tall, best_short = bh_short;
        const int rows = hi1 - lo1;
        for (int c : cand) {
            if (forced && c != forced) continue;
            const int tw_ = COLS_PER_THREAD * c;
            const int strips = (j.C + tw_ - 1) / tw_;
            const long long units = (long long)j.nplanes * strips;
            const size_t sm = smem_for(tw_, ns_req);
            const int o = occ_for(32 + c, sm);
            if (o < 1) continue;
            const long long g = (long long)di.sms * o;
            // band heights scale with the job: fewer than ~8 waves of 128-row items
            // per CTA -> 64/16 (measured: cfg2 -11%, cfg3 -2.5% time; cfg5 keeps 128/32)
            int tall = bh_tall, shrt = bh_short;
            if (!kn.band_h && !kn.band_h2 && !tall_bands && units * (long long)rows < 8LL * g * 128) {
                tall = 64;
                shrt = 16;
            }
            // padding columns + the 8-column halo of every strip
            double cost = (double)(strips * tw_ + 2 * HL * strips) / j.C;
            // the in-place two-pass (split / no scratch) also snapshots 8 columns around
            // every strip boundary (written, then read back): wider strips pay
            // (measured at cfg5: 1024-column strips -3%; cfg3 -3%). Not for the
            // single pass + copy-back, whose plan it moved the wrong way (+3.5%).
            if (j.mode == MODE_SPLITF) cost += 16.0 * (strips - 1) / j.C;
            int head = 0, bh = shrt;
            if (seg2) {
                cost *= (double)(bh_short + 2 * rad) / bh_short;
            } else {
                const long long tail_rows = ((tail_waves * g + units - 1) / units) * (long long)shrt;
                if (rows > tail_rows + tall) {
                    head = (int)(((rows - tail_rows) / tall) * tall);
                    const long long bands = head / tall + (rows - head + shrt - 1) / shrt;
                    cost *= 1.0 + (double)(2 * rad) * bands / rows;
                } else {
                    // ~2 items per CTA for load balance; when that makes bands shorter
                    // than 16 rows the 2r halo rows dominate, so one taller item per CTA
                    // (measured: 3x1152^2 -7%, 3x1728^2 -5%)
                    // band height for k items per CTA, rounded UP so that the job
                    // is at most k whole waves (a floor here left a few CTAs with one
                    // item more than the rest: 945 items on 888 CTAs at 3x1152^2)
                    auto bh_for = [&](long long k) {
                        long long bands = k * g / units;
                        if (bands < 1) bands = 1;
                        return (rows + bands - 1) / bands;
                    };
                    long long b = bh_for(kn.ipc > 0 ? kn.ipc : 2);
                    if (kn.ipc == 0 && b < 16) b = bh_for(1);
                    if (b > tall) b = tall;
                    if (b < 4) b = 4;
                    bh = (int)b;
                    cost *= (double)(bh + 2 * rad) / bh;
                }
            }
            // fewer than ~12 consumer warps per SM cannot keep enough rows in flight
            const double warps = (double)o * c / 32.0;
            if (warps < 12.0) cost *= 12.0 / warps;
            // prefer the first (widest default) candidate unless another is clearly cheaper
            if (cost < best_cost * 0.99) {
                best_cost = cost;
                nt = c;
                occ = o;
                G = g;
                best_head = head;
                best_tall = tall;
                best_short = shrt;
                h1 = h2 = bh;
            }
        }
        if (nt == 0) return fail(SC_INVALID_ARGUMENT, "no launch configuration fits shared memory (SC_NS / SC_NT too large)");
        tw = COLS_PER_THREAD * nt;
        nstrips = (j.C + tw - 1) / tw;
        ns = ns_req;
        threads = 32 + nt;
        smem = smem_for(tw, ns);
        if (seg2) {
            h1 = h2 = bh_short;
        } else if (best_head > 0) {
            lo2 = lo1 + best_head;
            hi2 = hi1;
            hi1 = lo2;
            h1 = best_tall;
            h2 = best_short;
            // SC_EXACT_WAVES=1: stretch the head bands so the head is a whole number
            // of waves of items (every CTA gets the same number of head items)
            if (kn.exact_waves) {
                const long long units = (long long)j.nplanes * nstrips;
                const int head_rows = hi1 - lo1;
                long long waves = (units * ((head_rows + best_tall - 1) / best_tall) + G / 2) / G;
                if (waves < 1) waves = 1;
                // smallest band count >= waves*G/units, i.e. units*nb is a multiple of G when possible
                const long long nb = (waves * G + units - 1) / units;
                const int hb = (int)((head_rows + nb - 1) / nb);
                if (hb >= 8) h1 = hb;
            }
        }
    }
    const long long units = (long long)j.nplanes * nstrips;
    if (h1 > hi1 - lo1 && hi1 > lo1) h1 = hi1 - lo1;
    if (hi2 > lo2 && h2 > hi2 - lo2) h2 = hi2 - lo2;
    pl.band_h = h1 > 0 ? h1 : 1;
    pl.band_h2 = h2 > 0 ? h2 : 1;
    const long long nitems0 = hi1 > lo1 ? units * ((hi1 - lo1 + pl.band_h - 1) / pl.band_h) : 0;
    const long long nitems = nitems0 + (hi2 > lo2 ? units * ((hi2 - lo2 + pl.band_h2 - 1) / pl.band_h2) : 0);
    if (nitems > 0x7fffffffLL) return fail(SC_INVALID_ARGUMENT, "too many work items");
    const long long ctas = direct ? (nitems + DWARPS - 1) / DWARPS : nitems;
    pl.nt = nt;
    pl.threads = threads;
    pl.ns = ns;
    pl.tw = tw;
    pl.nstrips = nstrips;
    pl.occ = occ;
    pl.smem = smem;
    pl.lo1 = lo1;
    pl.hi1 = hi1;
    pl.lo2 = lo2;
    pl.hi2 = hi2;
    pl.nitems = (int)nitems;
    pl.nitems0 = (int)nitems0;
    pl.grid = (int)(ctas < (long long)di.sms * occ ? ctas : (long long)di.sms * occ);
    // The FP32-bound single pass (8 columns per thread: a 4-stage ring of 1032-float
    // rows is 66 KB, 3 CTAs/SM) runs better with one stage less and a 4th CTA once
    // every CTA has several items (measured: 3x8192^2 -3.7%, 3x16384^2 -4.4%,
    // 512 x 3x1080x1920 -5..7%); with ~1-2 items per CTA (3x4096^2) the shallower
    // ring loses (+4-6%).
    if (single_like(j.mode) && !direct && kn.ns == 0 && ns == 16 / SROWS && pl.nitems >= 4LL * pl.grid) {
        Knobs k3 = kn;
        k3.ns = 3;
        Plan p3;
        if (plan_rows(j, kern, aligned, direct, dev, k3, p3) == SC_OK && p3.occ > pl.occ) pl = p3;
    }
    return SC_OK;
}

// launch_rows status: the one-pass in-place modes could not get their snapshot
// buffer; the entry point runs the equivalent two-launch path instead
static constexpr int kNeedTwoLaunches = -100;

static int cached_plan(const RowsJob& j, const void* kern, bool aligned, bool direct, int dev, const Knobs& kn,
                       Plan& pl) {
    static std::mutex mu;
    static std::map<PlanKey, Plan> cache;
    const PlanKey key = {(long long)(uintptr_t)kern, (long long)direct, dev, j.nplanes, j.C, j.out_lo, j.out_hi,
                         j.out_lo2, j.out_hi2, kn.occ, kn.ns, kn.nt, kn.band_h, kn.band_h2,
                         (long long)kn.tail_waves * 2 + (kn.exact_waves != 0), (long long)aligned * 1024 + kn.ipc};
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) {
            pl = it->second;
            return SC_OK;
        }
    }
    const int rc = plan_rows(j, kern, aligned, direct, dev, kn, pl);
    if (rc != SC_OK) return rc;
    std::lock_guard<std::mutex> lk(mu);
    if (cache.size() >= 4096) cache.clear();
    cache[key] = pl;
    return SC_OK;
}

int launch_rows(const RowsJob& j, cudaStream_t s) {
    const int rad = j.width / 2;
    const Knobs kn = read_knobs();
    // widths 11..31: the lane-strided kernels (any alignment, neighbouring bands'
    // halo rows included); wider ones, and the signalled peer bands / in-place
    // modes above width 9, the plain kernels of kern_wide.cu
    const bool lanes_wide = j.width > MAX_W && j.width <= MAX_W_LANES && !kn.no_lanes_wide && !j.sig_self &&
                            (j.mode == MODE_FUSED || j.mode == MODE_HPASS || j.mode == MODE_VPASS ||
                             (j.mode == MODE_SINGLE && rad <= MAX_RAD_LANES_SINGLE));
    if (j.width > MAX_W && !lanes_wide) return launch_wide(j, s);
    const void* kern = nullptr;
    const bool peers_aligned = (!j.above || (aligned16(j.above) && j.above_ps % 4 == 0 && j.above_rs % 4 == 0)) &&
                               (!j.below || (aligned16(j.below) && j.below_ps % 4 == 0 && j.below_rs % 4 == 0));
    bool aligned = (j.C % 4 == 0) && aligned16(j.src) && aligned16(j.dst) && (j.sps % 4 == 0) &&
                   (j.dps % 4 == 0) && (j.srs % 4 == 0) && (j.drs % 4 == 0) && peers_aligned &&
                   kn.force_generic == 0 &&
                   // widths 11..31: aligned rows have their own consumer in the two-pass modes up to r = 10
                   (!lanes_wide || (j.mode != MODE_SINGLE && rad <= MAX_RAD_ADJ && !kn.no_wide_adj));
    // single pass with a mirror-symmetric dense matrix (bitwise K[i][j] == K[2r-i][j],
    // e.g. outer(w, w) of symmetric taps): the kernel that reuses mirrored products
    // (measured: -17% at cfg5 size; the same reuse in the two-pass column fold
    // measured 0-3% slower, so the two-pass modes do not use it)
    int sym = 0;  // 1: mirror-symmetric rows, 2: rows and columns (outer product of symmetric taps)
    if (!kn.no_sym && (j.mode == MODE_SINGLE || j.mode == MODE_SINGLECB) && j.dense) {
        const int W = j.width;
        auto same = [](float a, float b) { return std::memcmp(&a, &b, sizeof(float)) == 0; };
        bool rows = true, cols = true;
        for (int a = 0; a < W; ++a)
            for (int b = 0; b < W; ++b) {
                rows = rows && same(j.dense[a * W + b], j.dense[(W - 1 - a) * W + b]);
                cols = cols && same(j.dense[a * W + b], j.dense[a * W + (W - 1 - b)]);
            }
        sym = rows ? (cols && !kn.no_colsym ? 2 : 1) : 0;
    }
    // 7 x 7 and 9 x 9 matrices without mirror symmetry: the lane-strided kernel with
    // the rolled row loop (kernels.cuh, lean_of) beats the aligned kernel's
    // unrolled bodies, which overflow the instruction cache (-30% / -40%)
    if (j.mode == MODE_SINGLE && rad >= SC_LEAN_MIN_RAD && sym == 0 && !kn.no_lean_single) aligned = false;
    // two-pass modes: mirror-symmetric taps (bitwise) share their products
    bool symw = !kn.no_sym && (j.mode == MODE_FUSED || j.mode == MODE_SPLITF) && j.taps;
    for (int i = 0; i < j.width && symw; ++i) symw = std::memcmp(&j.taps[i], &j.taps[j.width - 1 - i], sizeof(float)) == 0;
    if (lanes_wide) {
        kern = j.mode == MODE_SINGLE ? kernel_lanes_wide_single(rad)
                                     : (rad <= 10 ? kernel_lanes_wide(j.mode, rad, symw, aligned)
                                                  : kernel_lanes_wide2(j.mode, rad, symw));
    } else
    switch (j.mode) {
        case MODE_FUSED: kern = kernel_fused(rad, aligned, symw, j.sig_self != nullptr); break;
        case MODE_HPASS: kern = kernel_hpass(rad, aligned); break;
        case MODE_VPASS: kern = kernel_vpass(rad, aligned); break;
        case MODE_SINGLE: kern = kernel_single(rad, aligned, sym); break;
        case MODE_SPLITF:
            if (!aligned) return fail(SC_INVALID_ARGUMENT, "split-fused kernel needs 16-B aligned rows");
            kern = kernel_splitf(rad, symw);
            break;
        case MODE_SINGLECB:
            if (!aligned) return fail(SC_INVALID_ARGUMENT, "in-place copy-back kernel needs 16-B aligned rows");
            kern = kernel_single_cb(rad, sym);
            break;
    }
    if (!kern) return fail(SC_UNSUPPORTED_WIDTH, "no kernel for width " + std::to_string(j.width));
    const bool seg2 = j.out_hi2 > j.out_lo2;
    if ((j.out_hi <= j.out_lo && !seg2) || j.nplanes <= 0) return SC_OK;

    // Kernel family: the TMA stage pipeline (default) or the register-streaming
    // direct kernel (SC_DIRECT=1), both bit-identical.
    const bool direct = aligned && kn.direct != 0 && !j.above && !j.below && !j.sig_self && j.mode != MODE_SPLITF &&
                        j.mode != MODE_SINGLECB;  // direct reads src only, no signalling
    if (direct) {
        switch (j.mode) {
            case MODE_FUSED: kern = kernel_fused_direct(rad); break;
            case MODE_HPASS: kern = kernel_hpass_direct(rad); break;
            case MODE_VPASS: kern = kernel_vpass_direct(rad); break;
            case MODE_SINGLE: kern = kernel_single_direct(rad); break;
        }
    }
    int dev = 0;
    cudaGetDevice(&dev);
    Plan pl;
    {
        const int rc = cached_plan(j, kern, aligned, direct, dev, kn, pl);
        if (rc != SC_OK) return rc;
    }

    ParamsW pw;  // the r <= 4 kernels take its Params part only
    std::memset(&pw, 0, sizeof(pw));
    Params& p = pw;
    p.src = j.src;
    p.dst = j.dst;
    p.src_plane_stride = j.sps;
    p.dst_plane_stride = j.dps;
    p.src_row_stride = j.srs;
    p.dst_row_stride = j.drs;
    p.nplanes = j.nplanes;
    p.R = j.R;
    p.C = j.C;
    p.src_row0 = j.src_row0;
    p.src_rows = j.src_rows;
    p.avail_lo = j.above ? j.above_row0 : j.src_row0;
    p.avail_hi = j.below ? j.below_row0 + j.below_rows : j.src_row0 + j.src_rows;
    p.above = j.above;
    p.below = j.below;
    p.above_ps = j.above_ps;
    p.above_rs = j.above_rs;
    p.below_ps = j.below_ps;
    p.below_rs = j.below_rs;
    p.above_row0 = j.above_row0;
    p.below_row0 = j.below_row0;
    p.dst_row0 = j.dst_row0;
    p.hrow_lo = j.hrow_lo;
    p.hrow_hi = j.hrow_hi;
    p.flags = j.flags;
    p.one = 1.0f;
    if (kn.l2_evict_first) p.flags |= F_L2_EVICT_FIRST;
    p.sig_self = j.sig_self;
    p.sig_above = j.sig_above;
    p.sig_below = j.sig_below;
    p.epoch = j.sig_self ? j.epoch : 0;
    p.sig_err = j.sig_err;
    p.sig_timeout_ns = (long long)(kn.peer_timeout_ms > 0 ? kn.peer_timeout_ms : 20000) * 1000000LL;
    {
        float* w = lanes_wide ? pw.wide_w : p.w;
        float* k = lanes_wide ? pw.wide_k : p.k;
        for (int i = 0; i < j.width; ++i) w[i] = j.taps ? j.taps[i] : 0.0f;
        if (j.dense)
            for (int i = 0; i < j.width * j.width; ++i) k[i] = j.dense[i];
    }
    p.tw = pl.tw;
    p.nstrips = pl.nstrips;
    p.ns = pl.ns;
    p.out_lo = pl.lo1;
    p.out_hi = pl.hi1;
    p.out_lo2 = pl.lo2;
    p.out_hi2 = pl.hi2;
    p.band_h = pl.band_h;
    p.band_h2 = pl.band_h2;
    p.nitems = pl.nitems;
    p.nitems0 = pl.nitems0;
    p.work = work_slot(dev, s);
    if (!p.work) return fail(SC_CUDA_ERROR, "cannot allocate the work counters");
    float* side = nullptr;
    if (j.mode == MODE_SPLITF || j.mode == MODE_SINGLECB) {
        // halo snapshot: stream-ordered scratch from the device's default pool
        // (kept pooled: release threshold raised once), taken right before the launch
        p.scr = j.scr;
        p.scr_ps = j.scr_ps;
        p.scr_rs = j.scr_rs;
        const long long units = (long long)j.nplanes * pl.nstrips;
        const int nb1 = (int)(pl.nitems0 / units);
        const int nb = (int)(pl.nitems / units);
        const size_t rows_f = (size_t)j.nplanes * nb * 2 * rad * j.C;
        const size_t cols_f = (size_t)j.nplanes * (pl.nstrips - 1) * j.R * 8;
        static std::once_flag pool_once[64];
        if (dev >= 0 && dev < 64)
            std::call_once(pool_once[dev], [dev]() {
                cudaMemPool_t pool;
                if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                    uint64_t thr = ~0ULL;
                    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
                }
                cudaGetLastError();
            });
        cudaError_t e = kn.snapshot_fail ? cudaErrorMemoryAllocation
                                         : cudaMallocAsync(reinterpret_cast<void**>(&side),
                                                           (rows_f + cols_f + 4) * sizeof(float), s);
        if (e != cudaSuccess) {
            // no room (or no stream-ordered allocator): the caller falls back to two launches
            cudaGetLastError();
            set_error(std::string("split snapshot allocation: ") + cudaGetErrorString(e));
            return kNeedTwoLaunches;
        }
        p.side_rows = side;
        p.side_cols = side + rows_f;
        p.side_nb = nb;
        p.snap_lo = pl.lo1;
        p.snap_hi = pl.hi2 > pl.lo2 ? pl.hi2 : pl.hi1;
        SnapJob sj{};
        sj.img = j.src;
        sj.ps = j.sps;
        sj.rs = j.srs;
        sj.nplanes = j.nplanes;
        sj.R = j.R;
        sj.C = j.C;
        sj.rad = rad;
        sj.tw = pl.tw;
        sj.nstrips = pl.nstrips;
        sj.lo1 = pl.lo1;
        sj.bh1 = pl.band_h;
        sj.nb1 = nb1;
        sj.lo2 = pl.lo2;
        sj.bh2 = pl.band_h2;
        sj.nb = nb;
        sj.side_rows = side;
        sj.side_cols = side + rows_f;
        e = launch_split_snapshot(sj, s);
        if (e != cudaSuccess) {
            cudaFreeAsync(side, s);
            return cuda_fail(e, "split snapshot launch");
        }
    }
#ifdef SC_TRACE
    p.trace = trace_buffer();
    if (p.trace) cudaMemsetAsync(p.trace, 0, sizeof(unsigned long long) * TRACE_SLOTS * kTraceCtas, s);
    if (pl.grid > kTraceCtas) p.trace = nullptr;
#endif

    void* args[] = {&pw};  // Params is ParamsW's base: same address
    // Programmatic dependent launch: this grid may be scheduled while the previous
    // kernel on the stream drains (its launch and smem/mbarrier setup overlap that
    // kernel's tail); the kernel itself waits (griddepcontrol.wait) for the
    // previous grid to complete before touching global memory.
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    cfg.gridDim = dim3(pl.grid);
    cfg.blockDim = dim3(pl.threads);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = s;
    if (!kn.no_pdl) {
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
    }
    if (p.epoch) {
        // per-launch counts of the items that read the band above / below (each
        // counts once when its copies have landed, kernels.cuh): every row band of
        // the plan whose input rows leave src, times the (plane, strip) units
        const long long units = (long long)j.nplanes * pl.nstrips;
        unsigned long long na = 0, nb = 0;
        auto count = [&](int lo, int hi, int bh) {
            for (int y = lo; y < hi; y += bh) {
                const int in_lo = std::max(std::max(y - rad, 0), (int)p.avail_lo);
                const int in_hi = std::min(std::min(std::min(y + bh, hi) + rad, j.R), (int)p.avail_hi);
                if (in_lo < j.src_row0) na += units;
                if (in_hi > j.src_row0 + j.src_rows) nb += units;
            }
        };
        if (pl.hi1 > pl.lo1) count(pl.lo1, pl.hi1, pl.band_h);
        if (pl.hi2 > pl.lo2) count(pl.lo2, pl.hi2, pl.band_h2);
        p.sig_n_above = na;
        p.sig_n_below = nb;
    }
    cudaError_t e = cudaLaunchKernelExC(&cfg, kern, args);
    if (side) cudaFreeAsync(side, s);  // after the kernel, in stream order
    if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
    count_launch();
    if (kn.debug_plan)
        std::fprintf(stderr, "[sc] mode=%d rad=%d aligned=%d nt=%d tw=%d strips=%d ns=%d seg1=[%d,%d)/%d seg2=[%d,%d)/%d items=%d grid=%d occ=%d smem=%zu\n",
                     j.mode, rad, (int)aligned, pl.nt, p.tw, p.nstrips, pl.ns, p.out_lo, p.out_hi, p.band_h, p.out_lo2,
                     p.out_hi2, p.band_h2, p.nitems, pl.grid, pl.occ, pl.smem);
    return SC_OK;
}

// --------------------------------------------------------------------------
// Fused read_ppm -> two-pass -> write_ppm on interleaved u8 (kern_u8.cu)

int launch_rows_u8(const uint8_t* src, uint8_t* dst, long long srs, long long drs, int R, int C, const float* taps,
                   int width, int flags, cudaStream_t s) {
    const int rad = width / 2;
    const Knobs kn = read_knobs();
    bool symw = !kn.no_sym;  // mirror-symmetric taps: shared products (bit-identical)
    for (int i = 0; i < width && symw; ++i) symw = std::memcmp(&taps[i], &taps[width - 1 - i], sizeof(float)) == 0;
    // payloads below 32 Mpixel: the 3-CTA build (<= 128 consumer threads)
    const bool large = (long long)R * C >= (1LL << 25);
    const bool occ3 = !large && u8_occ3_fits(rad, symw) && !kn.u8_occ2;
    // rows the TMA can copy as they are (16-B aligned, whole 16-B multiples) and
    // 4-B aligned destination rows; anything else runs the general build
    const bool gen = (C % 16) || (srs % 16) || (drs % 4) || (reinterpret_cast<uintptr_t>(src) & 15) ||
                     (reinterpret_cast<uintptr_t>(dst) & 3) || kn.u8_gen;
    const void* kern = kernel_u8(rad, symw, occ3, gen);
    if (!kern) return fail(SC_UNSUPPORTED_WIDTH, "no kernel for width " + std::to_string(width));
    U8Params p;
    std::memset(&p, 0, sizeof(p));
    p.src = src;
    p.dst = dst;
    p.srs = srs;
    p.drs = drs;
    p.R = R;
    p.C = C;
    p.hrow_lo = (flags & SC_EXTENDED) ? 0 : rad;
    p.hrow_hi = (flags & SC_EXTENDED) ? R : R - rad;
    p.flags = flags;
    if (large) p.flags |= F_U8_LEAN;  // >= 32 Mpixel: the lean loops pay
    p.one = 1.0f;
    for (int i = 0; i < width; ++i) p.w[i] = taps[i];
    // 4 columns per consumer thread; strips of TW = 4*nt columns, nt minimising padding
    static const int cand[] = {128, 96, 64, 160, 192, 256, 32};
    int nt = 128;
    long long best = -1;
    for (int c : cand) {
        if (occ3 && c > 128) continue;  // the 3-CTA build is bounded to 160 threads
        const long long tw = 4LL * c, waste = ((C + tw - 1) / tw) * tw - C;
        if (best < 0 || waste < best) { best = waste; nt = c; }
    }
    p.tw = 4 * nt;
    p.nstrips = (C + p.tw - 1) / p.tw;
    p.rowb = 3 * (p.tw + 2 * U8_HALO) + (gen ? 32 : 0);  // GEN: up to 15 bytes of 16-B widening each side
    int ns = kn.ns ? kn.ns : 4;
    if (ns < 3) ns = 3;
    if (ns > 32) ns = 32;
    p.ns = ns;
    const int threads = 32 + nt;
    const size_t smem = (size_t)((2 * ns * 8 + ns * 4 + 127) / 128) * 128 + (size_t)ns * U8_SROWS * p.rowb;
    int dev = 0;
    cudaGetDevice(&dev);
    const DevInfo di = dev_info(dev);
    const int occ = occupancy(kern, threads, smem);
    if (occ < 1) return fail(SC_INVALID_ARGUMENT, "no launch configuration fits shared memory (SC_NS too large)");
    const long long G = (long long)di.sms * occ;
    int band_h = kn.band_h ? kn.band_h : 64;
    while (band_h > 8 && (long long)p.nstrips * ((R + band_h - 1) / band_h) < 2 * G) band_h /= 2;
    if (band_h > R) band_h = R;
    p.band_h = band_h;
    const long long nitems = (long long)p.nstrips * ((R + band_h - 1) / band_h);
    p.nitems = (int)nitems;
    const int grid = (int)(nitems < G ? nitems : G);
    p.work = work_slot(dev, s);
    if (!p.work) return fail(SC_CUDA_ERROR, "cannot allocate the work counters");
    void* args[] = {&p};
    cudaError_t e = cudaLaunchKernel(kern, dim3(grid), dim3(threads), args, smem, s);
    if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
    count_launch();
    return SC_OK;
}

// --------------------------------------------------------------------------
// Validation helpers

static int check_width(int width) {
    if (width < 1 || width % 2 == 0)
        return fail(SC_INVALID_ARGUMENT, "kernel width must be odd and >= 1, got " + std::to_string(width));
    if (width > MAX_W_WIDE)
        return fail(SC_UNSUPPORTED_WIDTH,
                    "kernel width " + std::to_string(width) + " > " + std::to_string(MAX_W_WIDE) + " not supported");
    return SC_OK;
}

static int check_dims(int nplanes, int rows, int cols, int width) {
    if (nplanes < 1 || rows < 1 || cols < 1)
        return fail(SC_INVALID_ARGUMENT, "plane count and dimensions must be positive");
    if (rows < width || cols < width)
        return fail(SC_INVALID_DIMENSION, "plane " + std::to_string(rows) + "x" + std::to_string(cols) +
                                              " smaller than kernel width " + std::to_string(width));
    return SC_OK;
}

static int check_strides(int nplanes, int rows, int cols, long long ps, long long rs, const char* what) {
    if (rs < cols || (nplanes > 1 && ps < (long long)rows * rs))
        return fail(SC_INVALID_ARGUMENT, std::string(what) + ": strides overlap rows or planes");
    return SC_OK;
}

static long long extent_bytes(int nplanes, int rows, int cols, long long ps, long long rs) {
    return ((long long)(nplanes - 1) * ps + (long long)(rows - 1) * rs + cols) * 4LL;
}

static bool overlaps(const void* a, long long na, const void* b, long long nb) {
    const char* pa = static_cast<const char*>(a);
    const char* pb = static_cast<const char*>(b);
    return pa < pb + nb && pb < pa + na;
}

static int prepare(const void* ptr) {
    if (!ptr) return fail(SC_INVALID_ARGUMENT, "null buffer");
    if (select_device(ptr) < 0) return fail(SC_INVALID_ARGUMENT, "buffer is not device memory");
    return SC_OK;
}

}  // namespace sc

using namespace sc;

#define SC_TRY(x)                \
    do {                         \
        int _rc = (x);           \
        if (_rc != SC_OK) return _rc; \
    } while (0)

extern "C" {

int sc_abi_version(void) { return 1; }

const char* sc_last_error(void) { return t_err.c_str(); }

uint64_t sc_launch_count(void) { return g_launches.load(); }

#ifdef SC_TRACE
// dev-only (SC_TRACE builds): copy the last launch's per-CTA timeline to host
int sc_trace_copy(void* host, long long words) {
    if (!g_trace) return SC_INVALID_ARGUMENT;
    const long long n = words < (long long)TRACE_SLOTS * kTraceCtas ? words : (long long)TRACE_SLOTS * kTraceCtas;
    return cudaMemcpy(host, g_trace, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost) == cudaSuccess
               ? SC_OK : SC_CUDA_ERROR;
}
#endif

int sc_two_pass_band2_f32(const float* src, float* dst, int nplanes, int global_rows, int cols,
                          int64_t src_plane_stride, int64_t dst_plane_stride, int64_t src_row_stride,
                          int64_t dst_row_stride, int src_row0, int src_rows, int dst_row0, int out_lo, int out_hi,
                          int out_lo2, int out_hi2, const float* taps, int width, int flags, void* stream) {
    set_error("");
    SC_TRY(check_width(width));
    SC_TRY(check_dims(nplanes, global_rows, cols, width));
    if (!taps) return fail(SC_INVALID_ARGUMENT, "null taps");
    const int r = width / 2;
    if (out_lo < 0 || out_hi > global_rows || out_lo > out_hi || out_lo2 < 0 || out_hi2 > global_rows ||
        out_lo2 > out_hi2)
        return fail(SC_INVALID_ARGUMENT, "output rows out of range");
    const bool has1 = out_hi > out_lo, has2 = out_hi2 > out_lo2;
    if (has1 && has2 && out_lo < out_hi2 && out_lo2 < out_hi)
        return fail(SC_INVALID_ARGUMENT, "output segments overlap");
    if (!has1 && !has2) return SC_OK;
    const int lo_all = has1 && has2 ? (out_lo < out_lo2 ? out_lo : out_lo2) : (has1 ? out_lo : out_lo2);
    const int hi_all = has1 && has2 ? (out_hi > out_hi2 ? out_hi : out_hi2) : (has1 ? out_hi : out_hi2);
    const int need_lo = lo_all - r > 0 ? lo_all - r : 0;
    const int need_hi = hi_all + r < global_rows ? hi_all + r : global_rows;
    if (src_row0 > need_lo || src_row0 + src_rows < need_hi || src_row0 < 0 || src_row0 + src_rows > global_rows)
        return fail(SC_INVALID_ARGUMENT, "source band does not cover the output rows plus halo");
    if (dst_row0 > lo_all) return fail(SC_INVALID_ARGUMENT, "destination band starts after the output rows");
    SC_TRY(check_strides(nplanes, src_rows, cols, src_plane_stride, src_row_stride, "src"));
    SC_TRY(check_strides(nplanes, hi_all - dst_row0, cols, dst_plane_stride, dst_row_stride, "dst"));
    SC_TRY(prepare(src));
    SC_TRY(prepare(dst));
    if (overlaps(src, extent_bytes(nplanes, src_rows, cols, src_plane_stride, src_row_stride), dst,
                 extent_bytes(nplanes, hi_all - dst_row0, cols, dst_plane_stride, dst_row_stride)))
        return fail(SC_INVALID_ARGUMENT, "source and destination must be distinct buffers");
    RowsJob j{};
    j.mode = MODE_FUSED;
    j.src = src;
    j.dst = dst;
    j.sps = src_plane_stride;
    j.dps = dst_plane_stride;
    j.srs = src_row_stride;
    j.drs = dst_row_stride;
    j.nplanes = nplanes;
    j.R = global_rows;
    j.C = cols;
    j.src_row0 = src_row0;
    j.src_rows = src_rows;
    j.dst_row0 = dst_row0;
    j.out_lo = has1 ? out_lo : out_lo2;
    j.out_hi = has1 ? out_hi : out_hi2;
    j.out_lo2 = has1 ? out_lo2 : 0;
    j.out_hi2 = has1 ? out_hi2 : 0;
    j.hrow_lo = (flags & SC_EXTENDED) ? 0 : r;
    j.hrow_hi = (flags & SC_EXTENDED) ? global_rows : global_rows - r;
    j.flags = flags;
    j.width = width;
    j.taps = taps;
    return launch_rows(j, static_cast<cudaStream_t>(stream));
}

static int band_peer(const float* src, float* dst, int nplanes, int global_rows, int cols,
                     int64_t src_plane_stride, int64_t dst_plane_stride, int64_t src_row_stride,
                     int64_t dst_row_stride, int src_row0, int src_rows, const float* above,
                     int above_row0, int above_rows, int64_t above_plane_stride, int64_t above_row_stride,
                     const float* below, int below_row0, int below_rows, int64_t below_plane_stride,
                     int64_t below_row_stride, int dst_row0, int out_lo, int out_hi, const float* taps,
                     int width, int flags, uint64_t* sig_self, const uint64_t* sig_above, const uint64_t* sig_below,
                     uint64_t epoch, uint32_t* sig_err, void* stream) {
    set_error("");
    SC_TRY(check_width(width));
    SC_TRY(check_dims(nplanes, global_rows, cols, width));
    if (!taps) return fail(SC_INVALID_ARGUMENT, "null taps");
    const int r = width / 2;
    if (out_lo < 0 || out_hi > global_rows || out_lo > out_hi) return fail(SC_INVALID_ARGUMENT, "output rows out of range");
    if (out_hi == out_lo) return SC_OK;
    if (src_row0 < 0 || src_rows < 1 || src_row0 + src_rows > global_rows)
        return fail(SC_INVALID_ARGUMENT, "source band outside the image");
    // neighbours must be the adjacent bands: above ends where src starts, below starts where src ends
    if (above && (above_rows < 1 || above_row0 < 0 || above_row0 + above_rows != src_row0))
        return fail(SC_INVALID_ARGUMENT, "the band above must end at src_row0");
    if (below && (below_rows < 1 || below_row0 != src_row0 + src_rows || below_row0 + below_rows > global_rows))
        return fail(SC_INVALID_ARGUMENT, "the band below must start at src_row0 + src_rows");
    const int avail_lo = above ? above_row0 : src_row0;
    const int avail_hi = below ? below_row0 + below_rows : src_row0 + src_rows;
    const int need_lo = out_lo - r > 0 ? out_lo - r : 0;
    const int need_hi = out_hi + r < global_rows ? out_hi + r : global_rows;
    if (avail_lo > need_lo || avail_hi < need_hi)
        return fail(SC_INVALID_ARGUMENT, "source band and neighbours do not cover the output rows plus halo");
    if (dst_row0 > out_lo) return fail(SC_INVALID_ARGUMENT, "destination band starts after the output rows");
    SC_TRY(check_strides(nplanes, src_rows, cols, src_plane_stride, src_row_stride, "src"));
    SC_TRY(check_strides(nplanes, out_hi - dst_row0, cols, dst_plane_stride, dst_row_stride, "dst"));
    if (above) SC_TRY(check_strides(nplanes, above_rows, cols, above_plane_stride, above_row_stride, "above"));
    if (below) SC_TRY(check_strides(nplanes, below_rows, cols, below_plane_stride, below_row_stride, "below"));
    // the caller's own buffers pick the device; neighbours are peer mappings (never
    // passed to the device selection, which would switch to their owning GPU)
    SC_TRY(prepare(src));
    SC_TRY(prepare(dst));
    if (overlaps(src, extent_bytes(nplanes, src_rows, cols, src_plane_stride, src_row_stride), dst,
                 extent_bytes(nplanes, out_hi - dst_row0, cols, dst_plane_stride, dst_row_stride)))
        return fail(SC_INVALID_ARGUMENT, "source and destination must be distinct buffers");
    RowsJob j{};
    j.mode = MODE_FUSED;
    j.src = src;
    j.dst = dst;
    j.sps = src_plane_stride;
    j.dps = dst_plane_stride;
    j.srs = src_row_stride;
    j.drs = dst_row_stride;
    j.nplanes = nplanes;
    j.R = global_rows;
    j.C = cols;
    j.src_row0 = src_row0;
    j.src_rows = src_rows;
    j.dst_row0 = dst_row0;
    j.out_lo = out_lo;
    j.out_hi = out_hi;
    j.hrow_lo = (flags & SC_EXTENDED) ? 0 : r;
    j.hrow_hi = (flags & SC_EXTENDED) ? global_rows : global_rows - r;
    j.flags = flags;
    j.width = width;
    j.taps = taps;
    j.above = above;
    j.above_row0 = above_row0;
    j.above_rows = above_rows;
    j.above_ps = above_plane_stride;
    j.above_rs = above_row_stride;
    j.below = below;
    j.below_row0 = below_row0;
    j.below_rows = below_rows;
    j.below_ps = below_plane_stride;
    j.below_rs = below_row_stride;
    if (sig_self && epoch) {
        if (width > MAX_W) return fail(SC_UNSUPPORTED_WIDTH, "signalled row bands support widths up to 9");
        j.sig_self = reinterpret_cast<unsigned long long*>(sig_self);
        j.sig_above = reinterpret_cast<const unsigned long long*>(sig_above);
        j.sig_below = reinterpret_cast<const unsigned long long*>(sig_below);
        j.epoch = epoch;
        j.sig_err = sig_err;
    }
    return launch_rows(j, static_cast<cudaStream_t>(stream));
}

int sc_two_pass_band_peer_f32(const float* src, float* dst, int nplanes, int global_rows, int cols,
                              int64_t src_plane_stride, int64_t dst_plane_stride, int64_t src_row_stride,
                              int64_t dst_row_stride, int src_row0, int src_rows, const float* above,
                              int above_row0, int above_rows, int64_t above_plane_stride, int64_t above_row_stride,
                              const float* below, int below_row0, int below_rows, int64_t below_plane_stride,
                              int64_t below_row_stride, int dst_row0, int out_lo, int out_hi, const float* taps,
                              int width, int flags, void* stream) {
    return band_peer(src, dst, nplanes, global_rows, cols, src_plane_stride, dst_plane_stride, src_row_stride,
                     dst_row_stride, src_row0, src_rows, above, above_row0, above_rows, above_plane_stride,
                     above_row_stride, below, below_row0, below_rows, below_plane_stride, below_row_stride, dst_row0,
                     out_lo, out_hi, taps, width, flags, nullptr, nullptr, nullptr, 0, nullptr, stream);
}

int sc_two_pass_band_peer_sig_f32(const float* src, float* dst, int nplanes, int global_rows, int cols,
                                  int64_t src_plane_stride, int64_t dst_plane_stride, int64_t src_row_stride,
                                  int64_t dst_row_stride, int src_row0, int src_rows, const float* above,
                                  int above_row0, int above_rows, int64_t above_plane_stride,
                                  int64_t above_row_stride, const float* below, int below_row0, int below_rows,
                                  int64_t below_plane_stride, int64_t below_row_stride, int dst_row0, int out_lo,
                                  int out_hi, const float* taps, int width, int flags, uint64_t* sig_self,
                                  const uint64_t* sig_above, const uint64_t* sig_below, uint64_t epoch,
                                  uint32_t* sig_err, void* stream) {
    if (!sig_self || epoch == 0) {
        set_error("signalled band step needs this band's signal words and an epoch > 0");
        return SC_INVALID_ARGUMENT;
    }
    return band_peer(src, dst, nplanes, global_rows, cols, src_plane_stride, dst_plane_stride, src_row_stride,
                     dst_row_stride, src_row0, src_rows, above, above_row0, above_rows, above_plane_stride,
                     above_row_stride, below, below_row0, below_rows, below_plane_stride, below_row_stride, dst_row0,
                     out_lo, out_hi, taps, width, flags, sig_self, sig_above, sig_below, epoch, sig_err, stream);
}

int sc_band_signal_wait(const uint64_t* sig_above, const uint64_t* sig_below, int word, uint64_t value,
                        uint32_t* sig_err, void* stream) {
    set_error("");
    if (word < 0 || word > 1) return fail(SC_INVALID_ARGUMENT, "signal word must be 0 (ready) or 1 (done)");
    if (!sig_above && !sig_below) return SC_OK;
    const Knobs kn = read_knobs();
    const long long tmo = (long long)(kn.peer_timeout_ms > 0 ? kn.peer_timeout_ms : 20000) * 1000000LL;
    cudaError_t e = launch_signal_wait(reinterpret_cast<const unsigned long long*>(sig_above),
                                       reinterpret_cast<const unsigned long long*>(sig_below), word, value, sig_err,
                                       tmo, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "signal wait launch");
    return SC_OK;
}

// IPC: export a device buffer to another process (its allocation's handle plus the
// buffer's offset inside the allocation), and map such a buffer into this process
// on the CURRENT device (peer access over NVLink enabled on demand).
typedef int (*AddrRangeFn)(unsigned long long*, size_t*, unsigned long long);

int sc_ipc_export(const void* ptr, void* handle_out, int64_t* offset_out) {
    set_error("");
    if (!ptr || !handle_out || !offset_out) return fail(SC_INVALID_ARGUMENT, "null argument");
    SC_TRY(prepare(ptr));
    static AddrRangeFn range = nullptr;
    if (!range) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
            cudaGetLastError();
            return fail(SC_CUDA_ERROR, "cuMemGetAddressRange unavailable");
        }
        range = reinterpret_cast<AddrRangeFn>(fn);
    }
    unsigned long long base = 0;
    size_t size = 0;
    if (range(&base, &size, reinterpret_cast<unsigned long long>(ptr)) != 0)
        return fail(SC_CUDA_ERROR, "cannot resolve the allocation of the buffer");
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
    std::memcpy(handle_out, &h, sizeof(h));
    *offset_out = (int64_t)(reinterpret_cast<unsigned long long>(ptr) - base);
    return SC_OK;
}

int sc_ipc_open(const void* handle, int64_t offset, int device, void** ptr_out) {
    set_error("");
    if (!handle || !ptr_out || offset < 0) return fail(SC_INVALID_ARGUMENT, "null argument or negative offset");
    // this library carries its own CUDA runtime: its current device is not the
    // caller's, so the device that will read the mapping is named explicitly
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess || cur != device) {
        cudaError_t se = cudaSetDevice(device);
        if (se != cudaSuccess) return cuda_fail(se, "cudaSetDevice");
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void* base = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
    *ptr_out = static_cast<char*>(base) + offset;
    return SC_OK;
}

int sc_ipc_close(void* ptr, int64_t offset) {
    set_error("");
    if (!ptr) return fail(SC_INVALID_ARGUMENT, "null pointer");
    cudaError_t e = cudaIpcCloseMemHandle(static_cast<char*>(ptr) - offset);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcCloseMemHandle");
    return SC_OK;
}

int sc_two_pass_band_f32(const float* src, float* dst, int nplanes, int global_rows, int cols,
                         int64_t src_plane_stride, int64_t dst_plane_stride, int64_t src_row_stride,
                         int64_t dst_row_stride, int src_row0, int src_rows, int dst_row0, int out_lo, int out_hi,
                         const float* taps, int width, int flags, void* stream) {
    return sc_two_pass_band2_f32(src, dst, nplanes, global_rows, cols, src_plane_stride, dst_plane_stride,
                                 src_row_stride, dst_row_stride, src_row0, src_rows, dst_row0, out_lo, out_hi, 0, 0,
                                 taps, width, flags, stream);
}

int sc_two_pass_fused_f32(const float* src, float* dst, int nplanes, int rows, int cols, int64_t src_plane_stride,
                          int64_t dst_plane_stride, int64_t src_row_stride, int64_t dst_row_stride,
                          const float* taps, int width, int flags, void* stream) {
    return sc_two_pass_band_f32(src, dst, nplanes, rows, cols, src_plane_stride, dst_plane_stride, src_row_stride,
                                dst_row_stride, 0, rows, 0, 0, rows, taps, width, flags, stream);
}

static int pass_common(int mode, const float* src, float* dst, int nplanes, int rows, int cols, int64_t sps,
                       int64_t dps, int64_t srs, int64_t drs, int row_lo, int row_hi, const float* taps,
                       const float* dense, int width, int flags, void* stream) {
    SC_TRY(check_width(width));
    SC_TRY(check_dims(nplanes, rows, cols, width));
    if (single_like(mode) ? !dense : !taps) return fail(SC_INVALID_ARGUMENT, "null taps");
    SC_TRY(check_strides(nplanes, rows, cols, sps, srs, "src"));
    SC_TRY(check_strides(nplanes, rows, cols, dps, drs, "dst"));
    const int r = width / 2;
    if (mode == MODE_HPASS) {
        if (row_lo < 0 || row_hi > rows || row_lo > row_hi)
            return fail(SC_INVALID_ARGUMENT, "row range out of bounds");
    } else {
        if (row_lo > row_hi || (row_hi > row_lo && (row_lo < r || row_hi > rows - r)))
            return fail(SC_INVALID_ARGUMENT, "row range must lie inside the valid rows");
    }
    SC_TRY(prepare(src));
    SC_TRY(prepare(dst));
    if (overlaps(src, extent_bytes(nplanes, rows, cols, sps, srs), dst, extent_bytes(nplanes, rows, cols, dps, drs)))
        return fail(SC_INVALID_ARGUMENT, "source and destination must be distinct buffers");
    RowsJob j{};
    j.mode = mode;
    j.src = src;
    j.dst = dst;
    j.sps = sps;
    j.dps = dps;
    j.srs = srs;
    j.drs = drs;
    j.nplanes = nplanes;
    j.R = rows;
    j.C = cols;
    j.src_row0 = 0;
    j.src_rows = rows;
    j.dst_row0 = 0;
    j.hrow_lo = row_lo;
    j.hrow_hi = row_hi;
    if (mode == MODE_HPASS && (flags & SC_ZERO_FILL)) {
        j.out_lo = 0;
        j.out_hi = rows;
    } else {
        j.out_lo = row_lo;
        j.out_hi = row_hi;
    }
    j.flags = flags;
    j.width = width;
    j.taps = taps;
    j.dense = dense;
    if (single_like(mode)) {
        static float zeros[MAX_W_WIDE] = {0};
        j.taps = zeros;
    }
    if (mode == MODE_SINGLECB) {  // second destination: the source image itself (copy-back, in place)
        j.scr = const_cast<float*>(src);
        j.scr_ps = sps;
        j.scr_rs = srs;
    }
    return launch_rows(j, static_cast<cudaStream_t>(stream));
}

int sc_hpass_f32(const float* src, float* dst, int nplanes, int rows, int cols, int64_t src_plane_stride,
                 int64_t dst_plane_stride, int64_t src_row_stride, int64_t dst_row_stride, int row_lo, int row_hi,
                 const float* taps, int width, int flags, void* stream) {
    set_error("");
    return pass_common(MODE_HPASS, src, dst, nplanes, rows, cols, src_plane_stride, dst_plane_stride,
                       src_row_stride, dst_row_stride, row_lo, row_hi, taps, nullptr, width, flags, stream);
}

int sc_vpass_f32(const float* src, float* dst, int nplanes, int rows, int cols, int64_t src_plane_stride,
                 int64_t dst_plane_stride, int64_t src_row_stride, int64_t dst_row_stride, int row_lo, int row_hi,
                 const float* taps, int width, int flags, void* stream) {
    set_error("");
    return pass_common(MODE_VPASS, src, dst, nplanes, rows, cols, src_plane_stride, dst_plane_stride,
                       src_row_stride, dst_row_stride, row_lo, row_hi, taps, nullptr, width, flags, stream);
}

int sc_two_pass_split_f32(float* image, float* scratch, int nplanes, int rows, int cols, int64_t image_plane_stride,
                          int64_t scratch_plane_stride, int64_t image_row_stride, int64_t scratch_row_stride,
                          const float* taps, int width, int flags, void* stream) {
    set_error("");
    SC_TRY(check_width(width));
    SC_TRY(check_dims(nplanes, rows, cols, width));
    const int r = width / 2;
    const int h_lo = (flags & SC_EXTENDED) ? 0 : r;
    const int h_hi = (flags & SC_EXTENDED) ? rows : rows - r;
    // One pass (image read once; scratch and image written once) when every row is
    // 16-B aligned; otherwise (or SC_SPLIT_PASSES=1) the row pass + column pass pair.
    const Knobs kn = read_knobs();
    const bool aligned = cols % 4 == 0 && aligned16(image) && aligned16(scratch) && image_plane_stride % 4 == 0 &&
                         scratch_plane_stride % 4 == 0 && image_row_stride % 4 == 0 && scratch_row_stride % 4 == 0 &&
                         !kn.force_generic;
    if (aligned && !kn.split_passes && width <= MAX_W) {
        SC_TRY(check_strides(nplanes, rows, cols, image_plane_stride, image_row_stride, "image"));
        SC_TRY(check_strides(nplanes, rows, cols, scratch_plane_stride, scratch_row_stride, "scratch"));
        SC_TRY(prepare(image));
        SC_TRY(prepare(scratch));
        if (overlaps(image, extent_bytes(nplanes, rows, cols, image_plane_stride, image_row_stride), scratch,
                     extent_bytes(nplanes, rows, cols, scratch_plane_stride, scratch_row_stride)))
            return fail(SC_INVALID_ARGUMENT, "source and destination must be distinct buffers");
        if (!taps) return fail(SC_INVALID_ARGUMENT, "null taps");
        RowsJob j{};
        j.mode = MODE_SPLITF;
        j.src = image;
        j.dst = image;
        j.sps = image_plane_stride;
        j.dps = image_plane_stride;
        j.srs = image_row_stride;
        j.drs = image_row_stride;
        j.nplanes = nplanes;
        j.R = rows;
        j.C = cols;
        j.src_row0 = 0;
        j.src_rows = rows;
        j.dst_row0 = 0;
        j.out_lo = 0;
        j.out_hi = rows;
        j.hrow_lo = h_lo;
        j.hrow_hi = h_hi;
        j.flags = (flags & SC_EXTENDED) | SC_NO_RING;
        j.width = width;
        j.taps = taps;
        j.scr = scratch;
        j.scr_ps = scratch_plane_stride;
        j.scr_rs = scratch_row_stride;
        const int rc = launch_rows(j, static_cast<cudaStream_t>(stream));
        if (rc != kNeedTwoLaunches) return rc;
        set_error("");
    }
    SC_TRY(pass_common(MODE_HPASS, image, scratch, nplanes, rows, cols, image_plane_stride, scratch_plane_stride,
                       image_row_stride, scratch_row_stride, h_lo, h_hi, taps, nullptr, width, SC_ZERO_FILL,
                       stream));
    return pass_common(MODE_VPASS, scratch, image, nplanes, rows, cols, scratch_plane_stride, image_plane_stride,
                       scratch_row_stride, image_row_stride, r, rows - r, taps, nullptr, width, 0, stream);
}

int sc_two_pass_inplace_f32(float* image, int nplanes, int rows, int cols, int64_t plane_stride, int64_t row_stride,
                            const float* taps, int width, int flags, void* stream) {
    set_error("");
    SC_TRY(check_width(width));
    SC_TRY(check_dims(nplanes, rows, cols, width));
    if (!taps) return fail(SC_INVALID_ARGUMENT, "null taps");
    SC_TRY(check_strides(nplanes, rows, cols, plane_stride, row_stride, "image"));
    SC_TRY(prepare(image));
    const int r = width / 2;
    const int h_lo = (flags & SC_EXTENDED) ? 0 : r;
    const int h_hi = (flags & SC_EXTENDED) ? rows : rows - r;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const Knobs kn = read_knobs();
    const bool aligned = cols % 4 == 0 && aligned16(image) && plane_stride % 4 == 0 && row_stride % 4 == 0 &&
                         !kn.force_generic;
    if (aligned && !kn.split_passes && width <= MAX_W) {
        // the one-pass split kernel without its scratch writes: each item reads its
        // own rows before overwriting them, other items' halos from the pre-launch
        // snapshot -- 2 traversals (+ the ~5% snapshot) instead of 3
        RowsJob j{};
        j.mode = MODE_SPLITF;
        j.src = image;
        j.dst = image;
        j.sps = j.dps = plane_stride;
        j.srs = j.drs = row_stride;
        j.nplanes = nplanes;
        j.R = rows;
        j.C = cols;
        j.src_row0 = 0;
        j.src_rows = rows;
        j.dst_row0 = 0;
        j.out_lo = 0;
        j.out_hi = rows;
        j.hrow_lo = h_lo;
        j.hrow_hi = h_hi;
        j.flags = (flags & SC_EXTENDED) | SC_NO_RING;
        j.width = width;
        j.taps = taps;
        j.scr = nullptr;
        const int rc = launch_rows(j, s);
        if (rc != kNeedTwoLaunches) return rc;
        set_error("");
    }
    // any other shape: H0 into a stream-ordered temporary, then the column pass
    float* tmp = nullptr;
    const size_t n = (size_t)nplanes * rows * cols;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&tmp), n * sizeof(float), s);
    if (e != cudaSuccess) return cuda_fail(e, "in-place two-pass scratch allocation");
    const long long tps = (long long)rows * cols;
    int rc = pass_common(MODE_HPASS, image, tmp, nplanes, rows, cols, plane_stride, tps, row_stride, cols, h_lo, h_hi,
                         taps, nullptr, width, SC_ZERO_FILL, stream);
    if (rc == SC_OK)
        rc = pass_common(MODE_VPASS, tmp, image, nplanes, rows, cols, tps, plane_stride, cols, row_stride, r, rows - r,
                         taps, nullptr, width, 0, stream);
    cudaFreeAsync(tmp, s);
    return rc;
}

int sc_single_pass_f32(float* src, float* dst, int nplanes, int rows, int cols, int64_t src_plane_stride,
                       int64_t dst_plane_stride, int64_t src_row_stride, int64_t dst_row_stride, const float* dense,
                       int width, int flags, void* stream) {
    set_error("");
    SC_TRY(check_width(width));
    SC_TRY(check_dims(nplanes, rows, cols, width));
    const int r = width / 2;
    const Knobs kn = read_knobs();
    const bool aligned = cols % 4 == 0 && aligned16(src) && aligned16(dst) && src_plane_stride % 4 == 0 &&
                         dst_plane_stride % 4 == 0 && src_row_stride % 4 == 0 && dst_row_stride % 4 == 0 &&
                         !kn.force_generic && !kn.direct;
    // a 7 x 7 / 9 x 9 matrix without mirror-symmetric rows: the rolled single pass +
    // the region copy beat the one-pass kernel's unrolled bodies (instruction cache;
    // measured at 3 x 8192^2: 1.32 -> 1.00 ms, 2.28 -> 1.47 ms)
    bool lean_two_launches = false;
    if ((flags & SC_COPY_BACK) && r >= SC_LEAN_MIN_RAD && width <= MAX_W && dense && !kn.no_lean_single) {
        bool rows_sym = !kn.no_sym;
        for (int a = 0; a < width && rows_sym; ++a)
            for (int b = 0; b < width && rows_sym; ++b)
                rows_sym = std::memcmp(&dense[a * width + b], &dense[(width - 1 - a) * width + b], sizeof(float)) == 0;
        lean_two_launches = !rows_sym;
    }
    if ((flags & SC_COPY_BACK) && aligned && !kn.split_passes && width <= MAX_W && !lean_two_launches) {
        // one pass: the valid region into the workspace and back into the image
        const int rc = pass_common(MODE_SINGLECB, src, dst, nplanes, rows, cols, src_plane_stride,
                                   dst_plane_stride, src_row_stride, dst_row_stride, r, rows - r, nullptr, dense,
                                   width, flags, stream);
        if (rc != kNeedTwoLaunches) return rc;
        set_error("");
    }
    SC_TRY(pass_common(MODE_SINGLE, src, dst, nplanes, rows, cols, src_plane_stride, dst_plane_stride,
                       src_row_stride, dst_row_stride, r, rows - r, nullptr, dense, width, flags, stream));
    if (flags & SC_COPY_BACK) {
        cudaError_t e = launch_copy_region(dst, src, dst_plane_stride, src_plane_stride, dst_row_stride,
                                           src_row_stride, nplanes, r, rows - 2 * r, r, cols - 2 * r,
                                           static_cast<cudaStream_t>(stream));
        if (e != cudaSuccess) return cuda_fail(e, "copy-back launch");
    }
    return SC_OK;
}

int sc_copy_region_f32(const float* src, float* dst, int nplanes, int rows, int cols, int64_t src_plane_stride,
                       int64_t dst_plane_stride, int64_t src_row_stride, int64_t dst_row_stride, int row_lo,
                       int row_hi, int col_lo, int col_hi, void* stream) {
    set_error("");
    if (nplanes < 1 || rows < 1 || cols < 1) return fail(SC_INVALID_ARGUMENT, "dimensions must be positive");
    if (!(0 <= row_lo && row_lo <= row_hi && row_hi <= rows && 0 <= col_lo && col_lo <= col_hi && col_hi <= cols))
        return fail(SC_INVALID_ARGUMENT, "region out of bounds");
    SC_TRY(check_strides(nplanes, rows, cols, src_plane_stride, src_row_stride, "src"));
    SC_TRY(check_strides(nplanes, rows, cols, dst_plane_stride, dst_row_stride, "dst"));
    SC_TRY(prepare(src));
    SC_TRY(prepare(dst));
    if (overlaps(src, extent_bytes(nplanes, rows, cols, src_plane_stride, src_row_stride), dst,
                 extent_bytes(nplanes, rows, cols, dst_plane_stride, dst_row_stride)))
        return fail(SC_INVALID_ARGUMENT, "source and destination must be distinct buffers");
    cudaError_t e = launch_copy_region(src, dst, src_plane_stride, dst_plane_stride, src_row_stride, dst_row_stride,
                                       nplanes, row_lo, row_hi - row_lo, col_lo, col_hi - col_lo,
                                       static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "copy launch");
    return SC_OK;
}

int sc_fill_synthetic_f32(float* dst, int64_t count, uint64_t seed, uint64_t offset, int kind, void* stream) {
    set_error("");
    if (count < 0 || kind < 0 || kind > 2) return fail(SC_INVALID_ARGUMENT, "bad count or kind");
    if (count == 0) return SC_OK;
    SC_TRY(prepare(dst));
    cudaError_t e = launch_fill_synthetic(dst, count, seed, offset, kind, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "fill launch");
    return SC_OK;
}

}  // extern "C"
