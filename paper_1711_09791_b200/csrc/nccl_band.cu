// nccl_band.cu -- the NCCL transport of the multi-GPU row-band step (SURVEY.md
// section 8e: "ncclGroupStart; ncclSend(rows [lo, lo+2) -> g-1); ncclRecv(rows
// [lo-2, lo) <- g-1); ncclSend(rows [hi-2, hi) -> g+1); ncclRecv(rows [hi, hi+2)
// <- g+1); ncclGroupEnd, as one packed 3x2xC buffer per neighbour. Overlap with
// the interior kernel; the boundary rows run after the recv").
//
// A band plan owns, per neighbour, ONE packed send buffer and ONE receive buffer
// of nplanes x r x cols floats, a communication stream and two events. A step:
//   comm stream : wait(inputs ready) -> pack the r boundary rows of every plane
//                 (one launch for both sides) -> one NCCL group (send + recv per
//                 neighbour)
//   caller's    : interior rows [lo+r, hi-r) (they need no halo) -> wait(exchange)
//   stream        -> ONE launch for both boundary strips, whose producer reads the
//                 halo rows straight from the receive buffers (the kernel's
//                 above/below row sources, no unpack copy)
// Steps are issued eagerly by default (~25 us of host time, measured; far below
// the GPU time of a step). use_graph captures the step once into a CUDA graph
// (NCCL operations capture); measured on one B200 its launch cost the host MORE
// (~100 us per step with the NCCL nodes), so it is opt-in.
//
// libnccl.so.2 is loaded at run time (the one torch already mapped, if any):
// the library itself does not link against NCCL.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/sepconv_b200.h"
#include "kernels.cuh"
#include "launch.h"

namespace sc {

struct NcclApi {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    bool ok = false;
    std::string why;
};

static const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            api.why = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
            return;
        }
#define SC_SYM(field, name)                                                   \
    api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, #name));       \
    if (!api.field) {                                                         \
        api.why = "libnccl.so.2 lacks " #name;                                \
        return;                                                               \
    }
        SC_SYM(get_unique_id, ncclGetUniqueId)
        SC_SYM(comm_init_rank, ncclCommInitRank)
        SC_SYM(comm_destroy, ncclCommDestroy)
        SC_SYM(group_start, ncclGroupStart)
        SC_SYM(group_end, ncclGroupEnd)
        SC_SYM(send, ncclSend)
        SC_SYM(recv, ncclRecv)
        SC_SYM(error_string, ncclGetErrorString)
#undef SC_SYM
        api.ok = true;
    });
    return api;
}

static int nccl_fail(ncclResult_t r, const char* what) {
    const NcclApi& a = nccl();
    set_error(std::string(what) + ": " + (a.error_string ? a.error_string(r) : "nccl error"));
    return SC_NCCL_ERROR;
}

struct BandPlan {
    int device = 0;
    ncclComm_t comm = nullptr;
    const float* src = nullptr;
    float* dst = nullptr;
    int P = 0, R = 0, C = 0, r = 0, lo = 0, hi = 0, above = -1, below = -1;
    long long sps = 0, dps = 0, srs = 0, drs = 0;
    float taps[MAX_W_LANES] = {};
    int width = 0, flags = 0;
    float *send_top = nullptr, *send_bot = nullptr, *recv_top = nullptr, *recv_bot = nullptr;
    cudaStream_t cs = nullptr;
    cudaEvent_t ev_in = nullptr, ev_x = nullptr;
    cudaGraphExec_t exec = nullptr;
    std::mutex mu;
};

static RowsJob band_job(const BandPlan& b) {
    RowsJob j{};
    j.mode = MODE_FUSED;
    j.src = b.src;
    j.dst = b.dst;
    j.sps = b.sps;
    j.dps = b.dps;
    j.srs = b.srs;
    j.drs = b.drs;
    j.nplanes = b.P;
    j.R = b.R;
    j.C = b.C;
    j.src_row0 = b.lo;
    j.src_rows = b.hi - b.lo;
    j.dst_row0 = b.lo;
    j.hrow_lo = (b.flags & SC_EXTENDED) ? 0 : b.r;
    j.hrow_hi = (b.flags & SC_EXTENDED) ? b.R : b.R - b.r;
    j.flags = b.flags & (SC_EXTENDED | SC_NO_RING);
    j.width = b.width;
    j.taps = b.taps;
    return j;
}

static double host_us() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// The step's operations on stream s (eager, or under capture). SC_BAND_TIMING=1
// prints the host time of each phase (tools/band_host_time.py).
static int issue_step(BandPlan& b, cudaStream_t s) {
    const NcclApi& api = nccl();
    const bool timing = std::getenv("SC_BAND_TIMING") != nullptr;
    double t[5] = {timing ? host_us() : 0.0, 0, 0, 0, 0};
    const bool has_a = b.above >= 0, has_b = b.below >= 0;
    cudaError_t e;
    const size_t n = (size_t)b.P * b.r * b.C;
    if (has_a || has_b) {
        if ((e = cudaEventRecord(b.ev_in, s)) != cudaSuccess || (e = cudaStreamWaitEvent(b.cs, b.ev_in, 0)) != cudaSuccess)
            return fail_cuda(e, "band step: event");
        // both packs in one launch (two 2-D copies cost the host more than a launch)
        if ((e = launch_pack_rows(b.src, b.sps, b.srs, b.P, b.r, b.C, 0, has_a ? b.send_top : nullptr,
                                  b.hi - b.lo - b.r, has_b ? b.send_bot : nullptr, b.cs)) != cudaSuccess)
            return fail_cuda(e, "band step: pack");
        if (timing) t[1] = host_us();
        ncclResult_t nr = api.group_start();
        if (nr == ncclSuccess && has_a) nr = api.send(b.send_top, n, ncclFloat32, b.above, b.comm, b.cs);
        if (nr == ncclSuccess && has_a) nr = api.recv(b.recv_top, n, ncclFloat32, b.above, b.comm, b.cs);
        if (nr == ncclSuccess && has_b) nr = api.send(b.send_bot, n, ncclFloat32, b.below, b.comm, b.cs);
        if (nr == ncclSuccess && has_b) nr = api.recv(b.recv_bot, n, ncclFloat32, b.below, b.comm, b.cs);
        const ncclResult_t ne = api.group_end();
        if (nr != ncclSuccess) return nccl_fail(nr, "band step: send/recv");
        if (ne != ncclSuccess) return nccl_fail(ne, "band step: group");
        if ((e = cudaEventRecord(b.ev_x, b.cs)) != cudaSuccess) return fail_cuda(e, "band step: event");
    }
    if (timing) t[2] = host_us();
    const int ilo = b.lo + (has_a ? b.r : 0), ihi = b.hi - (has_b ? b.r : 0);
    RowsJob j = band_job(b);
    if (ihi > ilo && (has_a || has_b)) {
        // interior rows first: no halo needed, overlapped with the exchange
        j.out_lo = ilo;
        j.out_hi = ihi;
        const int rc = launch_rows(j, s);
        if (rc != SC_OK) return rc;
    }
    if (timing) t[3] = host_us();
    if ((has_a || has_b) && (e = cudaStreamWaitEvent(s, b.ev_x, 0)) != cudaSuccess)
        return fail_cuda(e, "band step: event");
    j = band_job(b);
    if (has_a) {
        j.above = b.recv_top;
        j.above_row0 = b.lo - b.r;
        j.above_rows = b.r;
        j.above_ps = (long long)b.r * b.C;
        j.above_rs = b.C;
    }
    if (has_b) {
        j.below = b.recv_bot;
        j.below_row0 = b.hi;
        j.below_rows = b.r;
        j.below_ps = (long long)b.r * b.C;
        j.below_rs = b.C;
    }
    if (ihi > ilo && (has_a || has_b)) {
        // both boundary strips in ONE launch (either may be empty at the image edges)
        j.out_lo = has_a ? b.lo : ihi;
        j.out_hi = has_a ? ilo : b.hi;
        j.out_lo2 = has_a && has_b ? ihi : 0;
        j.out_hi2 = has_a && has_b ? b.hi : 0;
    } else {
        j.out_lo = b.lo;  // band too short for an interior (or no neighbours): one launch
        j.out_hi = b.hi;
    }
    const int rc = launch_rows(j, s);
    if (timing) {
        t[4] = host_us();
        std::fprintf(stderr, "[sc band step] pack+events %.1f us, nccl group %.1f us, interior launch %.1f us, "
                     "boundary launch %.1f us\n", t[1] - t[0], t[2] - t[1], t[3] - t[2], t[4] - t[3]);
    }
    return rc;
}

}  // namespace sc

using namespace sc;

extern "C" {

int sc_nccl_unique_id(void* id_out) {
    set_error("");
    if (!id_out) return fail_arg("null id buffer");
    const NcclApi& api = nccl();
    if (!api.ok) {
        set_error(api.why);
        return SC_NCCL_ERROR;
    }
    ncclUniqueId id;
    const ncclResult_t r = api.get_unique_id(&id);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id_out, &id, sizeof(id));
    return SC_OK;
}

int sc_nccl_comm_init(const void* id, int nranks, int rank, int device, void** comm_out) {
    set_error("");
    if (!id || !comm_out || nranks < 1 || rank < 0 || rank >= nranks) return fail_arg("bad communicator arguments");
    const NcclApi& api = nccl();
    if (!api.ok) {
        set_error(api.why);
        return SC_NCCL_ERROR;
    }
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return fail_cuda(e, "cudaSetDevice");
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclComm_t comm = nullptr;
    const ncclResult_t r = api.comm_init_rank(&comm, nranks, uid, rank);
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
    *comm_out = comm;
    return SC_OK;
}

int sc_nccl_comm_destroy(void* comm) {
    set_error("");
    if (!comm) return SC_OK;
    const NcclApi& api = nccl();
    if (!api.ok) {
        set_error(api.why);
        return SC_NCCL_ERROR;
    }
    const ncclResult_t r = api.comm_destroy(static_cast<ncclComm_t>(comm));
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommDestroy");
    return SC_OK;
}

int sc_band_plan_destroy(void* plan) {
    set_error("");
    BandPlan* b = static_cast<BandPlan*>(plan);
    if (!b) return SC_OK;
    cudaSetDevice(b->device);
    if (b->cs) cudaStreamSynchronize(b->cs);
    if (b->exec) cudaGraphExecDestroy(b->exec);
    for (float* p : {b->send_top, b->send_bot, b->recv_top, b->recv_bot})
        if (p) cudaFree(p);
    if (b->ev_in) cudaEventDestroy(b->ev_in);
    if (b->ev_x) cudaEventDestroy(b->ev_x);
    if (b->cs) cudaStreamDestroy(b->cs);
    delete b;
    return SC_OK;
}

int sc_band_plan_create(void* comm, const float* src, float* dst, int nplanes, int global_rows, int cols,
                        int64_t src_plane_stride, int64_t dst_plane_stride, int64_t src_row_stride,
                        int64_t dst_row_stride, int band_lo, int band_hi, int rank_above, int rank_below,
                        const float* taps, int width, int flags, int use_graph, void** plan_out) {
    set_error("");
    if (!plan_out || !src || !dst || !taps) return fail_arg("null argument");
    *plan_out = nullptr;
    if (width < 1 || width % 2 == 0) return fail_arg("kernel width must be odd and >= 1");
    if (width > MAX_W_LANES) {
        set_error("NCCL band plans support widths up to 31");
        return SC_UNSUPPORTED_WIDTH;
    }
    if (nplanes < 1 || cols < 1 || global_rows < 1) return fail_arg("dimensions must be positive");
    if (global_rows < width || cols < width) {
        set_error("plane smaller than kernel width");
        return SC_INVALID_DIMENSION;
    }
    const int r = width / 2;
    if (band_lo < 0 || band_hi > global_rows || band_lo >= band_hi) return fail_arg("band rows out of range");
    if ((rank_above >= 0 || rank_below >= 0) && !comm) return fail_arg("a band with neighbours needs a communicator");
    if (rank_above >= 0 && (band_lo < r || band_hi - band_lo < r)) return fail_arg("band above: band too short");
    if (rank_below >= 0 && (band_hi + r > global_rows || band_hi - band_lo < r))
        return fail_arg("band below: band too short");
    if (rank_above < 0 && band_lo != 0) return fail_arg("only the first band may lack a neighbour above");
    if (rank_below < 0 && band_hi != global_rows) return fail_arg("only the last band may lack a neighbour below");
    const int rows = band_hi - band_lo;
    if (src_row_stride < cols || dst_row_stride < cols || (nplanes > 1 && (src_plane_stride < (long long)rows * src_row_stride ||
                                                                          dst_plane_stride < (long long)rows * dst_row_stride)))
        return fail_arg("strides overlap rows or planes");
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, src) != cudaSuccess || a.type != cudaMemoryTypeDevice) {
        cudaGetLastError();
        return fail_arg("band buffers must be device memory");
    }
    BandPlan* b = new BandPlan();
    b->device = a.device;
    cudaSetDevice(b->device);
    b->comm = static_cast<ncclComm_t>(comm);
    b->src = src;
    b->dst = dst;
    b->P = nplanes;
    b->R = global_rows;
    b->C = cols;
    b->r = r;
    b->lo = band_lo;
    b->hi = band_hi;
    b->above = rank_above;
    b->below = rank_below;
    b->sps = src_plane_stride;
    b->dps = dst_plane_stride;
    b->srs = src_row_stride;
    b->drs = dst_row_stride;
    for (int i = 0; i < width; ++i) b->taps[i] = taps[i];
    b->width = width;
    b->flags = flags;
    const size_t n = (size_t)nplanes * r * cols * sizeof(float);
    cudaError_t e = cudaSuccess;
    if (rank_above >= 0 && e == cudaSuccess) e = cudaMalloc(&b->send_top, n);
    if (rank_above >= 0 && e == cudaSuccess) e = cudaMalloc(&b->recv_top, n);
    if (rank_below >= 0 && e == cudaSuccess) e = cudaMalloc(&b->send_bot, n);
    if (rank_below >= 0 && e == cudaSuccess) e = cudaMalloc(&b->recv_bot, n);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&b->cs, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&b->ev_in, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&b->ev_x, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        cudaGetLastError();
        sc_band_plan_destroy(b);
        return fail_cuda(e, "band plan allocation");
    }
    if ((rank_above >= 0 || rank_below >= 0) && !nccl().ok) {
        set_error(nccl().why);
        sc_band_plan_destroy(b);
        return SC_NCCL_ERROR;
    }
    if (use_graph) {
        // capture one step on a private stream; any refusal -> eager steps
        cudaStream_t cap = nullptr;
        cudaGraph_t g = nullptr;
        if (cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamBeginCapture(cap, cudaStreamCaptureModeRelaxed) == cudaSuccess) {
            const int rc = issue_step(*b, cap);
            const cudaError_t ec = cudaStreamEndCapture(cap, &g);
            if (rc == SC_OK && ec == cudaSuccess && g &&
                cudaGraphInstantiateWithFlags(&b->exec, g, 0) != cudaSuccess)
                b->exec = nullptr;
        }
        if (g) cudaGraphDestroy(g);
        if (cap) cudaStreamDestroy(cap);
        cudaGetLastError();
        set_error("");
    }
    *plan_out = b;
    return SC_OK;
}

int sc_band_plan_graphed(void* plan) {
    BandPlan* b = static_cast<BandPlan*>(plan);
    return b && b->exec ? 1 : 0;
}

int sc_band_plan_step(void* plan, void* stream) {
    set_error("");
    BandPlan* b = static_cast<BandPlan*>(plan);
    if (!b) return fail_arg("null plan");
    std::lock_guard<std::mutex> lk(b->mu);
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess || cur != b->device) cudaSetDevice(b->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (b->exec) {
        const cudaError_t e = cudaGraphLaunch(b->exec, s);
        if (e != cudaSuccess) return fail_cuda(e, "band step: graph launch");
        count_launch(((b->above >= 0 || b->below >= 0) && b->hi - b->lo > (b->above >= 0) * b->r + (b->below >= 0) * b->r)
                         ? 2 : 1);
        return SC_OK;
    }
    return issue_step(*b, s);
}

}  // extern "C"
