// stream.cu -- end-to-end two-pass on HOST planes (sc_two_pass_host_f32).
//
// The reference convolves numpy planes in host memory and blocks until done
// (convolve_image, S/executors.py:269-405). This entry point keeps that contract
// for host buffers: each plane is cut into row chunks; chunk k's input rows
// [lo-r, hi+r) go H2D on one stream, the fused kernel runs on a second, and the
// output rows [lo, hi) go D2H on a third, with NSLOT device slots so copy-in,
// compute and copy-out of consecutive chunks overlap (PCIe is full duplex).
// D2H of chunk k is ordered after H2D of chunk k+1, so in-place use
// (dst_planes == src_planes, as conv_two_pass mutates `plane`) never reads a row
// that was already overwritten.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <map>
#include <thread>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/sepconv_b200.h"
#include "kernels.cuh"
#include "launch.h"

namespace sc {

static constexpr int NSLOT = 3;

struct HostCtx {
    int device = -1;
    cudaStream_t h2d = nullptr, cmp = nullptr, d2h = nullptr;
    float* in_buf[NSLOT] = {};
    float* out_buf[NSLOT] = {};
    size_t in_cap = 0, out_cap = 0;  // floats per slot
    cudaEvent_t ev_h2d[NSLOT] = {}, ev_cmp[NSLOT] = {}, ev_d2h[NSLOT] = {};
    std::mutex mu;
};

static HostCtx* host_ctx(int device) {
    static std::mutex mu;
    static std::map<int, std::unique_ptr<HostCtx>> ctxs;
    std::lock_guard<std::mutex> lk(mu);
    auto& c = ctxs[device];
    if (!c) {
        c.reset(new HostCtx());
        c->device = device;
    }
    return c.get();
}

static int ensure(HostCtx* c, size_t in_floats, size_t out_floats, std::string& err) {
    cudaError_t e;
    if (!c->h2d) {
        if ((e = cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking)) != cudaSuccess ||
            (e = cudaStreamCreateWithFlags(&c->cmp, cudaStreamNonBlocking)) != cudaSuccess ||
            (e = cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking)) != cudaSuccess) {
            err = cudaGetErrorString(e);
            return SC_CUDA_ERROR;
        }
        for (int i = 0; i < NSLOT; ++i) {
            cudaEventCreateWithFlags(&c->ev_h2d[i], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&c->ev_cmp[i], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&c->ev_d2h[i], cudaEventDisableTiming);
        }
    }
    if (in_floats > c->in_cap || out_floats > c->out_cap) {
        for (int i = 0; i < NSLOT; ++i) {
            if (c->in_buf[i]) cudaFree(c->in_buf[i]);
            if (c->out_buf[i]) cudaFree(c->out_buf[i]);
            c->in_buf[i] = c->out_buf[i] = nullptr;
        }
        c->in_cap = c->out_cap = 0;
        for (int i = 0; i < NSLOT; ++i) {
            if ((e = cudaMalloc(&c->in_buf[i], in_floats * sizeof(float))) != cudaSuccess ||
                (e = cudaMalloc(&c->out_buf[i], out_floats * sizeof(float))) != cudaSuccess) {
                err = std::string("staging allocation: ") + cudaGetErrorString(e);
                return SC_CUDA_ERROR;
            }
        }
        c->in_cap = in_floats;
        c->out_cap = out_floats;
    }
    return SC_OK;
}

}  // namespace sc

using namespace sc;

// halo_top / halo_bot (optional, per plane): r rows holding global rows
// [out_lo - r, out_lo) / [out_hi, out_hi + r), read instead of the source planes
// (the multi-device path: neighbouring bands overwrite those rows in place)
static int host_band(const float* const* src_planes, float* const* dst_planes, int nplanes, int rows, int cols,
                     int out_lo, int out_hi, const float* taps, int width, int flags, int device,
                     const float* const* halo_top = nullptr, const float* const* halo_bot = nullptr);

extern "C" int sc_two_pass_host_f32(const float* const* src_planes, float* const* dst_planes, int nplanes, int rows,
                                    int cols, const float* taps, int width, int flags, int device) {
    return host_band(src_planes, dst_planes, nplanes, rows, cols, 0, rows, taps, width, flags, device);
}

extern "C" int sc_two_pass_host_band_f32(const float* const* src_planes, float* const* dst_planes, int nplanes,
                                         int rows, int cols, int out_lo, int out_hi, const float* taps, int width,
                                         int flags, int device) {
    set_error("");
    if (out_lo < 0 || out_hi > rows || out_lo >= out_hi) {
        set_error("output rows out of range");
        return SC_INVALID_ARGUMENT;
    }
    return host_band(src_planes, dst_planes, nplanes, rows, cols, out_lo, out_hi, taps, width, flags, device);
}

// One process, several GPUs (the reference's single-process plan model): the
// image is split into ndev row bands by the reference's balanced block split
// (S/executors.py:121-139); every band streams through its own GPU (and PCIe
// link) concurrently, one host thread per device. Before any device starts, the
// 2r rows around every band boundary are copied aside on the host, so that in
// place (dst == src) a band never reads halo rows its neighbour has already
// overwritten. A device listed twice runs its bands one after the other.
extern "C" int sc_two_pass_host_multi_f32(const float* const* src_planes, float* const* dst_planes, int nplanes,
                                          int rows, int cols, const float* taps, int width, int flags,
                                          const int* devices, int ndev) {
    set_error("");
    if (!devices || ndev < 1) {
        set_error("need at least one device");
        return SC_INVALID_ARGUMENT;
    }
    if (!src_planes || !dst_planes || !taps || nplanes < 1 || rows < 1 || cols < 1) {
        set_error("null pointer or non-positive dimension");
        return SC_INVALID_ARGUMENT;
    }
    const int r = width / 2;
    // bands no shorter than r rows, so that a halo comes from the adjacent band only
    int nb = ndev;
    while (nb > 1 && rows / nb < (r > 1 ? r : 1)) --nb;
    if (nb == 1) return host_band(src_planes, dst_planes, nplanes, rows, cols, 0, rows, taps, width, flags, devices[0]);
    std::vector<int> lo(nb + 1);
    const int q = rows / nb, rem = rows % nb;
    for (int g = 0; g <= nb; ++g) lo[g] = g * q + (g < rem ? g : rem);
    // halo copies: boundary g (1..nb-1) keeps rows [lo[g] - r, lo[g] + r) of every plane
    std::vector<float> side((size_t)(nb - 1) * nplanes * 2 * r * cols);
    auto side_rows = [&](int g, int p) { return side.data() + (((size_t)(g - 1) * nplanes + p) * 2 * r) * cols; };
    for (int g = 1; g < nb && r > 0; ++g)
        for (int p = 0; p < nplanes; ++p) {
            if (!src_planes[p]) {
                set_error("null plane pointer");
                return SC_INVALID_ARGUMENT;
            }
            std::memcpy(side_rows(g, p), src_planes[p] + (size_t)(lo[g] - r) * cols, sizeof(float) * 2 * r * cols);
        }
    std::vector<int> rcs(nb, SC_OK);
    std::vector<std::string> errs(nb);
    auto run = [&](int g) {
        std::vector<const float*> top(nplanes), bot(nplanes);
        for (int p = 0; p < nplanes; ++p) {
            top[p] = g > 0 ? side_rows(g, p) : nullptr;                                // rows [lo-r, lo)
            bot[p] = g + 1 < nb ? side_rows(g + 1, p) + (size_t)r * cols : nullptr;  // rows [hi, hi+r)
        }
        rcs[g] = host_band(src_planes, dst_planes, nplanes, rows, cols, lo[g], lo[g + 1], taps, width, flags,
                           devices[g % ndev], g > 0 && r > 0 ? top.data() : nullptr,
                           g + 1 < nb && r > 0 ? bot.data() : nullptr);
        errs[g] = sc_last_error();
    };
    std::vector<std::thread> threads;
    for (int g = 1; g < nb; ++g) threads.emplace_back(run, g);
    run(0);
    for (auto& t : threads) t.join();
    for (int g = 0; g < nb; ++g)
        if (rcs[g] != SC_OK) {
            set_error("band " + std::to_string(g) + ": " + errs[g]);
            return rcs[g];
        }
    set_error("");
    return SC_OK;
}

// Rows [out_lo, out_hi) of a rows x cols image (global-row rules), reading host
// rows [out_lo - r, out_hi + r) clipped to the image and writing host rows
// [out_lo, out_hi); plane pointers address row 0 (the rows outside are not touched).
static int host_band(const float* const* src_planes, float* const* dst_planes, int nplanes, int rows, int cols,
                     int out_lo, int out_hi, const float* taps, int width, int flags, int device,
                     const float* const* halo_top, const float* const* halo_bot) {
    set_error("");
    if (!src_planes || !dst_planes || !taps || nplanes < 1 || rows < 1 || cols < 1) {
        set_error("null pointer or non-positive dimension");
        return SC_INVALID_ARGUMENT;
    }
    if (width < 1 || width % 2 == 0) {
        set_error("kernel width must be odd and >= 1");
        return SC_INVALID_ARGUMENT;
    }
    if (width > MAX_W_WIDE) {
        set_error("kernel width > 255 not supported");
        return SC_UNSUPPORTED_WIDTH;
    }
    if (rows < width || cols < width) {
        set_error("plane smaller than kernel width");
        return SC_INVALID_DIMENSION;
    }
    for (int p = 0; p < nplanes; ++p)
        if (!src_planes[p] || !dst_planes[p]) {
            set_error("null plane pointer");
            return SC_INVALID_ARGUMENT;
        }
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) {
        set_error(std::string("cudaSetDevice: ") + cudaGetErrorString(e));
        return SC_CUDA_ERROR;
    }
    const int r = width / 2;
    HostCtx* c = host_ctx(device);
    std::lock_guard<std::mutex> lk(c->mu);

    // chunk rows: ~1/24 of the image per chunk, clamped to [4, 32] MiB, so that
    // mid-size images still overlap H2D / kernel / D2H over several chunks while
    // large ones keep per-chunk overheads negligible (measured: 2592^2 -16%,
    // 4096^2 -11% vs fixed 32 MiB; tools/e2e_chunks.py). SC_HOST_CHUNK_MB overrides.
    const char* mbs = std::getenv("SC_HOST_CHUNK_MB");
    long long chunk_bytes;
    if (mbs && *mbs) {
        chunk_bytes = (long long)std::atoi(mbs) << 20;
    } else {
        const long long total = (long long)nplanes * (out_hi - out_lo) * cols * 4;
        chunk_bytes = total / 24;
        if (chunk_bytes < (4LL << 20)) chunk_bytes = 4LL << 20;
        if (chunk_bytes > (32LL << 20)) chunk_bytes = 32LL << 20;
    }
    long long ch = chunk_bytes / ((long long)cols * 4);
    if (ch < 16) ch = 16;
    if (ch > out_hi - out_lo) ch = out_hi - out_lo;
    const int chunk = (int)ch;
    std::string err;
    int rc = ensure(c, (size_t)(chunk + 2 * r) * cols, (size_t)chunk * cols, err);
    if (rc != SC_OK) {
        set_error(err);
        return rc;
    }

    struct Chunk {
        int plane, lo, hi, in_lo, in_hi;
    };
    std::vector<Chunk> chunks;
    for (int p = 0; p < nplanes; ++p)
        for (int lo = out_lo; lo < out_hi; lo += chunk) {
            Chunk k;
            k.plane = p;
            k.lo = lo;
            k.hi = lo + chunk < out_hi ? lo + chunk : out_hi;
            k.in_lo = k.lo - r > 0 ? k.lo - r : 0;
            k.in_hi = k.hi + r < rows ? k.hi + r : rows;
            chunks.push_back(k);
        }
    const size_t n = chunks.size();
    const size_t row_bytes = (size_t)cols * sizeof(float);

    auto issue_h2d = [&](size_t k) -> cudaError_t {
        const Chunk& q = chunks[k];
        const int s = (int)(k % NSLOT);
        if (k >= NSLOT) cudaStreamWaitEvent(c->h2d, c->ev_cmp[s], 0);  // slot's previous kernel done
        // rows [in_lo, in_hi): own rows from the source planes, halo rows outside
        // [out_lo, out_hi) from the halo copies when given
        cudaError_t e2 = cudaSuccess;
        int y = q.in_lo;
        float* d = c->in_buf[s];
        if (halo_top && y < out_lo) {
            const int n_top = out_lo - y;
            e2 = cudaMemcpyAsync(d, halo_top[q.plane] + (size_t)(r - n_top) * cols, (size_t)n_top * row_bytes,
                                 cudaMemcpyHostToDevice, c->h2d);
            d += (size_t)n_top * cols;
            y = out_lo;
        }
        const int own_hi = (halo_bot && q.in_hi > out_hi) ? out_hi : q.in_hi;
        if (e2 == cudaSuccess && own_hi > y) {
            e2 = cudaMemcpyAsync(d, src_planes[q.plane] + (size_t)y * cols, (size_t)(own_hi - y) * row_bytes,
                                 cudaMemcpyHostToDevice, c->h2d);
            d += (size_t)(own_hi - y) * cols;
        }
        if (e2 == cudaSuccess && own_hi < q.in_hi)
            e2 = cudaMemcpyAsync(d, halo_bot[q.plane], (size_t)(q.in_hi - own_hi) * row_bytes, cudaMemcpyHostToDevice,
                                 c->h2d);
        cudaEventRecord(c->ev_h2d[s], c->h2d);
        return e2;
    };

    if (n > 0 && (e = issue_h2d(0)) != cudaSuccess) {
        set_error(std::string("H2D: ") + cudaGetErrorString(e));
        return SC_CUDA_ERROR;
    }
    for (size_t k = 0; k < n; ++k) {
        const Chunk& q = chunks[k];
        const int s = (int)(k % NSLOT);
        if (k + 1 < n && (e = issue_h2d(k + 1)) != cudaSuccess) {
            set_error(std::string("H2D: ") + cudaGetErrorString(e));
            return SC_CUDA_ERROR;
        }
        cudaStreamWaitEvent(c->cmp, c->ev_h2d[s], 0);
        if (k >= NSLOT) cudaStreamWaitEvent(c->cmp, c->ev_d2h[s], 0);  // out slot drained
        RowsJob j{};
        j.mode = MODE_FUSED;
        j.src = c->in_buf[s];
        j.dst = c->out_buf[s];
        j.sps = (long long)(q.in_hi - q.in_lo) * cols;
        j.dps = (long long)(q.hi - q.lo) * cols;
        j.srs = cols;
        j.drs = cols;
        j.nplanes = 1;
        j.R = rows;
        j.C = cols;
        j.src_row0 = q.in_lo;
        j.src_rows = q.in_hi - q.in_lo;
        j.dst_row0 = q.lo;
        j.out_lo = q.lo;
        j.out_hi = q.hi;
        j.hrow_lo = (flags & SC_EXTENDED) ? 0 : r;
        j.hrow_hi = (flags & SC_EXTENDED) ? rows : rows - r;
        j.flags = flags & (SC_EXTENDED | SC_NO_RING);
        j.width = width;
        j.taps = taps;
        rc = launch_rows(j, c->cmp);
        if (rc != SC_OK) return rc;
        cudaEventRecord(c->ev_cmp[s], c->cmp);
        cudaStreamWaitEvent(c->d2h, c->ev_cmp[s], 0);
        if (k + 1 < n) cudaStreamWaitEvent(c->d2h, c->ev_h2d[(k + 1) % NSLOT], 0);  // in-place safety
        if (flags & SC_NO_RING) {
            // only valid rows/cols leave the device: the host ring keeps its values
            const int vlo = q.lo > r ? q.lo : r;
            const int vhi = q.hi < rows - r ? q.hi : rows - r;
            if (vhi > vlo)
                e = cudaMemcpy2DAsync(dst_planes[q.plane] + (size_t)vlo * cols + r, row_bytes,
                                      c->out_buf[s] + (size_t)(vlo - q.lo) * cols + r, row_bytes,
                                      (size_t)(cols - 2 * r) * sizeof(float), (size_t)(vhi - vlo),
                                      cudaMemcpyDeviceToHost, c->d2h);
        } else {
            e = cudaMemcpyAsync(dst_planes[q.plane] + (size_t)q.lo * cols, c->out_buf[s],
                                (size_t)(q.hi - q.lo) * row_bytes, cudaMemcpyDeviceToHost, c->d2h);
        }
        if (e != cudaSuccess) {
            set_error(std::string("D2H: ") + cudaGetErrorString(e));
            return SC_CUDA_ERROR;
        }
        cudaEventRecord(c->ev_d2h[s], c->d2h);
    }
    e = cudaStreamSynchronize(c->d2h);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->cmp);
    if (e != cudaSuccess) {
        set_error(std::string("stream sync: ") + cudaGetErrorString(e));
        return SC_CUDA_ERROR;
    }
    return SC_OK;
}
