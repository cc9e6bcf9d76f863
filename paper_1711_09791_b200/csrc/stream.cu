// stream.cu -- end-to-end two-pass on HOST planes (sc_two_pass_host_f32 and
// friends).
//
// The reference convolves numpy planes in host memory and blocks until done
// (convolve_image, S/executors.py:269-405). These entry points keep that
// contract for host buffers: each plane is cut into row chunks; chunk k's input
// rows [lo-r, hi+r) go H2D on one stream, the kernels run on a second, and the
// output rows [lo, hi) go D2H on a third, with NSLOT device slots so copy-in,
// compute and copy-out of consecutive chunks overlap (PCIe is full duplex).
//
// Host memory kinds (decided per plane with cudaPointerGetAttributes):
//  * pinned / registered planes are copied by DMA straight from and into the
//    caller's rows;
//  * pageable planes (plain numpy arrays, the reference's Plane, S/image.py:37-39)
//    go through pinned staging slots: a pool of host threads copies the rows of
//    chunk k+1 into a staging slot while chunk k computes, and copies finished
//    chunks out of their staging slot while later chunks stream -- the CUDA
//    driver's own pageable path would serialise each copy behind a single
//    bounce buffer.
//
// In-place use (dst == src, as conv_two_pass mutates `plane`) is exact: chunks
// are at least r rows tall, so the input rows of chunk k+1 are the only ones
// that overlap the output rows of chunk k; the write-back of chunk k (a DMA into
// pinned rows, or the host copy out of staging) is ordered after chunk k+1's
// input left those rows.
//
// Split mode (sc_two_pass_host_split_f32): the reference's exact end state of
// BOTH buffers of convolve_image(TWO_PASS) with a workspace -- scratch = H0 (the
// zeroed workspace with the row pass on the live rows, S/executors.py:312-323),
// image[valid] = V(H0), image ring untouched. Each chunk also runs the row pass
// with zero fill over its own rows into a scratch slot that is written back to
// the workspace rows.
#include <cuda_runtime.h>

#include <immintrin.h>

#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/sepconv_b200.h"
#include "kernels.cuh"
#include "launch.h"

namespace sc {

static constexpr int NSLOT = 3;

// ---------------------------------------------------------------------------
// Host copy pool: memcpy segments spread over worker threads; the thread that
// waits for a group helps drain it.

struct Seg {
    void* dst;
    const void* src;
    size_t bytes;
};

// Large host copies with non-temporal (streaming) stores: the destination is
// either a pinned staging slot the DMA engine reads next or the caller's rows,
// neither of which the CPU reads back soon, so write-allocating them in cache
// (a read-for-ownership per line: 3 DRAM transfers per byte instead of 2) only
// costs host memory bandwidth -- which the staged path is bound by.
__attribute__((target("avx2"))) static void copy_nt_avx2(char* d, const char* s, size_t n) {
    while (n && (reinterpret_cast<uintptr_t>(d) & 31)) {  // align the destination to 32 B
        *d++ = *s++;
        --n;
    }
    size_t i = 0;
    for (; i + 128 <= n; i += 128) {
        const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i));
        const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 32));
        const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 64));
        const __m256i e = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 96));
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i), a);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 32), b);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 64), c);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 96), e);
    }
    _mm_sfence();
    if (i < n) std::memcpy(d + i, s + i, n - i);
}

static void host_copy(void* d, const void* s, size_t n) {
    static const bool avx2 = __builtin_cpu_supports("avx2") && !std::getenv("SC_HOST_COPY_PLAIN");
    if (avx2 && n >= 4096)
        copy_nt_avx2(static_cast<char*>(d), static_cast<const char*>(s), n);
    else
        std::memcpy(d, s, n);
}

struct CopyGroup {
    std::vector<Seg> segs;
    std::atomic<size_t> next{0};
    std::atomic<size_t> done{0};
};

class CopyPool {
public:
    explicit CopyPool(int n) {
        for (int i = 0; i < n; ++i) threads_.emplace_back([this] { run(); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : threads_) t.join();
    }
    std::shared_ptr<CopyGroup> submit(std::vector<Seg> segs) {
        auto g = std::make_shared<CopyGroup>();
        // split large segments so every worker gets a share
        const size_t piece = 2u << 20;
        for (const Seg& s : segs) {
            for (size_t off = 0; off < s.bytes; off += piece) {
                const size_t n = s.bytes - off < piece ? s.bytes - off : piece;
                g->segs.push_back({static_cast<char*>(s.dst) + off, static_cast<const char*>(s.src) + off, n});
            }
        }
        if (g->segs.empty()) return g;
        {
            std::lock_guard<std::mutex> lk(mu_);
            queue_.push_back(g);
        }
        cv_.notify_all();
        return g;
    }
    void wait(const std::shared_ptr<CopyGroup>& g) {
        if (!g) return;
        const size_t n = g->segs.size();
        for (;;) {  // help
            const size_t i = g->next.fetch_add(1);
            if (i >= n) break;
            host_copy(g->segs[i].dst, g->segs[i].src, g->segs[i].bytes);
            g->done.fetch_add(1);
        }
        while (g->done.load() < n) std::this_thread::yield();
    }

private:
    void run() {
        for (;;) {
            std::shared_ptr<CopyGroup> g;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [this] { return stop_ || !queue_.empty(); });
                if (stop_) return;
                g = queue_.front();
            }
            const size_t n = g->segs.size();
            const size_t i = g->next.fetch_add(1);
            if (i >= n) {
                std::lock_guard<std::mutex> lk(mu_);
                if (!queue_.empty() && queue_.front() == g) queue_.pop_front();
                continue;
            }
            host_copy(g->segs[i].dst, g->segs[i].src, g->segs[i].bytes);
            g->done.fetch_add(1);
        }
    }
    std::vector<std::thread> threads_;
    std::deque<std::shared_ptr<CopyGroup>> queue_;
    std::mutex mu_;
    std::condition_variable cv_;
    bool stop_ = false;
};

static CopyPool& copy_pool() {
    static CopyPool* pool = [] {
        int n = (int)std::thread::hardware_concurrency();
        const char* e = std::getenv("SC_HOST_COPY_THREADS");
        if (e && *e) n = std::atoi(e);
        if (n < 1) n = 1;
        if (n > 32) n = 32;
        return new CopyPool(n - 1 > 0 ? n - 1 : 1);  // the waiting thread is the n-th
    }();
    return *pool;
}

// ---------------------------------------------------------------------------
// Per-device context: streams, device slots, pinned staging slots, events.

struct HostCtx {
    int device = -1;
    cudaStream_t h2d = nullptr, cmp = nullptr, d2h = nullptr;
    float* in_buf[NSLOT] = {};
    float* out_buf[NSLOT] = {};
    float* scr_buf[NSLOT] = {};
    size_t in_cap = 0, out_cap = 0, scr_cap = 0;  // floats per slot
    float* pin_in[NSLOT] = {};
    float* pin_out[NSLOT] = {};
    float* pin_scr[NSLOT] = {};
    size_t pin_in_cap = 0, pin_out_cap = 0, pin_scr_cap = 0;
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

static cudaError_t grow_dev(float* (&bufs)[NSLOT], size_t& cap, size_t need) {
    if (need <= cap) return cudaSuccess;
    for (int i = 0; i < NSLOT; ++i) {
        if (bufs[i]) cudaFree(bufs[i]);
        bufs[i] = nullptr;
    }
    cap = 0;
    for (int i = 0; i < NSLOT; ++i) {
        cudaError_t e = cudaMalloc(&bufs[i], need * sizeof(float));
        if (e != cudaSuccess) return e;
    }
    cap = need;
    return cudaSuccess;
}

static cudaError_t grow_pinned(float* (&bufs)[NSLOT], size_t& cap, size_t need) {
    if (need <= cap) return cudaSuccess;
    for (int i = 0; i < NSLOT; ++i) {
        if (bufs[i]) cudaFreeHost(bufs[i]);
        bufs[i] = nullptr;
    }
    cap = 0;
    for (int i = 0; i < NSLOT; ++i) {
        cudaError_t e = cudaMallocHost(&bufs[i], need * sizeof(float));
        if (e != cudaSuccess) return e;
    }
    cap = need;
    return cudaSuccess;
}

static int ensure_streams(HostCtx* c, std::string& err) {
    if (c->h2d) return SC_OK;
    cudaError_t e;
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
    return SC_OK;
}

// pageable host memory (not pinned, not registered, not device)?
static bool pageable(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

// DMA between device memory and the caller's (pinned or registered) host rows.
// Measured on the B200 box (tools/dma_align_probe.py): with H2D and D2H running
// at once, a transfer whose HOST address is not 256-B aligned runs at 41-44 GB/s
// each way instead of 49-50 (numpy's large arrays start 16 bytes into a page);
// the device address does not matter. So a large copy is issued as a head up to
// the next 256-B host boundary plus an aligned body: 48.9 GB/s.
static cudaError_t dma_copy(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, cudaStream_t s) {
    const void* host = kind == cudaMemcpyHostToDevice ? src : dst;
    const size_t head = (256 - (reinterpret_cast<uintptr_t>(host) & 255)) & 255;
    if (head == 0 || bytes < head + (64u << 10)) return cudaMemcpyAsync(dst, src, bytes, kind, s);
    cudaError_t e = cudaMemcpyAsync(dst, src, head, kind, s);
    if (e != cudaSuccess) return e;
    return cudaMemcpyAsync(static_cast<char*>(dst) + head, static_cast<const char*>(src) + head, bytes - head, kind, s);
}

struct HostJob {
    const float* const* src;
    float* const* dst;
    float* const* scr;  // split mode: workspace planes (H0), else null
    int nplanes, rows, cols, out_lo, out_hi;
    const float* taps;
    int width, flags, device;
    const float* const* halo_top;  // optional: r rows holding global rows [out_lo - r, out_lo)
    const float* const* halo_bot;  // optional: r rows holding global rows [out_hi, out_hi + r)
    // single pass (sc_single_pass_host_f32): the dense width x width matrix; dst =
    // the workspace planes (valid region only); dst2 = the image planes when the
    // valid region is also copied back (S/executors.py:330-331), else null
    const float* dense = nullptr;
    float* const* dst2 = nullptr;
    // row pass (1) or column pass (2) alone (sc_pass_host_f32): dst[valid] only
    int one_pass = 0;
};

static int validate(const HostJob& j) {
    if (!j.src || !j.dst || (!j.taps && !j.dense) || j.nplanes < 1 || j.rows < 1 || j.cols < 1) {
        set_error("null pointer or non-positive dimension");
        return SC_INVALID_ARGUMENT;
    }
    if (j.width < 1 || j.width % 2 == 0) {
        set_error("kernel width must be odd and >= 1");
        return SC_INVALID_ARGUMENT;
    }
    if (j.width > MAX_W_WIDE) {
        set_error("kernel width > 255 not supported");
        return SC_UNSUPPORTED_WIDTH;
    }
    if (j.rows < j.width || j.cols < j.width) {
        set_error("plane smaller than kernel width");
        return SC_INVALID_DIMENSION;
    }
    for (int p = 0; p < j.nplanes; ++p)
        if (!j.src[p] || !j.dst[p] || (j.scr && !j.scr[p]) || (j.dst2 && !j.dst2[p])) {
            set_error("null plane pointer");
            return SC_INVALID_ARGUMENT;
        }
    if (j.dense || j.one_pass) {
        // the workspace must not alias the image (S/conv.py:68-75 _check_pair)
        const size_t bytes = (size_t)j.rows * j.cols * sizeof(float);
        for (int a = 0; a < j.nplanes; ++a)
            for (int b = 0; b < j.nplanes; ++b) {
                const char* x = reinterpret_cast<const char*>(j.dst[a]);
                const char* z = reinterpret_cast<const char*>(j.src[b]);
                if (x < z + bytes && z < x + bytes) {
                    set_error("workspace planes must not overlap the image");
                    return SC_INVALID_ARGUMENT;
                }
            }
    }
    if (j.scr) {
        // the workspace must not alias the image (S/conv.py:68-75 _check_pair)
        const size_t bytes = (size_t)j.rows * j.cols * sizeof(float);
        for (int a = 0; a < j.nplanes; ++a)
            for (int b = 0; b < j.nplanes; ++b) {
                const char* x = reinterpret_cast<const char*>(j.scr[a]);
                const char* y = reinterpret_cast<const char*>(j.dst[b]);
                const char* z = reinterpret_cast<const char*>(j.src[b]);
                if ((x < y + bytes && y < x + bytes) || (x < z + bytes && z < x + bytes)) {
                    set_error("workspace planes must not overlap the image");
                    return SC_INVALID_ARGUMENT;
                }
            }
    }
    return SC_OK;
}

// Rows [out_lo, out_hi) of a rows x cols image (global-row rules), reading host
// rows [out_lo - r, out_hi + r) clipped to the image and writing host rows
// [out_lo, out_hi) (and the same rows of the workspace in split mode); plane
// pointers address row 0, rows outside are not touched.
static int host_band(const HostJob& J) {
    set_error("");
    int rc = validate(J);
    if (rc != SC_OK) return rc;
    cudaError_t e = cudaSetDevice(J.device);
    if (e != cudaSuccess) {
        set_error(std::string("cudaSetDevice: ") + cudaGetErrorString(e));
        return SC_CUDA_ERROR;
    }
    const int r = J.width / 2, rows = J.rows, cols = J.cols;
    HostCtx* c = host_ctx(J.device);
    std::lock_guard<std::mutex> lk(c->mu);
    std::string err;
    if ((rc = ensure_streams(c, err)) != SC_OK) {
        set_error(err);
        return rc;
    }

    // chunk rows: ~1/24 of the band per chunk, clamped to [4, 32] MiB, so that
    // mid-size images still overlap H2D / kernel / D2H over several chunks while
    // large ones keep per-chunk overheads negligible (measured: 2592^2 -16%,
    // 4096^2 -11% vs fixed 32 MiB; tools/e2e_chunks.py). SC_HOST_CHUNK_MB
    // overrides. Never fewer than max(16, r) rows: in place, chunk k+1's input
    // must be the only one overlapping chunk k's output rows.
    const char* mbs = std::getenv("SC_HOST_CHUNK_MB");
    long long chunk_bytes;
    if (mbs && *mbs) {
        chunk_bytes = (long long)std::atoi(mbs) << 20;
    } else {
        const long long total = (long long)J.nplanes * (J.out_hi - J.out_lo) * cols * 4;
        chunk_bytes = total / 24;
        if (chunk_bytes < (4LL << 20)) chunk_bytes = 4LL << 20;
        if (chunk_bytes > (32LL << 20)) chunk_bytes = 32LL << 20;
    }
    long long ch = chunk_bytes / ((long long)cols * 4);
    if (ch < 16) ch = 16;
    if (ch < r) ch = r;
    if (ch > J.out_hi - J.out_lo) ch = J.out_hi - J.out_lo;
    const int chunk = (int)ch;
    const bool split = J.scr != nullptr;

    // memory kinds: stage pageable planes through pinned slots
    std::vector<char> stage_src(J.nplanes), stage_dst(J.nplanes), stage_scr(J.nplanes), stage_dst2(J.nplanes);
    bool any_in = false, any_out = false;
    for (int p = 0; p < J.nplanes; ++p) {
        // (the multi-device halo copies are small host vectors: their rows go by a
        // plain pageable cudaMemcpyAsync, the band's own rows by DMA when they can)
        stage_src[p] = pageable(J.src[p]);
        stage_dst[p] = pageable(J.dst[p]);
        stage_scr[p] = split && pageable(J.scr[p]);
        stage_dst2[p] = J.dst2 && pageable(J.dst2[p]);
        any_in |= stage_src[p] != 0;
        any_out |= stage_dst[p] || stage_scr[p] || stage_dst2[p];
    }
    const size_t in_f = (size_t)(chunk + 2 * r) * cols, out_f = (size_t)chunk * cols;
    if ((e = grow_dev(c->in_buf, c->in_cap, in_f)) != cudaSuccess ||
        (e = grow_dev(c->out_buf, c->out_cap, out_f)) != cudaSuccess ||
        (split && (e = grow_dev(c->scr_buf, c->scr_cap, out_f)) != cudaSuccess) ||
        (any_in && (e = grow_pinned(c->pin_in, c->pin_in_cap, in_f)) != cudaSuccess) ||
        (any_out && (e = grow_pinned(c->pin_out, c->pin_out_cap, out_f)) != cudaSuccess) ||
        (any_out && split && (e = grow_pinned(c->pin_scr, c->pin_scr_cap, out_f)) != cudaSuccess)) {
        cudaGetLastError();
        set_error(std::string("staging allocation: ") + cudaGetErrorString(e));
        return SC_CUDA_ERROR;
    }

    struct Chunk {
        int plane, lo, hi, in_lo, in_hi;
    };
    std::vector<Chunk> chunks;
    for (int p = 0; p < J.nplanes; ++p)
        for (int lo = J.out_lo; lo < J.out_hi; lo += chunk) {
            Chunk k;
            k.plane = p;
            k.lo = lo;
            k.hi = lo + chunk < J.out_hi ? lo + chunk : J.out_hi;
            k.in_lo = k.lo - r > 0 ? k.lo - r : 0;
            k.in_hi = k.hi + r < rows ? k.hi + r : rows;
            chunks.push_back(k);
        }
    const size_t n = chunks.size();
    const size_t row_bytes = (size_t)cols * sizeof(float);
    // the single pass writes the valid region only: nothing else leaves the device
    const bool no_ring = (J.flags & SC_NO_RING) != 0 || J.dense != nullptr || J.one_pass != 0;
    CopyPool& pool = copy_pool();
    std::vector<std::shared_ptr<CopyGroup>> in_grp(n), out_grp(n);

    // host segments of chunk k's input rows [in_lo, in_hi), in order: own rows
    // from the source plane, halo rows outside [out_lo, out_hi) from the halo
    // copies when given; `base` = where row in_lo lands
    auto in_segments = [&](size_t k, float* base, std::vector<Seg>& segs) {
        const Chunk& q = chunks[k];
        int y = q.in_lo;
        float* d = base;
        if (J.halo_top && y < J.out_lo) {
            const int n_top = J.out_lo - y;
            segs.push_back({d, J.halo_top[q.plane] + (size_t)(r - n_top) * cols, (size_t)n_top * row_bytes});
            d += (size_t)n_top * cols;
            y = J.out_lo;
        }
        const int own_hi = (J.halo_bot && q.in_hi > J.out_hi) ? J.out_hi : q.in_hi;
        if (own_hi > y) {
            segs.push_back({d, J.src[q.plane] + (size_t)y * cols, (size_t)(own_hi - y) * row_bytes});
            d += (size_t)(own_hi - y) * cols;
        }
        if (own_hi < q.in_hi) segs.push_back({d, J.halo_bot[q.plane], (size_t)(q.in_hi - own_hi) * row_bytes});
    };
    // stage chunk k's input into its pinned slot (asynchronously, on the pool)
    auto stage_in = [&](size_t k) -> cudaError_t {
        const Chunk& q = chunks[k];
        if (!stage_src[q.plane]) return cudaSuccess;
        const int s = (int)(k % NSLOT);
        // the slot's previous H2D (chunk k - NSLOT) must have left it
        if (k >= NSLOT) {
            cudaError_t e2 = cudaEventSynchronize(c->ev_h2d[s]);
            if (e2 != cudaSuccess) return e2;
        }
        std::vector<Seg> segs;
        in_segments(k, c->pin_in[s], segs);
        in_grp[k] = pool.submit(std::move(segs));
        return cudaSuccess;
    };
    auto issue_h2d = [&](size_t k) -> cudaError_t {
        const Chunk& q = chunks[k];
        const int s = (int)(k % NSLOT);
        if (k >= NSLOT) cudaStreamWaitEvent(c->h2d, c->ev_cmp[s], 0);  // slot's previous kernel done
        cudaError_t e2 = cudaSuccess;
        if (stage_src[q.plane]) {
            pool.wait(in_grp[k]);
            in_grp[k].reset();
            e2 = cudaMemcpyAsync(c->in_buf[s], c->pin_in[s], (size_t)(q.in_hi - q.in_lo) * row_bytes,
                                 cudaMemcpyHostToDevice, c->h2d);
        } else {
            std::vector<Seg> segs;
            in_segments(k, c->in_buf[s], segs);
            for (const Seg& g : segs) {
                if (e2 != cudaSuccess) break;
                e2 = dma_copy(g.dst, g.src, g.bytes, cudaMemcpyHostToDevice, c->h2d);
            }
        }
        cudaEventRecord(c->ev_h2d[s], c->h2d);
        return e2;
    };
    // host copy of chunk k out of its pinned slots into the caller's rows
    auto copy_out = [&](size_t k) -> cudaError_t {
        const Chunk& q = chunks[k];
        if (!stage_dst[q.plane] && !stage_scr[q.plane] && !stage_dst2[q.plane]) return cudaSuccess;
        const int s = (int)(k % NSLOT);
        cudaError_t e2 = cudaEventSynchronize(c->ev_d2h[s]);
        if (e2 != cudaSuccess) return e2;
        std::vector<Seg> segs;
        auto from_pinned = [&](float* plane) {
            if (no_ring) {
                const int vlo = q.lo > r ? q.lo : r;
                const int vhi = q.hi < rows - r ? q.hi : rows - r;
                for (int y = vlo; y < vhi; ++y)
                    segs.push_back({plane + (size_t)y * cols + r, c->pin_out[s] + (size_t)(y - q.lo) * cols + r,
                                    (size_t)(cols - 2 * r) * sizeof(float)});
            } else {
                segs.push_back({plane + (size_t)q.lo * cols, c->pin_out[s], (size_t)(q.hi - q.lo) * row_bytes});
            }
        };
        if (stage_dst[q.plane]) from_pinned(J.dst[q.plane]);
        if (stage_dst2[q.plane]) from_pinned(J.dst2[q.plane]);
        if (stage_scr[q.plane])
            segs.push_back({J.scr[q.plane] + (size_t)q.lo * cols, c->pin_scr[s], (size_t)(q.hi - q.lo) * row_bytes});
        out_grp[k] = pool.submit(std::move(segs));
        return cudaSuccess;
    };

    // On an error after the first enqueue: let every queued copy, kernel and host
    // copy finish before returning, so nothing touches the caller's buffers later.
    auto drain = [&](int code, const std::string& msg) {
        cudaStreamSynchronize(c->h2d);
        cudaStreamSynchronize(c->cmp);
        cudaStreamSynchronize(c->d2h);
        for (auto& g : in_grp) pool.wait(g);
        for (auto& g : out_grp) pool.wait(g);
        cudaGetLastError();
        set_error(msg);
        return code;
    };

    if (n > 0) {
        if ((e = stage_in(0)) != cudaSuccess || (e = issue_h2d(0)) != cudaSuccess)
            return drain(SC_CUDA_ERROR, std::string("H2D: ") + cudaGetErrorString(e));
    }
    for (size_t k = 0; k < n; ++k) {
        const Chunk& q = chunks[k];
        const int s = (int)(k % NSLOT);
        if (k + 1 < n && (e = stage_in(k + 1)) != cudaSuccess)
            return drain(SC_CUDA_ERROR, std::string("staging: ") + cudaGetErrorString(e));
        cudaStreamWaitEvent(c->cmp, c->ev_h2d[s], 0);
        if (k >= NSLOT) cudaStreamWaitEvent(c->cmp, c->ev_d2h[s], 0);  // out slots drained
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
        j.hrow_lo = (J.flags & SC_EXTENDED) ? 0 : r;
        j.hrow_hi = (J.flags & SC_EXTENDED) ? rows : rows - r;
        j.flags = J.flags & (SC_EXTENDED | SC_NO_RING);
        j.width = J.width;
        j.taps = J.taps;
        if (J.dense) {
            static const float zeros[MAX_W_WIDE] = {0};
            j.mode = MODE_SINGLE;
            j.dense = J.dense;
            j.taps = zeros;
            j.flags = 0;
            j.out_lo = q.lo > r ? q.lo : r;  // the valid rows of this chunk
            j.out_hi = q.hi < rows - r ? q.hi : rows - r;
        }
        if (J.one_pass) {
            j.mode = J.one_pass == 1 ? MODE_HPASS : MODE_VPASS;
            j.flags = 0;
            j.hrow_lo = r;
            j.hrow_hi = rows - r;
            j.out_lo = q.lo > r ? q.lo : r;  // the valid rows of this chunk
            j.out_hi = q.hi < rows - r ? q.hi : rows - r;
        }
        rc = ((J.dense || J.one_pass) && j.out_hi <= j.out_lo) ? SC_OK : launch_rows(j, c->cmp);
        if (rc == SC_OK && split) {
            // H0 of the chunk's own rows: the zeroed workspace with the row pass on
            // the live rows (zero on dead rows and on the column ring)
            RowsJob h = j;
            h.mode = MODE_HPASS;
            h.dst = c->scr_buf[s];
            h.flags = SC_ZERO_FILL;
            rc = launch_rows(h, c->cmp);
        }
        if (rc != SC_OK) {
            const std::string msg = sc_last_error();
            return drain(rc, msg);
        }
        cudaEventRecord(c->ev_cmp[s], c->cmp);
        // the next chunk's input goes up while this one computes (enqueued before
        // this chunk's write-back, which waits for it)
        if (k + 1 < n && (e = issue_h2d(k + 1)) != cudaSuccess)
            return drain(SC_CUDA_ERROR, std::string("H2D: ") + cudaGetErrorString(e));
        cudaStreamWaitEvent(c->d2h, c->ev_cmp[s], 0);
        // in-place safety of DMA write-backs: chunk k+1's input has left the host rows
        if (k + 1 < n) cudaStreamWaitEvent(c->d2h, c->ev_h2d[(k + 1) % NSLOT], 0);
        // the slot's previous host copy-out (chunk k - NSLOT) must be done
        if (k >= NSLOT) {
            pool.wait(out_grp[k - NSLOT]);
            out_grp[k - NSLOT].reset();
        }
        e = cudaSuccess;
        // only valid rows/cols leave the device under no_ring: the host ring keeps its values
        auto valid_region_d2h = [&](float* plane) -> cudaError_t {
            const int vlo = q.lo > r ? q.lo : r;
            const int vhi = q.hi < rows - r ? q.hi : rows - r;
            if (vhi <= vlo) return cudaSuccess;
            return cudaMemcpy2DAsync(plane + (size_t)vlo * cols + r, row_bytes,
                                     c->out_buf[s] + (size_t)(vlo - q.lo) * cols + r, row_bytes,
                                     (size_t)(cols - 2 * r) * sizeof(float), (size_t)(vhi - vlo),
                                     cudaMemcpyDeviceToHost, c->d2h);
        };
        if (stage_dst[q.plane] || stage_dst2[q.plane])
            e = cudaMemcpyAsync(c->pin_out[s], c->out_buf[s], (size_t)(q.hi - q.lo) * row_bytes,
                                cudaMemcpyDeviceToHost, c->d2h);
        if (e == cudaSuccess && !stage_dst[q.plane]) {
            if (no_ring)
                e = valid_region_d2h(J.dst[q.plane]);
            else
                e = dma_copy(J.dst[q.plane] + (size_t)q.lo * cols, c->out_buf[s], (size_t)(q.hi - q.lo) * row_bytes,
                             cudaMemcpyDeviceToHost, c->d2h);
        }
        if (e == cudaSuccess && J.dst2 && !stage_dst2[q.plane]) e = valid_region_d2h(J.dst2[q.plane]);
        if (e == cudaSuccess && split)
            e = dma_copy(stage_scr[q.plane] ? c->pin_scr[s] : J.scr[q.plane] + (size_t)q.lo * cols, c->scr_buf[s],
                         (size_t)(q.hi - q.lo) * row_bytes, cudaMemcpyDeviceToHost, c->d2h);
        if (e != cudaSuccess) return drain(SC_CUDA_ERROR, std::string("D2H: ") + cudaGetErrorString(e));
        cudaEventRecord(c->ev_d2h[s], c->d2h);
        // write back the previous chunk (its D2H had a whole chunk's time)
        if (k >= 1 && (e = copy_out(k - 1)) != cudaSuccess)
            return drain(SC_CUDA_ERROR, std::string("write-back: ") + cudaGetErrorString(e));
    }
    if (n > 0 && (e = copy_out(n - 1)) != cudaSuccess)
        return drain(SC_CUDA_ERROR, std::string("write-back: ") + cudaGetErrorString(e));
    for (auto& g : out_grp) pool.wait(g);
    e = cudaStreamSynchronize(c->d2h);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->cmp);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->h2d);
    if (e != cudaSuccess) return drain(SC_CUDA_ERROR, std::string("stream sync: ") + cudaGetErrorString(e));
    return SC_OK;
}

}  // namespace sc

using namespace sc;

// Page-locking of caller host buffers (cached by the Python layer for the
// lifetime of the array): registered planes take the direct-DMA path above.
extern "C" int sc_host_register(void* ptr, int64_t bytes) {
    set_error("");
    if (!ptr || bytes <= 0) {
        set_error("null pointer or empty range");
        return SC_INVALID_ARGUMENT;
    }
    cudaError_t e = cudaHostRegister(ptr, (size_t)bytes, cudaHostRegisterPortable);
    if (e != cudaSuccess) {
        cudaGetLastError();
        set_error(std::string("cudaHostRegister: ") + cudaGetErrorString(e));
        return SC_CUDA_ERROR;
    }
    return SC_OK;
}

extern "C" int sc_host_unregister(void* ptr) {
    set_error("");
    if (!ptr) return SC_OK;
    cudaError_t e = cudaHostUnregister(ptr);
    if (e != cudaSuccess) {
        cudaGetLastError();
        set_error(std::string("cudaHostUnregister: ") + cudaGetErrorString(e));
        return SC_CUDA_ERROR;
    }
    return SC_OK;
}

extern "C" int sc_two_pass_host_f32(const float* const* src_planes, float* const* dst_planes, int nplanes, int rows,
                                    int cols, const float* taps, int width, int flags, int device) {
    HostJob j{src_planes, dst_planes, nullptr, nplanes, rows, cols, 0, rows, taps, width, flags, device, nullptr, nullptr};
    return host_band(j);
}

// Single pass over HOST planes (convolve_image's single-pass variants on numpy
// planes, S/executors.py:327-356): workspace[valid] = dense fold of the image;
// with SC_COPY_BACK the same samples also go back into image[valid] (in place:
// a chunk's write-back is ordered after the next chunk's input left its rows).
// Everything else in both buffers keeps its values.
extern "C" int sc_single_pass_host_f32(float* const* image_planes, float* const* workspace_planes, int nplanes,
                                       int rows, int cols, const float* dense, int width, int flags, int device) {
    set_error("");
    if (!workspace_planes || !dense) {
        set_error("null workspace planes or matrix");
        return SC_INVALID_ARGUMENT;
    }
    HostJob j{image_planes, workspace_planes, nullptr, nplanes, rows, cols, 0, rows, nullptr, width, 0, device,
              nullptr, nullptr};
    j.dense = dense;
    j.dst2 = (flags & SC_COPY_BACK) ? image_planes : nullptr;
    return host_band(j);
}

// horizontal_pass / vertical_pass on HOST planes (S/conv.py:362-389): dst[valid]
// := the row pass (vertical = 0) or the column pass (vertical != 0) of src over the
// valid rows [r, R-r) and columns [r, C-r); dst elsewhere keeps its values.
extern "C" int sc_pass_host_f32(const float* const* src_planes, float* const* dst_planes, int nplanes, int rows,
                                int cols, const float* taps, int width, int vertical, int device) {
    set_error("");
    HostJob j{src_planes, dst_planes, nullptr, nplanes, rows, cols, 0, rows, taps, width, 0, device, nullptr, nullptr};
    j.one_pass = vertical ? 2 : 1;
    return host_band(j);
}

extern "C" int sc_two_pass_host_split_f32(float* const* image_planes, float* const* scratch_planes, int nplanes,
                                          int rows, int cols, const float* taps, int width, int flags, int device) {
    set_error("");
    if (!scratch_planes) {
        set_error("null workspace planes");
        return SC_INVALID_ARGUMENT;
    }
    // the image ring is never written (the reference's column pass writes the
    // valid region only, S/conv.py:293)
    HostJob j{image_planes, image_planes, scratch_planes, nplanes, rows, cols, 0, rows, taps,
              width, (flags & SC_EXTENDED) | SC_NO_RING, device, nullptr, nullptr};
    return host_band(j);
}

extern "C" int sc_two_pass_host_band_f32(const float* const* src_planes, float* const* dst_planes, int nplanes,
                                         int rows, int cols, int out_lo, int out_hi, const float* taps, int width,
                                         int flags, int device) {
    set_error("");
    if (out_lo < 0 || out_hi > rows || out_lo >= out_hi) {
        set_error("output rows out of range");
        return SC_INVALID_ARGUMENT;
    }
    HostJob j{src_planes, dst_planes, nullptr, nplanes, rows, cols, out_lo, out_hi, taps, width, flags, device,
              nullptr, nullptr};
    return host_band(j);
}

// One process, several GPUs (the reference's single-process plan model): the
// image is split into ndev row bands by the reference's balanced block split
// (S/executors.py:121-139); every band streams through its own GPU (and PCIe
// link) concurrently, one host thread per device. Before any device starts, the
// 2r rows around every band boundary are copied aside on the host, so that in
// place (dst == src) a band never reads halo rows its neighbour has already
// overwritten. A device listed twice runs its bands one after the other.
static int host_multi(const float* const* src_planes, float* const* dst_planes, float* const* scr_planes,
                      int nplanes, int rows, int cols, const float* taps, int width, int flags, const int* devices,
                      int ndev, const float* dense = nullptr, float* const* dst2 = nullptr) {
    set_error("");
    if (!devices || ndev < 1) {
        set_error("need at least one device");
        return SC_INVALID_ARGUMENT;
    }
    if (!src_planes || !dst_planes || (!taps && !dense) || nplanes < 1 || rows < 1 || cols < 1) {
        set_error("null pointer or non-positive dimension");
        return SC_INVALID_ARGUMENT;
    }
    const int r = width / 2;
    // bands no shorter than r rows, so that a halo comes from the adjacent band only
    int nb = ndev;
    while (nb > 1 && rows / nb < (r > 1 ? r : 1)) --nb;
    if (nb == 1) {
        HostJob j{src_planes, dst_planes, scr_planes, nplanes, rows, cols, 0, rows, taps, width, flags, devices[0],
                  nullptr, nullptr};
        j.dense = dense;
        j.dst2 = dst2;
        return host_band(j);
    }
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
        HostJob j{src_planes, dst_planes, scr_planes, nplanes, rows, cols, lo[g], lo[g + 1], taps, width, flags,
                  devices[g % ndev], g > 0 && r > 0 ? top.data() : nullptr,
                  g + 1 < nb && r > 0 ? bot.data() : nullptr};
        j.dense = dense;
        j.dst2 = dst2;
        rcs[g] = host_band(j);
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

// sc_single_pass_host_f32 over several GPUs from one process (row bands, as
// sc_two_pass_host_multi_f32: the rows around every band boundary are copied aside
// first, so copy-back in place never reads rows a neighbouring band has rewritten).
extern "C" int sc_single_pass_host_multi_f32(float* const* image_planes, float* const* workspace_planes, int nplanes,
                                             int rows, int cols, const float* dense, int width, int flags,
                                             const int* devices, int ndev) {
    if (!workspace_planes || !dense) {
        set_error("null workspace planes or matrix");
        return SC_INVALID_ARGUMENT;
    }
    return host_multi(image_planes, workspace_planes, nullptr, nplanes, rows, cols, nullptr, width, 0, devices, ndev,
                      dense, (flags & SC_COPY_BACK) ? image_planes : nullptr);
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
    return host_multi(src_planes, dst_planes, nullptr, nplanes, rows, cols, taps, width, flags, devices, ndev);
}

// The same with the reference's workspace end state (sc_two_pass_host_split_f32
// per band: the image ring untouched, H0 into the workspace rows of each band).
extern "C" int sc_two_pass_host_multi_split_f32(float* const* image_planes, float* const* scratch_planes,
                                                int nplanes, int rows, int cols, const float* taps, int width,
                                                int flags, const int* devices, int ndev) {
    if (!scratch_planes) {
        set_error("null workspace planes");
        return SC_INVALID_ARGUMENT;
    }
    return host_multi(image_planes, image_planes, scratch_planes, nplanes, rows, cols, taps, width,
                      (flags & SC_EXTENDED) | SC_NO_RING, devices, ndev);
}
