// host_mem_probe.cu -- host-side memory numbers that decide the end-to-end path
// for pageable planes: multi-threaded host memcpy bandwidth, pinned H2D/D2H
// rates (alone and together), the driver's pageable copy rate, and the cost of
// cudaHostRegister. Build: nvcc -O2 -std=c++17 tools/host_mem_probe.cu -o tools/_host_mem_probe
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static double par_copy(char* dst, const char* src, size_t bytes, int nt) {
    const double t0 = now();
    std::vector<std::thread> th;
    for (int i = 0; i < nt; ++i)
        th.emplace_back([=] {
            const size_t lo = bytes * i / nt, hi = bytes * (i + 1) / nt;
            std::memcpy(dst + lo, src + lo, hi - lo);
        });
    for (auto& t : th) t.join();
    return bytes / (now() - t0) / 1e9;
}

int main() {
    const size_t GB = 1ull << 30;
    const size_t N = 2 * GB;
    char* a = (char*)std::malloc(N);
    char* b = (char*)std::malloc(N);
    std::memset(a, 1, N);
    std::memset(b, 2, N);
    const int hw = (int)std::thread::hardware_concurrency();
    std::printf("hardware_concurrency %d\n", hw);
    for (int nt : {1, 2, 4, 8, 16, 24, 32, 48, 64}) {
        if (nt > hw) break;
        double best = 0;
        for (int rep = 0; rep < 3; ++rep) {
            double g = par_copy(b, a, N, nt);
            if (g > best) best = g;
        }
        std::printf("host memcpy %2d threads: %.1f GB/s\n", nt, best);
    }
    cudaSetDevice(0);
    cudaFree(0);
    const size_t M = 1 * GB;
    char *d1, *d2, *h1, *h2;
    cudaMalloc(&d1, M);
    cudaMalloc(&d2, M);
    cudaMallocHost(&h1, M);
    cudaMallocHost(&h2, M);
    std::memset(h1, 3, M);
    std::memset(h2, 4, M);
    cudaStream_t s1, s2;
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    auto timeit = [&](auto fn) {
        fn();
        cudaDeviceSynchronize();
        const double t0 = now();
        fn();
        cudaDeviceSynchronize();
        return now() - t0;
    };
    double t = timeit([&] { cudaMemcpyAsync(d1, h1, M, cudaMemcpyHostToDevice, s1); });
    std::printf("pinned H2D alone: %.1f GB/s\n", M / t / 1e9);
    t = timeit([&] { cudaMemcpyAsync(h2, d2, M, cudaMemcpyDeviceToHost, s2); });
    std::printf("pinned D2H alone: %.1f GB/s\n", M / t / 1e9);
    t = timeit([&] {
        cudaMemcpyAsync(d1, h1, M, cudaMemcpyHostToDevice, s1);
        cudaMemcpyAsync(h2, d2, M, cudaMemcpyDeviceToHost, s2);
    });
    std::printf("pinned H2D+D2H together: %.1f GB/s each way\n", M / t / 1e9);
    t = timeit([&] { cudaMemcpy(d1, a, M, cudaMemcpyHostToDevice); });
    std::printf("pageable H2D (driver): %.1f GB/s\n", M / t / 1e9);
    t = timeit([&] { cudaMemcpy(b, d2, M, cudaMemcpyDeviceToHost); });
    std::printf("pageable D2H (driver): %.1f GB/s\n", M / t / 1e9);
    // cudaHostRegister of already-faulted pageable memory
    for (size_t sz : {64ull << 20, 256ull << 20, 1ull << 30}) {
        double t0 = now();
        cudaError_t e = cudaHostRegister(a, sz, cudaHostRegisterDefault);
        double tr = now() - t0;
        t0 = now();
        cudaHostUnregister(a);
        double tu = now() - t0;
        std::printf("cudaHostRegister %4zu MB: %.2f ms (%.1f GB/s) [%s], unregister %.2f ms\n", sz >> 20, tr * 1e3,
                    sz / tr / 1e9, cudaGetErrorString(e), tu * 1e3);
    }
    // staged pipeline estimate: threads copy pageable -> pinned while DMA runs
    for (int nt : {4, 8, 16}) {
        if (nt > hw) break;
        const size_t chunk = 32ull << 20;
        const double t0 = now();
        for (size_t off = 0; off + chunk <= M; off += chunk) {
            par_copy(h1 + (off % (256ull << 20)), a + off, chunk, nt);
            cudaMemcpyAsync(d1 + off, h1 + (off % (256ull << 20)), chunk, cudaMemcpyHostToDevice, s1);
        }
        cudaStreamSynchronize(s1);
        std::printf("naive staged H2D (%d threads, no overlap bookkeeping): %.1f GB/s\n", nt, M / (now() - t0) / 1e9);
    }
    return 0;
}
