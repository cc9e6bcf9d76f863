// tma1d_probe.cu -- semantics of a rank-1 TMA tensor map over a float buffer
// (dev probe): copies of a 176-float box from arbitrary element coordinates
// (unaligned, negative, past the end) into shared memory at several 16-B / 128-B
// offsets, and a tensor store back to an arbitrary coordinate. Prints PASS/FAIL
// per case, or the CUDA error a misaligned shared-memory address raises.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/tma1d_probe.cu -o tools/_tma1d_probe
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

constexpr int BOX = 176;

__global__ void load_kernel(const __grid_constant__ CUtensorMap map, float* out, int coord, int off_bytes, bool rank2) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ __align__(8) unsigned long long bar;
    float* dst = reinterpret_cast<float*>(sm + off_bytes);
    for (int i = threadIdx.x; i < BOX + 64; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = -1.0f;
    __syncthreads();
    const unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(BOX * 4));
        if (rank2)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                    (unsigned)__cvta_generic_to_shared(dst)),
                "l"(&map), "r"(coord), "r"(0), "r"(b)
                : "memory");
        else
            asm volatile(
                "cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];" ::"r"(
                    (unsigned)__cvta_generic_to_shared(dst)),
                "l"(&map), "r"(coord), "r"(b)
                : "memory");
    }
    __syncthreads();
    asm volatile(
        "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W; }" ::"r"(b)
        : "memory");
    for (int i = threadIdx.x; i < BOX; i += blockDim.x) out[i] = dst[i];
}

__global__ void store_kernel(const __grid_constant__ CUtensorMap map, int coord, int off_bytes, bool rank2) {
    extern __shared__ __align__(1024) unsigned char sm[];
    float* src = reinterpret_cast<float*>(sm + off_bytes);
    for (int i = threadIdx.x; i < BOX; i += blockDim.x) src[i] = 1000000.0f + i;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        if (rank2)
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&map),
                         "r"(coord), "r"(0), "r"((unsigned)__cvta_generic_to_shared(src))
                         : "memory");
        else
            asm volatile("cp.async.bulk.tensor.1d.global.shared::cta.bulk_group [%0, {%1}], [%2];" ::"l"(&map), "r"(coord),
                         "r"((unsigned)__cvta_generic_to_shared(src))
                         : "memory");
        asm volatile("cp.async.bulk.commit_group;");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const long long N = 1 << 20;
    float* d;
    cudaMalloc(&d, N * 4);
    std::vector<float> h(N);
    for (long long i = 0; i < N; ++i) h[i] = (float)i;
    cudaMemcpy(d, h.data(), N * 4, cudaMemcpyHostToDevice);
    float* out;
    cudaMalloc(&out, BOX * 4);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    alignas(64) CUtensorMap map;
    bool rank2 = false;
    cuuint64_t dim[1] = {(cuuint64_t)N};
    cuuint32_t box[1] = {BOX}, es[1] = {1};
    CUresult r = ((EncodeFn)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 1, d, dim, nullptr, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    std::printf("encode rank-1 map: %d (entry point %p, query %d)\n", (int)r, fn, (int)q);
    if (r != CUDA_SUCCESS) {
        // rank 2, one "row" of N elements
        cuuint64_t dim2[2] = {(cuuint64_t)N, 1};
        cuuint64_t str2[1] = {(cuuint64_t)N * 4};
        cuuint32_t box2[2] = {BOX, 1}, es2[2] = {1, 1};
        r = ((EncodeFn)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dim2, str2, box2, es2,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        std::printf("encode rank-2 map: %d\n", (int)r);
        if (r != CUDA_SUCCESS) return 1;
        rank2 = true;
    }
    const int coords[] = {0, 4, 1000, -4, (int)N - 100, 2};
    const int offs[] = {0, 16, 48, 128, 256};
    for (int off : offs)
        for (int c : coords) {
            load_kernel<<<1, 128, 4096>>>(map, out, c, off, rank2);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                std::printf("load coord %d smem+%d: CUDA error %s\n", c, off, cudaGetErrorString(e));
                return 1;
            }
            std::vector<float> o(BOX);
            cudaMemcpy(o.data(), out, BOX * 4, cudaMemcpyDeviceToHost);
            bool ok = true;
            for (int i = 0; i < BOX; ++i) {
                const long long g = (long long)c + i;
                const float want = (g < 0 || g >= N) ? 0.0f : (float)g;
                if (o[i] != want) ok = false;
            }
            std::printf("load coord %8d smem+%3d: %s (first %g last %g)\n", c, off, ok ? "PASS" : "FAIL", o[0], o[BOX - 1]);
        }
    for (int off : offs)
        for (int c : {1000, 8, (int)N - 100, 7}) {
            cudaMemcpy(d, h.data(), N * 4, cudaMemcpyHostToDevice);
            store_kernel<<<1, 128, 4096>>>(map, c, off, rank2);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                std::printf("store coord %d smem+%d: CUDA error %s\n", c, off, cudaGetErrorString(e));
                return 1;
            }
            std::vector<float> o(N);
            cudaMemcpy(o.data(), d, N * 4, cudaMemcpyDeviceToHost);
            bool ok = true;
            for (long long i = 0; i < N; ++i) {
                const float want = (i >= c && i < c + BOX) ? 1000000.0f + (float)(i - c) : (float)i;
                if (o[i] != want) ok = false;
            }
            std::printf("store coord %8d smem+%3d: %s\n", c, off, ok ? "PASS" : "FAIL");
        }
    return 0;
}
