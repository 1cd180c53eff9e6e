// Probe: SM-driven reads of pinned host memory over PCIe (zero-copy) against
// the copy engine, alone and together. Prints GB/s per mode.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o zc_probe tools/zc_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    std::printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

template <int U>
__global__ void __launch_bounds__(256) k_fetch(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                               size_t n16) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n16; i0 += stride * U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t i = i0 + (size_t)u * stride;
            if (i < n16) v[u] = __ldcs(src + i);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t i = i0 + (size_t)u * stride;
            if (i < n16) dst[i] = v[u];
        }
    }
}

int main() {
    const size_t bytes = 119232000;  // 256 grey frames at 1242 x 375
    void *h, *h2, *d, *d2;
    CK(cudaHostAlloc(&h, bytes, cudaHostAllocDefault));
    CK(cudaHostAlloc(&h2, bytes, cudaHostAllocDefault));
    CK(cudaMalloc(&d, bytes));
    CK(cudaMalloc(&d2, bytes));
    for (size_t i = 0; i < bytes; i += 4096) ((char*)h)[i] = (char)i, ((char*)h2)[i] = (char)i;
    cudaPointerAttributes at;
    CK(cudaPointerGetAttributes(&at, h));
    std::printf("host ptr %p device ptr %p type %d\n", h, at.devicePointer, (int)at.type);
    cudaStream_t s1, s2;
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    const size_t n16 = bytes / 16;
    auto run = [&](int mode, int grid, int unroll) -> float {
        float best = 1e9f;
        for (int rep = 0; rep < 4; ++rep) {
            CK(cudaDeviceSynchronize());
            CK(cudaEventRecord(a, s1));
            CK(cudaStreamWaitEvent(s2, a, 0));
            if (mode != 1) {
                if (unroll == 4) k_fetch<4><<<grid, 256, 0, s1>>>((const uint4*)at.devicePointer, (uint4*)d, n16);
                else k_fetch<8><<<grid, 256, 0, s1>>>((const uint4*)at.devicePointer, (uint4*)d, n16);
            }
            if (mode != 0) CK(cudaMemcpyAsync(d2, h2, bytes, cudaMemcpyHostToDevice, s2));
            cudaEvent_t c;
            CK(cudaEventCreate(&c));
            CK(cudaEventRecord(c, s2));
            CK(cudaStreamWaitEvent(s1, c, 0));
            CK(cudaEventRecord(b, s1));
            CK(cudaEventSynchronize(b));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            CK(cudaEventDestroy(c));
            if (ms < best) best = ms;
        }
        return best;
    };
    const float dma = run(1, 0, 4);
    std::printf("dma alone: %.2f ms  %.1f GB/s\n", dma, bytes / dma / 1e6);
    for (int grid : {16, 32, 64, 148, 296}) {
        for (int u : {4, 8}) {
            const float zc = run(0, grid, u);
            const float both = run(2, grid, u);
            std::printf("zero-copy grid %3d x256 U%d: %.2f ms %.1f GB/s | with dma: %.2f ms, %.1f GB/s combined\n",
                        grid, u, zc, bytes / zc / 1e6, both, 2 * bytes / both / 1e6);
        }
    }
    return 0;
}
