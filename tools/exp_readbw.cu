// HBM probe (experiment tool): read-only, read-mostly (5:1, the pack kernel's
// ratio) and copy bandwidth over 6 GB with 16-byte vector loads, grid-stride,
// one launch each, timed with CUDA events after a warm-up.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/exp_readbw tools/exp_readbw.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__global__ void rd(const uint4* __restrict__ p, size_t n, unsigned* sink) {
    uint32_t x = 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x) {
        const uint4 v = __ldcs(p + i);
        x ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (x == 0x12345678u) atomicAdd(sink, 1u);
}

__global__ void rd_wr(const uint4* __restrict__ p, size_t n, uint4* __restrict__ q, int ratio) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x) {
        const uint4 v = __ldcs(p + i);
        if (i % ratio == 0) __stcs(q + i / ratio, v);
    }
}

int main() {
    const size_t bytes = size_t(6) << 30, n = bytes / 16;
    uint4 *a, *b;
    unsigned* sink;
    cudaMalloc(&a, bytes);
    cudaMalloc(&b, bytes);
    cudaMalloc(&sink, 4);
    cudaMemset(a, 1, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int blocksPerSm : {4, 8, 16}) {
        const int grid = sms * blocksPerSm;
        for (int rep = 0; rep < 2; ++rep) {
            float ms;
            cudaEventRecord(e0);
            rd<<<grid, 256>>>(a, n, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep) printf("read-only  %2d CTAs/SM: %.0f GB/s\n", blocksPerSm, bytes / ms / 1e6);
            cudaEventRecord(e0);
            rd_wr<<<grid, 256>>>(a, n, b, 5);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep)
                printf("read 5:1 write %2d CTAs/SM: %.0f GB/s (read+write)\n", blocksPerSm,
                       (bytes + bytes / 5) / ms / 1e6);
            cudaEventRecord(e0);
            rd_wr<<<grid, 256>>>(a, n, b, 1);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep) printf("copy       %2d CTAs/SM: %.0f GB/s (read+write)\n", blocksPerSm, 2 * bytes / ms / 1e6);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
