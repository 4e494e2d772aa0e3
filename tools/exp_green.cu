// Green-context feasibility probe (experiment tool, not product code):
//  1. split the device's SMs into two green contexts (P and the rest),
//  2. launch a kernel that records %smid per CTA into a stream of each,
//     with runtime <<<>>> launches and buffers from cudaMalloc (primary context),
//  3. report how many distinct SMs each partition's kernel touched, and whether
//     two long kernels in the two partitions ran concurrently.
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/exp_green tools/exp_green.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <set>
#include <vector>

#define CK(x)                                                                          \
    do {                                                                               \
        CUresult r_ = (x);                                                             \
        if (r_ != CUDA_SUCCESS) {                                                      \
            const char* s_ = nullptr;                                                  \
            cuGetErrorString(r_, &s_);                                                 \
            std::printf("FAIL %s: %s\n", #x, s_ ? s_ : "?");                          \
            return 1;                                                                  \
        }                                                                              \
    } while (0)
#define RK(x)                                                                          \
    do {                                                                               \
        cudaError_t r_ = (x);                                                          \
        if (r_ != cudaSuccess) {                                                       \
            std::printf("FAIL %s: %s\n", #x, cudaGetErrorString(r_));                 \
            return 1;                                                                  \
        }                                                                              \
    } while (0)

__global__ void record_smid(unsigned* out, long long spin) {
    unsigned id;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
    if (threadIdx.x == 0) out[blockIdx.x] = id;
    long long t0 = clock64();
    while (clock64() - t0 < spin) {
    }
}

int main(int argc, char** argv) {
    const unsigned want = argc > 1 ? std::atoi(argv[1]) : 56;
    RK(cudaSetDevice(0));
    RK(cudaFree(nullptr));  // primary context up
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    CUdevResource all{};
    CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
    std::printf("device SMs: %u\n", all.sm.smCount);
    CUdevResource part{}, rest{};
    unsigned groups = 1;
    CK(cuDevSmResourceSplitByCount(&part, &groups, &all, &rest, 0, want));
    std::printf("split: %u groups, part %u SMs, rest %u SMs\n", groups, part.sm.smCount,
                rest.sm.smCount);
    CUdevResourceDesc d0, d1;
    CK(cuDevResourceGenerateDesc(&d0, &part, 1));
    CK(cuDevResourceGenerateDesc(&d1, &rest, 1));
    CUgreenCtx g0, g1;
    CK(cuGreenCtxCreate(&g0, d0, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CK(cuGreenCtxCreate(&g1, d1, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream s0, s1;
    CK(cuGreenCtxStreamCreate(&s0, g0, CU_STREAM_NON_BLOCKING, 0));
    CK(cuGreenCtxStreamCreate(&s1, g1, CU_STREAM_NON_BLOCKING, 0));
    const int blocks = 148 * 8;
    unsigned *b0, *b1;
    RK(cudaMalloc(&b0, blocks * sizeof(unsigned)));
    RK(cudaMalloc(&b1, blocks * sizeof(unsigned)));
    // 1. placement
    record_smid<<<blocks, 128, 0, (cudaStream_t)s0>>>(b0, 1000);
    RK(cudaGetLastError());
    record_smid<<<blocks, 128, 0, (cudaStream_t)s1>>>(b1, 1000);
    RK(cudaGetLastError());
    RK(cudaDeviceSynchronize());
    std::vector<unsigned> h0(blocks), h1(blocks);
    RK(cudaMemcpy(h0.data(), b0, blocks * 4, cudaMemcpyDeviceToHost));
    RK(cudaMemcpy(h1.data(), b1, blocks * 4, cudaMemcpyDeviceToHost));
    std::set<unsigned> u0(h0.begin(), h0.end()), u1(h1.begin(), h1.end());
    int overlap = 0;
    for (unsigned x : u0) overlap += u1.count(x);
    std::printf("partition 0 kernel used %zu SMs, partition 1 kernel used %zu SMs, shared %d\n",
                u0.size(), u1.size(), overlap);
    // 2. concurrency: a long kernel in each partition, timed together vs alone
    cudaEvent_t a, b;
    RK(cudaEventCreate(&a));
    RK(cudaEventCreate(&b));
    const long long spin = 20000000;  // ~10 ms at 2 GHz
    float alone = 0, together = 0;
    RK(cudaEventRecord(a, (cudaStream_t)s0));
    record_smid<<<part.sm.smCount, 128, 0, (cudaStream_t)s0>>>(b0, spin);
    RK(cudaEventRecord(b, (cudaStream_t)s0));
    RK(cudaEventSynchronize(b));
    RK(cudaEventElapsedTime(&alone, a, b));
    RK(cudaDeviceSynchronize());
    RK(cudaEventRecord(a, 0));
    RK(cudaStreamWaitEvent((cudaStream_t)s0, a, 0));
    RK(cudaStreamWaitEvent((cudaStream_t)s1, a, 0));
    record_smid<<<part.sm.smCount, 128, 0, (cudaStream_t)s0>>>(b0, spin);
    record_smid<<<rest.sm.smCount, 128, 0, (cudaStream_t)s1>>>(b1, spin);
    cudaEvent_t e0, e1;
    RK(cudaEventCreate(&e0));
    RK(cudaEventCreate(&e1));
    RK(cudaEventRecord(e0, (cudaStream_t)s0));
    RK(cudaEventRecord(e1, (cudaStream_t)s1));
    RK(cudaStreamWaitEvent(0, e0, 0));
    RK(cudaStreamWaitEvent(0, e1, 0));
    RK(cudaEventRecord(b, 0));
    RK(cudaEventSynchronize(b));
    RK(cudaEventElapsedTime(&together, a, b));
    std::printf("one partition kernel alone %.2f ms; both partitions together %.2f ms (%s)\n",
                alone, together, together < 1.5f * alone ? "concurrent" : "serialised");
    std::printf("OK\n");
    return 0;
}
