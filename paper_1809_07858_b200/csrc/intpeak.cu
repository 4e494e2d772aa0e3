// Integer pipe microbenchmark: the denominator of the INT roofline.
//
// BASELINE.md freezes P_int = SMs x (LOP3 lanes/clk/SM) x clock and asks for
// the lane rate to be measured on the box. Each thread runs 8 independent
// dependency chains of the chosen instruction (enough ILP to saturate the pipe
// at full occupancy); the grid covers every SM several times.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace sb {

namespace {

constexpr int kChains = 8;
constexpr int kIters = 4096;

template <int OP>
__global__ void __launch_bounds__(256) int_peak_kernel(uint32_t seed, uint32_t* out) {
    uint32_t x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = seed * (threadIdx.x + 1) + c * 0x9E3779B9u;
    const uint32_t y = seed ^ blockIdx.x, z = seed + threadIdx.x;
#pragma unroll 1
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
            for (int c = 0; c < kChains; ++c) {
                if (OP == 0)
                    asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(y), "r"(z));
                else if (OP == 1)
                    asm volatile("shf.l.wrap.b32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(y), "r"(z));
                else if (OP == 2)
                    asm volatile("prmt.b32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(y), "r"(z));
                else
                    asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(y), "r"(z));
            }
        }
    }
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc ^= x[c];
    if (acc == 0x12345678u) out[0] = acc;  // keep the chains alive
}

template <int OP>
cudaError_t run(cudaStream_t s, double* ops) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint32_t* out = nullptr;
    cudaError_t st = cudaMalloc(&out, sizeof(uint32_t));
    if (st != cudaSuccess) return st;
    const int blocks = sms * 8;  // 8 x 256 threads = full occupancy per SM
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int_peak_kernel<OP><<<blocks, 256, 0, s>>>(1u, out);  // warm-up
    cudaEventRecord(a, s);
    const int reps = 3;
    for (int r = 0; r < reps; ++r) int_peak_kernel<OP><<<blocks, 256, 0, s>>>(2u + r, out);
    cudaEventRecord(b, s);
    count_launch(reps + 1);
    st = cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
    if (st != cudaSuccess) return st;
    const double lane_ops = double(reps) * blocks * 256.0 * kIters * 8.0 * kChains;
    *ops = lane_ops / (ms * 1e-3);
    return cudaGetLastError();
}

}  // namespace

cudaError_t measure_int_peak(int op, cudaStream_t s, double* ops_per_second) {
    switch (op) {
        case 0: return run<0>(s, ops_per_second);
        case 1: return run<1>(s, ops_per_second);
        case 2: return run<2>(s, ops_per_second);
        case 3: return run<3>(s, ops_per_second);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace sb
