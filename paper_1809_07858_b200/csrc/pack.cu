// Stage 1: ASCII records -> pair-sliced planes (see pack.cuh for the layout).
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"
#include "pack.cuh"

namespace sb {

namespace {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
    }
}

// Bytes of dynamic shared memory for one pair block.
size_t tile_smem(size_t pitch, int m) {
    return 2 * size_t(kPackPairs) * pitch + size_t(2) * plane_cols(m) * 3 * kPackGroups * 4;
}

// One CTA per pair block: TMA the two record tiles into shared memory, gather
// 16-column x 32-pair tiles into planes (validating every byte), stage the
// block's planes in shared memory and write them out contiguously.
__global__ void __launch_bounds__(kPackNT)
pack_tile_kernel(const uint8_t* __restrict__ text, const uint8_t* __restrict__ pattern,
                 size_t pitch, long long n, int m, uint32_t* __restrict__ planes,
                 uint32_t* __restrict__ err_flag) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    const long long blk = blockIdx.x;
    const long long nblocks = (n + kPackPairs - 1) / kPackPairs;
    const long long row0 = blk * kPackPairs;
    const int rows = static_cast<int>(n - row0 < kPackPairs ? n - row0 : kPackPairs);
    const int mc = plane_cols(m);
    uint8_t* srec0 = sm;
    uint8_t* srec1 = sm + size_t(kPackPairs) * pitch;
    uint32_t* sout = reinterpret_cast<uint32_t*>(sm + 2 * size_t(kPackPairs) * pitch);
    const uint32_t bytes = static_cast<uint32_t>(rows * pitch);
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_expect_tx(&bar, 2 * bytes);
        bulk_g2s(srec0, text + row0 * pitch, bytes, &bar);
        bulk_g2s(srec1, pattern + row0 * pitch, bytes, &bar);
    }
    mbar_wait(&bar, 0);

    const int C = mc / CH;
    const int items = 2 * kPackGroups * C;
    uint32_t err = 0u;
    for (int it = threadIdx.x; it < items; it += kPackNT) {
        const int c = it % C;
        const int g = (it / C) % kPackGroups;
        const int s = it / (C * kPackGroups);
        const uint8_t* src = (s == 0 ? srec0 : srec1) + size_t(32 * g) * pitch;
        uint32_t* dst = sout + (size_t(s) * mc + c * CH) * 3 * kPackGroups + g;
        const int grows = rows - 32 * g;  // valid rows of this group (may be <= 0)
        err |= produce_chunk(src, pitch, 0, grows, c, m, dst, kPackGroups);
    }
    __syncthreads();
    if (planes) {
        // each sequence's block of planes is contiguous in global memory
        const int words = mc * 3 * kPackGroups;  // per sequence, multiple of 4
        for (int s = 0; s < 2; ++s) {
            const uint4* from = reinterpret_cast<const uint4*>(sout + size_t(s) * words);
            uint4* to = reinterpret_cast<uint4*>(planes + plane_index(s, blk * kPackGroups, 0, 0,
                                                                      nblocks, mc));
            for (int i = threadIdx.x; i < words / 4; i += kPackNT) to[i] = from[i];
        }
    }
    if (err) atomicOr(err_flag, 1u);
}

// Long records (tile does not fit in shared memory): each thread gathers one
// (group, chunk, sequence) tile straight from global memory.
__global__ void __launch_bounds__(kPackNT)
pack_direct_kernel(const uint8_t* __restrict__ text, const uint8_t* __restrict__ pattern,
                   size_t pitch, long long n, int m, uint32_t* __restrict__ planes,
                   uint32_t* __restrict__ err_flag) {
    const long long ngroups = (n + 31) / 32;
    const long long nblocks = (n + kPackPairs - 1) / kPackPairs;
    const int mc = plane_cols(m);
    const int C = mc / CH;
    const long long items = 2 * ngroups * C;
    const long long it = static_cast<long long>(blockIdx.x) * kPackNT + threadIdx.x;
    if (it >= items) return;
    const int c = static_cast<int>(it % C);
    const long long g = (it / C) % ngroups;
    const int s = static_cast<int>(it / (C * ngroups));
    uint32_t sink[CH * 3];
    uint32_t* dst = planes ? planes + plane_index(s, g, c * CH, 0, nblocks, mc) : sink;
    const int stride = planes ? kPackGroups : 1;
    const uint32_t err = produce_chunk(s == 0 ? text : pattern, pitch, g * 32, n, c, m, dst, stride);
    if (err) atomicOr(err_flag, 1u);
}

}  // namespace

cudaError_t launch_pack(const uint8_t* text, const uint8_t* pattern, size_t pitch, long long n,
                        int m, uint32_t* planes, uint32_t* err_flag, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const size_t smem = tile_smem(pitch, m);
    if (smem <= 200 * 1024) {
        static size_t attr = 0;  // largest dynamic smem configured so far (idempotent)
        if (smem > attr) {
            cudaError_t st = cudaFuncSetAttribute(pack_tile_kernel,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  static_cast<int>(200 * 1024));
            if (st != cudaSuccess) return st;
            attr = 200 * 1024;
        }
        const long long nblocks = (n + kPackPairs - 1) / kPackPairs;
        pack_tile_kernel<<<static_cast<unsigned>(nblocks), kPackNT, smem, s>>>(text, pattern, pitch,
                                                                              n, m, planes, err_flag);
    } else {
        const long long items = 2 * ((n + 31) / 32) * (plane_cols(m) / CH);
        pack_direct_kernel<<<static_cast<unsigned>((items + kPackNT - 1) / kPackNT), kPackNT, 0,
                             s>>>(text, pattern, pitch, n, m, planes, err_flag);
    }
    count_launch();
    return cudaGetLastError();
}

}  // namespace sb
