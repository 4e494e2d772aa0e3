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

// Shared-memory image of one tile: for each (sequence, group) the group's 32
// records, contiguous (one bulk copy each). Consecutive groups are offset by
// an extra 16 bytes and the pattern half by 64, so the 8 lanes of a
// quarter-warp (2 sequences x 4 groups reading the same row/column offset) hit
// 8 distinct 16-byte bank groups in their LDS.128.
__host__ __device__ inline size_t group_stride(size_t pitch) { return 32 * pitch + 16; }
__host__ __device__ inline size_t seq_stride(size_t pitch, int groups) {
    return groups * group_stride(pitch) + 64;
}
size_t tile_smem(size_t pitch, int groups) { return 2 * seq_stride(pitch, groups) + 128; }
int tile_groups(size_t pitch) { return pitch <= 128 ? 8 : 4; }

// One CTA per tile of GROUPS x 32 pairs: bulk-copy each group's records into
// shared memory (TMA, completion on one mbarrier), gather 16-column x 32-pair
// tiles into planes (validating every byte) and store them straight to the
// planes array (8 lanes of a warp fill one 32-byte sector per column/plane).
template <int GROUPS>
__global__ void __launch_bounds__(kPackNT)
pack_tile_kernel(const uint8_t* __restrict__ text, const uint8_t* __restrict__ pattern,
                 size_t pitch, long long n, int m, uint32_t* __restrict__ planes,
                 uint32_t* __restrict__ err_flag) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    const long long g0 = static_cast<long long>(blockIdx.x) * GROUPS;  // first group
    const long long row0 = g0 * 32;
    const long long nblocks = (n + kPackPairs - 1) / kPackPairs;
    const int rows = static_cast<int>(n - row0 < 32 * GROUPS ? n - row0 : 32 * GROUPS);
    const int mc = plane_cols(m);
    const size_t gs = group_stride(pitch), ss = seq_stride(pitch, GROUPS);
    auto rec = [&](int sq, int g) { return sm + sq * ss + g * gs; };
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_expect_tx(&bar, static_cast<uint32_t>(2 * rows * pitch));
    }
    __syncthreads();
    if (threadIdx.x < 2 * GROUPS) {
        const int sq = threadIdx.x / GROUPS, g = threadIdx.x % GROUPS;
        const int r = rows - 32 * g;
        if (r > 0) {
            const uint8_t* src = (sq == 0 ? text : pattern) + (row0 + 32 * g) * pitch;
            bulk_g2s(rec(sq, g), src, static_cast<uint32_t>((r < 32 ? r : 32) * pitch), &bar);
        }
    }
    mbar_wait(&bar, 0);
    if (rows < 32 * GROUPS) {
        // last tile: rows past n read as 'A' (valid; their results are masked)
        const int per_seq = (32 * GROUPS - rows) * static_cast<int>(pitch) / 16;
        const uint4 a4 = make_uint4(0x41414141u, 0x41414141u, 0x41414141u, 0x41414141u);
        for (int i = threadIdx.x; i < 2 * per_seq; i += kPackNT) {
            const int sq = i / per_seq;
            const int byte = rows * static_cast<int>(pitch) + (i % per_seq) * 16;
            const int g = byte / (32 * static_cast<int>(pitch));
            *reinterpret_cast<uint4*>(rec(sq, g) + (byte - g * 32 * static_cast<int>(pitch))) = a4;
        }
        __syncthreads();
    }
    // Items are (chunk, group, sequence) tiles of 32 pairs x 16 columns, the
    // sequence fastest. Full chunks come first and the one chunk straddling m
    // (if any) last, so no warp mixes the two gather variants.
    const int C = mc / CH;
    const int Cfull = m / CH;  // chunks entirely inside [0, m)
    uint32_t err = 0u;
    uint32_t sink[CH * 3];
    for (int it = threadIdx.x; it < 2 * GROUPS * C; it += kPackNT) {
        const int c = it / (2 * GROUPS);
        const int g = (it / 2) % GROUPS;
        const int sq = it % 2;
        uint32_t* dst = planes ? planes + plane_index(sq, g0 + g, c * CH, 0, nblocks, mc) : sink;
        const int stride = planes ? kPackGroups : 1;
        if (c < Cfull)
            err |= gather_chunk<false, false>(rec(sq, g), pitch, 0, 32, c * CH, m, dst, stride);
        else
            err |= gather_chunk<true, false>(rec(sq, g), pitch, 0, 32, c * CH, m, dst, stride);
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
    const int groups = tile_groups(pitch);
    const size_t smem = tile_smem(pitch, groups);
    const long long ngroups = (n + 31) / 32;
    if (smem <= 110 * 1024) {
        static bool attr = false;  // idempotent
        if (!attr) {
            cudaError_t st = cudaFuncSetAttribute(pack_tile_kernel<8>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  110 * 1024);
            if (st == cudaSuccess)
                st = cudaFuncSetAttribute(pack_tile_kernel<4>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
            if (st != cudaSuccess) return st;
            attr = true;
        }
        const unsigned grid = static_cast<unsigned>((ngroups + groups - 1) / groups);
        if (groups == 8)
            pack_tile_kernel<8><<<grid, kPackNT, smem, s>>>(text, pattern, pitch, n, m, planes,
                                                            err_flag);
        else
            pack_tile_kernel<4><<<grid, kPackNT, smem, s>>>(text, pattern, pitch, n, m, planes,
                                                            err_flag);
    } else {
        const long long items = 2 * ngroups * (plane_cols(m) / CH);
        pack_direct_kernel<<<static_cast<unsigned>((items + kPackNT - 1) / kPackNT), kPackNT, 0,
                             s>>>(text, pattern, pitch, n, m, planes, err_flag);
    }
    count_launch();
    return cudaGetLastError();
}

}  // namespace sb
