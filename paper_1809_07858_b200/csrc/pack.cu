// Stage 1: ASCII records -> pair-sliced planes (see pack.cuh for the layout).
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"
#include "pack.cuh"
#include "pack_tile.cuh"

namespace sb {

namespace {

// One CTA per tile of GROUPS x 32 pairs (pack_one_tile, pack_tile.cuh).
template <int GROUPS, int ALIGN, bool NIB>
__global__ void __launch_bounds__(kPackNT)
pack_tile_kernel(const uint8_t* __restrict__ text, const uint8_t* __restrict__ pattern,
                 size_t pitch, long long n, int m, uint32_t* __restrict__ planes,
                 uint32_t* __restrict__ err_flag) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    __syncthreads();
    const uint32_t err = pack_one_tile<ALIGN, kPackNT, NIB>(
        sm, &bar, 0, GROUPS, static_cast<long long>(blockIdx.x) * GROUPS, text, pattern, pitch, n, m,
        planes);
    if (!NIB && err) atomicOr(err_flag, 1u);
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
    const int C = (mc + CH - 1) / CH;
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

template <int GROUPS, int ALIGN, bool NIB = false>
static cudaError_t launch_tile(const uint8_t* text, const uint8_t* pattern, size_t pitch,
                               long long n, int m, uint32_t* planes, uint32_t* err_flag,
                               cudaStream_t s) {
    const cudaError_t st = ensure_smem_attr<pack_tile_kernel<GROUPS, ALIGN, NIB>>(110 * 1024);
    if (st != cudaSuccess) return st;
    const long long ngroups = (n + 31) / 32;
    const unsigned grid = static_cast<unsigned>((ngroups + GROUPS - 1) / GROUPS);
    pack_tile_kernel<GROUPS, ALIGN, NIB><<<grid, kPackNT, tile_smem(pitch, GROUPS), s>>>(
        text, pattern, pitch, n, m, planes, err_flag);
    return cudaGetLastError();
}

cudaError_t launch_pack(const uint8_t* text, const uint8_t* pattern, size_t pitch, long long n,
                        int m, uint32_t* planes, uint32_t* err_flag, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    if (pitch % 4 != 0) return cudaErrorInvalidValue;
    const int groups = tile_groups(pitch);
    const size_t smem = tile_smem(pitch, groups);
    cudaError_t st;
    if (smem <= 110 * 1024) {
        const bool a16 = pitch % 16 == 0;
        if (groups == 8)
            st = a16 ? launch_tile<8, 16>(text, pattern, pitch, n, m, planes, err_flag, s)
                     : launch_tile<8, 4>(text, pattern, pitch, n, m, planes, err_flag, s);
        else
            st = a16 ? launch_tile<4, 16>(text, pattern, pitch, n, m, planes, err_flag, s)
                     : launch_tile<4, 4>(text, pattern, pitch, n, m, planes, err_flag, s);
    } else {
        const long long items = 2 * ((n + 31) / 32) * ((plane_cols(m) + CH - 1) / CH);
        pack_direct_kernel<<<static_cast<unsigned>((items + kPackNT - 1) / kPackNT), kPackNT, 0,
                             s>>>(text, pattern, pitch, n, m, planes, err_flag);
        st = cudaGetLastError();
    }
    count_launch();
    return st;
}

bool nibble_pack_fits(int m) {
    const size_t np = nibble_pitch(m);
    return tile_smem(np, tile_groups(np)) <= 110 * 1024;
}

cudaError_t launch_pack_nibbles(const uint8_t* text, const uint8_t* pattern, long long n, int m,
                                uint32_t* planes, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    if (!nibble_pack_fits(m) || planes == nullptr) return cudaErrorInvalidValue;
    const size_t np = nibble_pitch(m);
    const cudaError_t st = tile_groups(np) == 8
                               ? launch_tile<8, 4, true>(text, pattern, np, n, m, planes, nullptr, s)
                               : launch_tile<4, 4, true>(text, pattern, np, n, m, planes, nullptr, s);
    count_launch();
    return st;
}

}  // namespace sb
