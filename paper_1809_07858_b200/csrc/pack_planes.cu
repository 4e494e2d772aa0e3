// Stage 1 for pre-packed input (SURVEY §8(b) "packed-planes variant"): pairs
// that the caller already packed with packed_sequence::from_string
// (proj/src/packed_sequence.cpp:7-34) arrive in that class's own storage —
// per sequence three LSB-first uint64 planes low/high/N
// (proj/include/prefilter/packed_sequence.hpp:50-53) — and are re-sliced here
// into the pair-sliced plane layout of pack.cuh.
//
// The re-slicing is a 32 x 32 bit-matrix transpose per (group of 32 pairs,
// 32-column block, plane): lane b of a warp holds pair b's 32 plane bits of
// the block (one 32-bit load), five shuffle-xor block-swap stages later lane c
// holds column c's word with bit b = pair b — exactly one planes word. A CTA
// covers one pair block (8 groups = 8 warps), so for each (column, plane) the
// block's 8 group words are written by the 8 warps side by side and merge into
// full sectors in L2. The codes differ from the ASCII path's (A/C/G/T =
// 00/01/10/11 instead of bits 1-2 of the byte) but the search only compares
// codes for equality and reads N from its own plane, so the mismatch word
// (Plo^Tlo)|(Phi^Thi)|PN|TN is the same.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"
#include "pack.cuh"
#include "pack_tile.cuh"

namespace sb {

namespace {

// Per-lane constants of the five block-swap stages (s = 16, 8, 4, 2, 1): the
// bits a lane keeps (its own half of each 2s-block) and the rotation that
// brings the partner's other half into place (left by s for the lower lane,
// right by s = left by 32 - s for the upper lane; the kept-mask hides the
// bits that wrapped around).
struct Transpose32 {
    uint32_t keep[5];
    uint32_t rot[5];
    __device__ __forceinline__ explicit Transpose32(int lane) {
        const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            const int s = 16 >> i;
            const bool upper = lane & s;
            keep[i] = upper ? ~masks[i] : masks[i];
            rot[i] = upper ? 32u - s : static_cast<uint32_t>(s);
        }
    }
    // lane b holds row b (bit c = element (b, c)); returns column `lane` (bit b = element (b, lane))
    __device__ __forceinline__ uint32_t operator()(uint32_t x) const {
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            const uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, x, 16 >> i);
            const uint32_t r = __funnelshift_l(y, y, rot[i]);  // rotate left
            x = (x & keep[i]) | (r & ~keep[i]);
        }
        return x;
    }
};

// Shared-memory staged form (W64 = ceil(m/64) <= 8, the default): one bulk
// copy (TMA, completion on an mbarrier) brings the pair block's rows — one
// contiguous range — into shared memory; each lane loads its own row into
// registers with 8-byte loads (rows are 24*W64 bytes apart: conflict-free per
// quarter warp); each warp transposes its group's 32 x 32 tiles and writes the
// column words into the block's [col][plane][group] image, which is exactly
// the block's contiguous region of the planes layout up to a padded column
// stride (25 words, so the 32 lanes' column stores hit 32 banks); the block
// then streams it out with 16-byte stores. grid: (pair blocks, sequences);
// block: 8 warps = 8 groups.
template <int W64>
__global__ void __launch_bounds__(256)
pack_planes_kernel(const uint64_t* __restrict__ text, const uint64_t* __restrict__ pattern,
                   long long n, int m, uint32_t* __restrict__ planes,
                   uint32_t* __restrict__ nflags) {
    constexpr int RW = 6 * W64;  // u32 words per pair row
    extern __shared__ __align__(128) uint32_t smem[];
    __shared__ __align__(8) uint64_t bar;
    uint32_t* in = smem;                       // [256][RW]
    constexpr int kOut = 3 * kPackGroups + 1;  // padded column stride
    uint32_t* out = smem + kPackPairs * RW;    // [m][kOut]
    const int s = blockIdx.y;
    const uint32_t* src = reinterpret_cast<const uint32_t*>(s == 0 ? text : pattern);
    const long long pair0 = static_cast<long long>(blockIdx.x) * kPackPairs;
    const int rows = static_cast<int>(n - pair0 < kPackPairs ? n - pair0 : kPackPairs);
    const uint32_t bytes = static_cast<uint32_t>(rows) * RW * 4u;
    const uint32_t bulk = bytes & ~15u;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_expect_tx(&bar, bulk);
        if (bulk) bulk_g2s(in, src + pair0 * RW, bulk, &bar);
    }
    // ragged tail (not a multiple of 16 bytes): plain loads
    for (uint32_t w = bulk / 4 + threadIdx.x; w < bytes / 4; w += blockDim.x)
        in[w] = __ldg(src + pair0 * RW + w);
    __syncthreads();
    mbar_wait(&bar, 0);
    const int lane = threadIdx.x & 31;
    const int gw = threadIdx.x >> 5;
    const int prow = gw * 32 + lane;
    uint32_t r[RW];
    if (prow < rows) {
        const uint2* row = reinterpret_cast<const uint2*>(in + prow * RW);
#pragma unroll
        for (int q = 0; q < RW / 2; ++q) {
            const uint2 v = row[q];
            r[2 * q] = v.x;
            r[2 * q + 1] = v.y;
        }
    } else {
#pragma unroll
        for (int q = 0; q < RW; ++q) r[q] = 0u;
    }
    // N-presence (nflags, pack.cuh): a group whose 32 rows hold no N stores no N
    // planes — the search then drops its N terms — and a block without any N
    // skips its N region altogether
    __shared__ int block_n;
    if (threadIdx.x == 0) block_n = 0;
    uint32_t nz = 0u;
#pragma unroll
    for (int j = 0; j < 2 * W64; ++j) nz |= r[2 * 2 * W64 + j];
    const bool group_n = nflags == nullptr || __any_sync(~0u, nz != 0u);
    __syncthreads();  // block_n initialised
    if (group_n && lane == 0) block_n = 1;
    const long long nblocks = (n + kPackPairs - 1) / kPackPairs;
    const long long g0 = static_cast<long long>(blockIdx.x) * kPackGroups;
    if (nflags != nullptr && lane == 0 && g0 + gw < (n + 31) / 32)
        nflags[nflag_index(s, g0 + gw, nblocks)] = group_n ? 1u : 0u;
    const Transpose32 transpose32(lane);
#pragma unroll
    for (int j = 0; j < 2 * W64; ++j) {
        if (32 * j < m) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                if (k == 2 && !group_n) break;  // warp-uniform
                const uint32_t col_word = transpose32(r[k * 2 * W64 + j]);
                const int col = 32 * j + lane;
                if (col < m) out[col * kOut + k * kPackGroups + gw] = col_word;
            }
        }
    }
    __syncthreads();
    // lo/hi region: 16 words per column (image words 0..15), then the N region:
    // 8 words per column (image words 16..23)
    uint4* dst = reinterpret_cast<uint4*>(planes + lohi_index(s, g0, 0, 0, nblocks, plane_cols(m)));
    for (int c = threadIdx.x; c < m * kLhColWords / 4; c += blockDim.x) {
        const uint32_t* src_w = out + (c >> 2) * kOut + 4 * (c & 3);
        dst[c] = make_uint4(src_w[0], src_w[1], src_w[2], src_w[3]);
    }
    if (!block_n) return;  // no group of this block reads its N planes
    uint4* ndst = reinterpret_cast<uint4*>(planes + nplane_index(s, g0, 0, nblocks, plane_cols(m)));
    for (int c = threadIdx.x; c < m * kNColWords / 4; c += blockDim.x) {
        const uint32_t* src_w = out + (c >> 1) * kOut + kLhColWords + 4 * (c & 1);
        ndst[c] = make_uint4(src_w[0], src_w[1], src_w[2], src_w[3]);
    }
}

size_t pack_planes_smem(int m) {
    const int w64 = (m + 63) / 64;
    return (static_cast<size_t>(kPackPairs) * 6 * w64 + static_cast<size_t>(m) * (3 * kPackGroups + 1)) * 4;
}

// Fallback for very long records (staging does not fit shared memory): the
// same transpose straight from global memory.
__global__ void __launch_bounds__(256)
pack_planes_direct_kernel(const uint64_t* __restrict__ text, const uint64_t* __restrict__ pattern,
                          long long n, int m, uint32_t* __restrict__ planes) {
    const int s = blockIdx.y;
    const uint32_t* src = reinterpret_cast<const uint32_t*>(s == 0 ? text : pattern);
    const int lane = threadIdx.x & 31;
    const long long g = static_cast<long long>(blockIdx.x) * kPackGroups + (threadIdx.x >> 5);
    const long long pair = g * 32 + lane;
    const int w64 = (m + 63) / 64;
    const size_t row_words = 6u * static_cast<size_t>(w64);
    const long long nblocks = (n + kPackPairs - 1) / kPackPairs;
    const int mc = plane_cols(m);
    const bool live = pair < n;
    const uint32_t* row = src + (live ? pair : 0) * row_words;
    const int nb32 = (m + 31) / 32;
    const Transpose32 transpose32(lane);
    for (int j = 0; j < nb32; ++j) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const uint32_t x = live ? __ldg(row + k * 2 * w64 + j) : 0u;
            const uint32_t col_word = transpose32(x);
            const int col = 32 * j + lane;
            if (col < m)
                planes[k < 2 ? lohi_index(s, g, col, k, nblocks, mc)
                             : nplane_index(s, g, col, nblocks, mc)] = col_word;
        }
    }
}

}  // namespace

bool pack_planes_writes_nflags(const uint64_t* text, const uint64_t* pattern, int m) {
    const bool aligned =
        (reinterpret_cast<uintptr_t>(text) | reinterpret_cast<uintptr_t>(pattern)) % 16 == 0;
    return (m + 63) / 64 <= 8 && pack_planes_smem(m) <= 200 * 1024 && aligned;
}

cudaError_t launch_pack_planes(const uint64_t* text, const uint64_t* pattern, long long n, int m,
                               uint32_t* planes, cudaStream_t s, uint32_t* nflags) {
    if (n <= 0) return cudaSuccess;
    if (planes == nullptr || m <= 0) return cudaErrorInvalidValue;
    if (nflags && !pack_planes_writes_nflags(text, pattern, m)) return cudaErrorInvalidValue;
    if (nflags) {  // the all-zero N column image N-free groups of mixed warps read
        const cudaError_t st = cudaMemsetAsync(nflags + nflag_words(n), 0,
                                               nzero_words(m) * sizeof(uint32_t), s);
        if (st != cudaSuccess) return st;
    }
    const long long nblocks = (n + kPackPairs - 1) / kPackPairs;
    const dim3 grid(static_cast<unsigned>(nblocks), 2);
    const size_t smem = pack_planes_smem(m);
    const int w64 = (m + 63) / 64;
    const bool aligned =
        (reinterpret_cast<uintptr_t>(text) | reinterpret_cast<uintptr_t>(pattern)) % 16 == 0;
    if (w64 <= 8 && smem <= 200 * 1024 && aligned) {
        switch (w64) {
#define SB_PP(W)                                                                               \
    case W: {                                                                                  \
        const cudaError_t st = ensure_smem_attr<pack_planes_kernel<W>>(200 * 1024);            \
        if (st != cudaSuccess) return st;                                                      \
        pack_planes_kernel<W><<<grid, 32 * kPackGroups, smem, s>>>(text, pattern, n, m, planes, nflags); \
        break;                                                                                 \
    }
            SB_PP(1) SB_PP(2) SB_PP(3) SB_PP(4) SB_PP(5) SB_PP(6) SB_PP(7) SB_PP(8)
#undef SB_PP
        }
    } else {
        pack_planes_direct_kernel<<<grid, 32 * kPackGroups, 0, s>>>(text, pattern, n, m, planes);
    }
    count_launch();
    return cudaGetLastError();
}

}  // namespace sb
