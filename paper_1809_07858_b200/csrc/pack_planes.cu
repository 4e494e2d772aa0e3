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

namespace sb {

namespace {

__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
    // stage s swaps the off-diagonal s x s blocks between lanes l and l ^ s
    const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const int s = 16 >> i;
        const uint32_t m = masks[i];
        const uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, x, s);
        x = (lane & s) ? ((x & ~m) | ((y >> s) & m)) : ((x & m) | ((y << s) & ~m));
    }
    return x;
}

// grid: (pair blocks, sequences); block: 8 warps = the 8 groups of a pair block.
__global__ void __launch_bounds__(256)
pack_planes_kernel(const uint64_t* __restrict__ text, const uint64_t* __restrict__ pattern,
                   long long n, int m, uint32_t* __restrict__ planes) {
    const int s = blockIdx.y;
    const uint32_t* src = reinterpret_cast<const uint32_t*>(s == 0 ? text : pattern);
    const int lane = threadIdx.x & 31;
    const long long g = static_cast<long long>(blockIdx.x) * kPackGroups + (threadIdx.x >> 5);
    const long long pair = g * 32 + lane;
    const int w64 = (m + 63) / 64;
    const size_t row_words = 3u * 2u * static_cast<size_t>(w64);  // u32 words per pair
    const long long nblocks = (n + kPackPairs - 1) / kPackPairs;
    const int mc = plane_cols(m);
    const bool live = pair < n;
    const uint32_t* row = src + (live ? pair : 0) * row_words;
    const int nb32 = (m + 31) / 32;
    for (int j = 0; j < nb32; ++j) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            // u32 word j of plane k (little-endian halves of the u64 words)
            const uint32_t x = live ? __ldg(row + k * 2 * w64 + j) : 0u;
            const uint32_t col_word = transpose32(x, lane);
            const int col = 32 * j + lane;
            if (col < m) planes[plane_index(s, g, col, k, nblocks, mc)] = col_word;
        }
    }
}

}  // namespace

cudaError_t launch_pack_planes(const uint64_t* text, const uint64_t* pattern, long long n, int m,
                               uint32_t* planes, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    if (planes == nullptr || m <= 0) return cudaErrorInvalidValue;
    const long long nblocks = (n + kPackPairs - 1) / kPackPairs;
    const dim3 grid(static_cast<unsigned>(nblocks), 2);
    pack_planes_kernel<<<grid, 32 * kPackGroups, 0, s>>>(text, pattern, n, m, planes);
    count_launch();
    return cudaGetLastError();
}

}  // namespace sb
