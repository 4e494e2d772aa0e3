// Exact edit distance on the GPU: the verification step after the filter and
// the alignment oracle of `eval`.
//
// Reference: banded_edit_distance(a, b, e), proj/src/edit_distance.cpp:26-70 —
// unit-cost Levenshtein restricted to the 2e+1 diagonals, the distance when it
// is <= e and "out of band" otherwise; an 'N' never matches (even 'N').
// Any alignment with <= e edits stays inside those diagonals, so the banded
// value equals the full Levenshtein distance d whenever d <= e, and the band
// can only make the value larger otherwise: within <=> d <= e. We therefore
// compute d exactly with Myers' bit-vector algorithm (Myers 1999, block form;
// global-distance boundary D[0][j] = j, i.e. +1 carried into block 0 every
// column) and report d <= e ? d : -1.
//
// One thread per pair; the read is the "pattern" whose match vectors Peq are
// built (A/C/G/T; an N sets no bit), the reference segment is scanned column by
// column (a text N matches nothing: Eq = 0).
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace sb {

namespace {

__device__ __forceinline__ int base_code(uint8_t c) {
    switch (c) {
        case 'A': return 0;
        case 'C': return 1;
        case 'G': return 2;
        case 'T': return 3;
        default: return -1;  // 'N' (bytes were validated before this kernel)
    }
}

// One block step of Myers' algorithm: returns the horizontal delta leaving the
// block's top row (hin/hout in {-1, 0, +1}).
__device__ __forceinline__ int advance_block(uint64_t& pv, uint64_t& mv, uint64_t eq, int hin,
                                             uint64_t high) {
    const uint64_t xv = eq | mv;
    if (hin < 0) eq |= 1ull;
    const uint64_t xh = (((eq & pv) + pv) ^ pv) | eq;
    uint64_t ph = mv | ~(xh | pv);
    uint64_t mh = pv & xh;
    int hout = 0;
    if (ph & high) hout = 1;
    if (mh & high) hout = -1;
    ph <<= 1;
    mh <<= 1;
    if (hin < 0)
        mh |= 1ull;
    else if (hin > 0)
        ph |= 1ull;
    pv = mh | ~(xv | ph);
    mv = ph & xv;
    return hout;
}

template <int W>
__global__ void __launch_bounds__(128)
myers_kernel(const uint8_t* __restrict__ text, const uint8_t* __restrict__ pattern, size_t pitch,
             long long n, int m, int e, int32_t* __restrict__ out) {
    const long long p = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const uint8_t* P = pattern + p * pitch;
    const uint8_t* T = text + p * pitch;
    uint64_t peq[4][W];
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int w = 0; w < W; ++w) peq[c][w] = 0ull;
    for (int i = 0; i < m; ++i) {
        const int c = base_code(P[i]);
        const uint64_t bit = 1ull << (i & 63);
#pragma unroll
        for (int w = 0; w < W; ++w)
            if (w == (i >> 6)) {
                if (c == 0) peq[0][w] |= bit;
                if (c == 1) peq[1][w] |= bit;
                if (c == 2) peq[2][w] |= bit;
                if (c == 3) peq[3][w] |= bit;
            }
    }
    uint64_t pv[W], mv[W];
#pragma unroll
    for (int w = 0; w < W; ++w) {
        pv[w] = ~0ull;
        mv[w] = 0ull;
    }
    const int last = (m - 1) >> 6;
    const uint64_t last_high = 1ull << ((m - 1) & 63);
    int score = m;
    for (int j = 0; j < m; ++j) {
        const int c = base_code(T[j]);
        int h = 1;  // D[0][j+1] - D[0][j] = +1
#pragma unroll
        for (int w = 0; w < W; ++w) {
            if (w > last) break;
            uint64_t eq = 0ull;
            if (c == 0) eq = peq[0][w];
            if (c == 1) eq = peq[1][w];
            if (c == 2) eq = peq[2][w];
            if (c == 3) eq = peq[3][w];
            h = advance_block(pv[w], mv[w], eq, h, w == last ? last_high : (1ull << 63));
        }
        score += h;
    }
    out[p] = score <= e ? score : -1;
}

}  // namespace

cudaError_t launch_edit_distance(const uint8_t* text, const uint8_t* pattern, size_t pitch,
                                 long long n, int m, int e, int32_t* out, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const unsigned grid = static_cast<unsigned>((n + 127) / 128);
    const int words = (m + 63) / 64;
    if (words <= 1)
        myers_kernel<1><<<grid, 128, 0, s>>>(text, pattern, pitch, n, m, e, out);
    else if (words <= 2)
        myers_kernel<2><<<grid, 128, 0, s>>>(text, pattern, pitch, n, m, e, out);
    else if (words <= 4)
        myers_kernel<4><<<grid, 128, 0, s>>>(text, pattern, pitch, n, m, e, out);
    else if (words <= 8)
        myers_kernel<8><<<grid, 128, 0, s>>>(text, pattern, pitch, n, m, e, out);
    else if (words <= 16)
        myers_kernel<16><<<grid, 128, 0, s>>>(text, pattern, pitch, n, m, e, out);
    else
        return cudaErrorInvalidValue;  // m > 1024: not supported by the verifier
    count_launch();
    return cudaGetLastError();
}

}  // namespace sb
