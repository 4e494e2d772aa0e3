// MAGNET pre-alignment filter on sm_100a.
//
// Reference: magnet_filter / recover_subsequences / exen / longest_zero_run
// (proj/src/magnet.cpp:9-87). With threshold e the reference runs e+1
// "extract and encapsulate" steps over the 2e+1 diagonals of the
// neighborhood map: in the active column range every diagonal nominates its
// longest zero run (earliest on ties), scanned in the order 0, -1, +1, -2, +2,
// ... where only a strictly longer run displaces the incumbent; the winner's
// columns are recovered (bv bits cleared), the run plus one flanking column
// on each side is retired, and the left range then the right range are
// searched, depth first, on the shared budget. estimate = popcount(bv),
// accept = estimate <= e.
//
// B200 form: the recursion is data dependent, so one thread owns one pair
// and keeps everything in registers as m-bit vectors (W 32-bit words, LSB =
// column 0):
//  * the pair's lo/hi/N planes are built from the ASCII bytes (bits 1/2/3);
//  * the recursion is an explicit stack of column ranges (pre-order, left
//    range on top), bounded by the budget;
//  * the sub-ranges of a step never include the retired columns, so the
//    reference's column masking (neighborhood_map::mask_columns) cannot change
//    any later nomination and is not materialised;
//  * a diagonal's mismatch vector D_d = (P<<|d| or P>>d vs T) is rebuilt on
//    the fly while the nomination walks d = 0, -1, +1, ...: the shifted
//    pattern planes advance by one bit per step (funnel shifts);
//  * the longest zero run of z = ~D_d & range is found with log-step
//    doubling on S_L (bit i set iff z[i..i+L-1] are all ones):
//    S_2L = S_L & (S_L >> L) up to the first empty vector, then a binary
//    refinement S_{L+2^k} = S_{2^k} & (S_L >> 2^k) — all shift amounts are
//    compile-time — and the earliest start is the lowest set bit of S_L.
// Input records are validated before this kernel runs (launch_validate), so
// every byte is one of A/C/G/T/N.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace sb {

namespace {

// x >> 1 (towards column 0), zero in at the top.
template <int W>
__device__ __forceinline__ void shr1(uint32_t (&x)[W]) {
#pragma unroll
    for (int i = 0; i < W; ++i) x[i] = __funnelshift_r(x[i], i + 1 < W ? x[i + 1] : 0u, 1);
}

// x << 1 (away from column 0), zero in at column 0.
template <int W>
__device__ __forceinline__ void shl1(uint32_t (&x)[W]) {
#pragma unroll
    for (int i = W - 1; i >= 0; --i) x[i] = __funnelshift_l(i > 0 ? x[i - 1] : 0u, x[i], 1);
}

// out = x >> S; S is a constant after unrolling at every call site, so the
// word selection folds away and x stays in registers.
template <int W>
__device__ __forceinline__ void shr_const(const uint32_t (&x)[W], uint32_t (&out)[W], int S) {
    const int Q = S / 32, R = S % 32;
#pragma unroll
    for (int i = 0; i < W; ++i) {
        const uint32_t a = i + Q < W ? x[i + Q] : 0u;
        const uint32_t b = i + Q + 1 < W ? x[i + Q + 1] : 0u;
        out[i] = R == 0 ? a : __funnelshift_r(a, b, R);
    }
}

template <int W>
__device__ __forceinline__ bool vany(const uint32_t (&x)[W]) {
    uint32_t o = 0u;
#pragma unroll
    for (int i = 0; i < W; ++i) o |= x[i];
    return o != 0u;
}

// Lowest set bit index of a non-zero vector.
template <int W>
__device__ __forceinline__ int vffs(const uint32_t (&x)[W]) {
    int r = 32 * W;
#pragma unroll
    for (int i = W - 1; i >= 0; --i)
        if (x[i]) r = 32 * i + __ffs(x[i]) - 1;
    return r;
}

// Bits [lo, hi) of word i.
__device__ __forceinline__ uint32_t range_word(int i, int lo, int hi) {
    const int a = min(max(lo - 32 * i, 0), 32);
    const int b = min(max(hi - 32 * i, 0), 32);
    const uint32_t below_b = b >= 32 ? ~0u : ((1u << b) - 1u);
    const uint32_t below_a = a >= 32 ? ~0u : ((1u << a) - 1u);
    return below_b & ~below_a;
}

__host__ __device__ constexpr int log2_ceil(int v) { return v <= 1 ? 0 : 1 + log2_ceil((v + 1) / 2); }

// Longest run of ones in z (the zero run of the diagonal), earliest start.
// Returns the length (0 if z is empty) and writes the start.
template <int W>
__device__ __forceinline__ int longest_run(const uint32_t (&z)[W], int* start) {
    constexpr int KMAX = log2_ceil(32 * W) + 1;  // S_{2^k} for k < KMAX
    uint32_t g[KMAX][W];
#pragma unroll
    for (int i = 0; i < W; ++i) g[0][i] = z[i];
    if (!vany(g[0])) return 0;
    int K = 0;
#pragma unroll
    for (int k = 1; k < KMAX; ++k) {
        if (K == k - 1) {
            uint32_t t[W];
            shr_const<W>(g[k - 1], t, 1 << (k - 1));
#pragma unroll
            for (int i = 0; i < W; ++i) g[k][i] = g[k - 1][i] & t[i];
            if (vany(g[k])) K = k;
        }
    }
    // runs of length >= 2^K exist, none of length 2^(K+1)
    uint32_t cur[W];
#pragma unroll
    for (int i = 0; i < W; ++i) cur[i] = g[0][i];
    int len = 1;
#pragma unroll
    for (int k = KMAX - 1; k >= 1; --k) {
        if (k == K) {
#pragma unroll
            for (int i = 0; i < W; ++i) cur[i] = g[k][i];
            len = 1 << k;
        }
    }
#pragma unroll
    for (int k = KMAX - 2; k >= 0; --k) {
        if (k < K) {  // S_{len + 2^k} = S_{2^k} & (S_len >> 2^k)
            uint32_t t[W];
            shr_const<W>(cur, t, 1 << k);
#pragma unroll
            for (int i = 0; i < W; ++i) t[i] &= g[k][i];
            if (vany(t)) {
#pragma unroll
                for (int i = 0; i < W; ++i) cur[i] = t[i];
                len += 1 << k;
            }
        }
    }
    *start = vffs(cur);
    return len;
}

// Planes (bits 1/2/3 of the ASCII bytes) of one record row, m <= 32 W.
template <int W>
__device__ __forceinline__ void load_planes(const uint8_t* __restrict__ row, int m,
                                            uint32_t (&lo)[W], uint32_t (&hi)[W],
                                            uint32_t (&nn)[W]) {
    constexpr uint32_t K = (1u << 24) | (1u << 17) | (1u << 10) | (1u << 3);
#pragma unroll
    for (int i = 0; i < W; ++i) {
        uint32_t a = 0u, b = 0u, c = 0u;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int col = 32 * i + 4 * q;
            if (col < m) {
                uint32_t x = *reinterpret_cast<const uint32_t*>(row + col);
                // bytes past m (padding of the row) read as 'A'
                if (col + 4 > m) {
                    const uint32_t keep = (1u << (8 * (m - col))) - 1u;
                    x = (x & keep) | (0x41414141u & ~keep);
                }
                // bit k of byte j (at 8j+k) -> bit j of a nibble: (x>>k)&0x01010101, times K, >> 24
                a |= (((((x >> 1) & 0x01010101u) * K) >> 24) & 0xFu) << (4 * q);
                b |= (((((x >> 2) & 0x01010101u) * K) >> 24) & 0xFu) << (4 * q);
                c |= (((((x >> 3) & 0x01010101u) * K) >> 24) & 0xFu) << (4 * q);
            }
        }
        lo[i] = a;
        hi[i] = b;
        nn[i] = c;
    }
}

template <int W>
__global__ void __launch_bounds__(128)
magnet_kernel(const uint8_t* __restrict__ text, const uint8_t* __restrict__ pattern, size_t pitch,
              long long n, int m, int e, uint32_t* __restrict__ accept,
              uint32_t* __restrict__ estimates, uint64_t* __restrict__ bits) {
    const long long pair = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool live = pair < n;
    uint32_t bv[W];
    uint32_t valid[W];
#pragma unroll
    for (int i = 0; i < W; ++i) valid[i] = range_word(i, 0, m);
    int est = 0;
    if (live) {
        uint32_t Tlo[W], Thi[W], TN[W], Plo[W], Phi[W], PN[W];
        load_planes<W>(text + pair * pitch, m, Tlo, Thi, TN);
        load_planes<W>(pattern + pair * pitch, m, Plo, Phi, PN);
#pragma unroll
        for (int i = 0; i < W; ++i) bv[i] = valid[i];
        // explicit pre-order stack of column ranges [lo, hi] (hi may be < lo)
        constexpr int kStack = 16 * W + 4;
        int16_t st_lo[kStack], st_hi[kStack];
        int sp = 0;
        st_lo[0] = 0;
        st_hi[0] = static_cast<int16_t>(m - 1);
        sp = 1;
        int budget = e + 1;
        while (sp > 0 && budget > 0) {
            --sp;
            const int lo = st_lo[sp], hi = st_hi[sp];
            if (lo > hi) continue;
            const int clo = max(lo, 0), chi = min(hi, m - 1);
            if (clo > chi) continue;
            uint32_t rng[W];
#pragma unroll
            for (int i = 0; i < W; ++i) rng[i] = range_word(i, clo, chi + 1);
            const int width = chi - clo + 1;
            // nomination: d = 0, -1, +1, -2, +2, ...; shifted pattern planes
            // (and the in-range mask) advance one column per step
            uint32_t Llo[W], Lhi[W], LN[W], Lv[W], Rlo[W], Rhi[W], RN[W], Rv[W];
#pragma unroll
            for (int i = 0; i < W; ++i) {
                Llo[i] = Rlo[i] = Plo[i];
                Lhi[i] = Rhi[i] = Phi[i];
                LN[i] = RN[i] = PN[i];
                Lv[i] = Rv[i] = valid[i];
            }
            int best_len = 0, best_start = 0;
            for (int step = 0; step <= e && best_len < width; ++step) {
                if (step > 0) {
                    shl1<W>(Llo);
                    shl1<W>(Lhi);
                    shl1<W>(LN);
                    shl1<W>(Lv);
                    shr1<W>(Rlo);
                    shr1<W>(Rhi);
                    shr1<W>(RN);
                    shr1<W>(Rv);
                }
#pragma unroll 1
                for (int side = 0; side < (step == 0 ? 1 : 2); ++side) {
                    uint32_t z[W];
#pragma unroll
                    for (int i = 0; i < W; ++i) {
                        const uint32_t slo = side == 0 ? Llo[i] : Rlo[i];
                        const uint32_t shi = side == 0 ? Lhi[i] : Rhi[i];
                        const uint32_t sN = side == 0 ? LN[i] : RN[i];
                        const uint32_t sv = side == 0 ? Lv[i] : Rv[i];
                        // match = in range, neither N, same (lo, hi) code
                        const uint32_t mm = (slo ^ Tlo[i]) | (shi ^ Thi[i]) | sN | TN[i];
                        z[i] = ~mm & sv & rng[i];
                    }
                    int s = 0;
                    const int len = longest_run<W>(z, &s);
                    if (len > best_len) {
                        best_len = len;
                        best_start = s;
                    }
                    if (best_len >= width) break;
                }
            }
            if (best_len == 0) continue;
            --budget;
#pragma unroll
            for (int i = 0; i < W; ++i) bv[i] &= ~range_word(i, best_start, best_start + best_len);
            // right range below the left one: left is searched first
            if (sp + 2 <= kStack) {
                st_lo[sp] = static_cast<int16_t>(best_start + best_len + 1);
                st_hi[sp] = static_cast<int16_t>(hi);
                ++sp;
                st_lo[sp] = static_cast<int16_t>(lo);
                st_hi[sp] = static_cast<int16_t>(best_start - 2);
                ++sp;
            }
        }
#pragma unroll
        for (int i = 0; i < W; ++i) est += __popc(bv[i]);
    }
    const bool acc = live && est <= e;
    const uint32_t word = __ballot_sync(0xFFFFFFFFu, acc);
    if ((threadIdx.x & 31) == 0 && pair < n) accept[pair / 32] = word;
    if (!live) return;
    if (estimates) estimates[pair] = static_cast<uint32_t>(est);
    if (bits) {
        const int wpp = (m + 63) / 64;
        uint64_t* dst = bits + pair * wpp;
#pragma unroll
        for (int i = 0; i < W; i += 2) {
            if (i / 2 < wpp) {
                const uint64_t lo = bv[i];
                const uint64_t hi = i + 1 < W ? bv[i + 1] : 0u;
                dst[i / 2] = lo | (hi << 32);
            }
        }
    }
}

template <int W>
cudaError_t launch_magnet_w(const uint8_t* text, const uint8_t* pattern, size_t pitch, long long n,
                            int m, int e, uint32_t* accept, uint32_t* estimates, uint64_t* bits,
                            cudaStream_t s) {
    const unsigned grid = static_cast<unsigned>((n + 127) / 128);
    magnet_kernel<W><<<grid, 128, 0, s>>>(text, pattern, pitch, n, m, e, accept, estimates, bits);
    count_launch();
    return cudaGetLastError();
}

}  // namespace

bool magnet_supported(int m) { return m >= 1 && m <= kMagnetMaxM; }

cudaError_t launch_magnet(const uint8_t* text, const uint8_t* pattern, size_t pitch, long long n,
                          int m, int e, uint32_t* accept, uint32_t* estimates, uint64_t* bits,
                          cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    if (!magnet_supported(m) || pitch % 4 != 0 || e < 0 || e >= m) return cudaErrorInvalidValue;
    if (m <= 32) return launch_magnet_w<1>(text, pattern, pitch, n, m, e, accept, estimates, bits, s);
    if (m <= 64) return launch_magnet_w<2>(text, pattern, pitch, n, m, e, accept, estimates, bits, s);
    if (m <= 128) return launch_magnet_w<4>(text, pattern, pitch, n, m, e, accept, estimates, bits, s);
    if (m <= 256) return launch_magnet_w<8>(text, pattern, pitch, n, m, e, accept, estimates, bits, s);
    return launch_magnet_w<16>(text, pattern, pitch, n, m, e, accept, estimates, bits, s);
}

}  // namespace sb
