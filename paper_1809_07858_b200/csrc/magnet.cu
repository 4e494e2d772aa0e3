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
#include <cstdlib>

#include "kernels.cuh"
#include "pack.cuh"

#include <type_traits>

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

// x >> 1 / x << 1 with ones shifted in (out-of-range pattern columns read as N).
template <int W>
__device__ __forceinline__ void shr1_ones(uint32_t (&x)[W]) {
#pragma unroll
    for (int i = 0; i < W; ++i) x[i] = __funnelshift_r(x[i], i + 1 < W ? x[i + 1] : ~0u, 1);
}
template <int W>
__device__ __forceinline__ void shl1_ones(uint32_t (&x)[W]) {
#pragma unroll
    for (int i = W - 1; i >= 0; --i) x[i] = __funnelshift_l(i > 0 ? x[i - 1] : ~0u, x[i], 1);
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
    // doubling: cur = S_{2^K} for the largest K with a non-empty S_{2^K}
    uint32_t cur[W];
#pragma unroll
    for (int i = 0; i < W; ++i) cur[i] = z[i];
    int K = 0;
#pragma unroll
    for (int k = 1; k < KMAX; ++k) {
        uint32_t t[W];
        shr_const<W>(g[k - 1], t, 1 << (k - 1));
        uint32_t o = 0u;
#pragma unroll
        for (int i = 0; i < W; ++i) {
            g[k][i] = g[k - 1][i] & t[i];
            o |= g[k][i];
        }
        if (o == 0u) break;
#pragma unroll
        for (int i = 0; i < W; ++i) cur[i] = g[k][i];
        K = k;
    }
    // refinement: S_{len + 2^k} = S_{2^k} & (S_len >> 2^k), k = K-1 .. 0
    int len = 1 << K;
#pragma unroll
    for (int k = KMAX - 2; k >= 0; --k) {
        if (k >= K) continue;
        uint32_t t[W];
        shr_const<W>(cur, t, 1 << k);
        uint32_t o = 0u;
#pragma unroll
        for (int i = 0; i < W; ++i) {
            t[i] &= g[k][i];
            o |= t[i];
        }
        if (o != 0u) {
#pragma unroll
            for (int i = 0; i < W; ++i) cur[i] = t[i];
            len += 1 << k;
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

// Record sources: where a pair's planes come from. AsciiSrc reads validated
// ASCII records (pitch bytes per row); DibitSrc reads host-packed dibit records
// (pack.cuh, 4*ceil(m/16) bytes per row) plus optional N-plane rows.
struct AsciiSrc {
    const uint8_t* text;
    const uint8_t* pattern;
    size_t pitch;
    template <int W>
    __device__ __forceinline__ void load(long long pair, int seq, int m, uint32_t (&lo)[W],
                                         uint32_t (&hi)[W], uint32_t (&nn)[W]) const {
        load_planes<W>((seq ? pattern : text) + pair * pitch, m, lo, hi, nn);
    }
};

struct DibitSrc {
    const uint8_t* text;
    const uint8_t* pattern;
    const uint8_t* ntext;  // null: no N in the batch
    const uint8_t* npattern;
    template <int W>
    __device__ __forceinline__ void load(long long pair, int seq, int m, uint32_t (&lo)[W],
                                         uint32_t (&hi)[W], uint32_t (&nn)[W]) const {
        constexpr uint32_t K = (1u << 24) | (1u << 17) | (1u << 10) | (1u << 3);
        const size_t dp = dibit_pitch(m), np = nplane_pitch(m);
        const uint32_t* row =
            reinterpret_cast<const uint32_t*>((seq ? pattern : text) + pair * dp);
        const uint8_t* nb = seq ? npattern : ntext;
        const uint32_t* nrow = nb ? reinterpret_cast<const uint32_t*>(nb + pair * np) : nullptr;
        const int nw16 = (m + 15) / 16;
#pragma unroll
        for (int i = 0; i < W; ++i) {
            uint32_t a = 0u, b = 0u;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (2 * i + h < nw16) {
                    const uint32_t w = row[2 * i + h];
                    // byte q holds columns q, q+4, q+8, q+12 at bit pairs 2t: column 4t+q
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        a |= (((((w >> (2 * t)) & 0x01010101u) * K) >> 24) & 0xFu) << (16 * h + 4 * t);
                        b |= (((((w >> (2 * t + 1)) & 0x01010101u) * K) >> 24) & 0xFu) << (16 * h + 4 * t);
                    }
                }
            }
            lo[i] = a;
            hi[i] = b;
            nn[i] = (nrow && i < (m + 31) / 32) ? nrow[i] : 0u;
        }
    }
};

// Up to 128 columns: 4 CTAs (16 warps) per SM at 128 registers (ptxas would
// take 141 and fit 3): m=100 E=2/5/10 +15-17%. 129-256 columns: 3 CTAs at 168
// (from 255 + spills at 2): m=150 E=7 +5%, m=250 E=10 +10%, E<=5 within 1%.
// Longer records keep the compiler's choice.
template <int W, class Src>
__global__ void __launch_bounds__(128, (W <= 4 ? 4 : (W <= 8 ? 3 : 1)))
magnet_kernel(Src src, long long n, int m, int e, uint32_t* __restrict__ accept,
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
        src.template load<W>(pair, 0, m, Tlo, Thi, TN);
        src.template load<W>(pair, 1, m, Plo, Phi, PN);
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
            // nomination: d = 0, -1, +1, -2, +2, ...; the shifted pattern planes
            // advance one column per step; out-of-range pattern columns are
            // folded into the N plane (ones shifted in)
            uint32_t Llo[W], Lhi[W], LN[W], Rlo[W], Rhi[W], RN[W];
#pragma unroll
            for (int i = 0; i < W; ++i) {
                Llo[i] = Rlo[i] = Plo[i];
                Lhi[i] = Rhi[i] = Phi[i];
                LN[i] = RN[i] = PN[i] | ~valid[i];
            }
            int best_len = 0, best_start = 0;
            auto nominate = [&](const uint32_t (&slo)[W], const uint32_t (&shi)[W],
                                const uint32_t (&sN)[W]) {
                uint32_t z[W];
#pragma unroll
                for (int i = 0; i < W; ++i)
                    z[i] = ~((slo[i] ^ Tlo[i]) | (shi[i] ^ Thi[i]) | sN[i] | TN[i]) & rng[i];
                int st = 0;
                const int len = longest_run<W>(z, &st);
                if (len > best_len) {
                    best_len = len;
                    best_start = st;
                }
            };
            nominate(Llo, Lhi, LN);  // d = 0
            for (int step = 1; step <= e && best_len < width; ++step) {
                shl1<W>(Llo);
                shl1<W>(Lhi);
                shl1_ones<W>(LN);
                nominate(Llo, Lhi, LN);  // d = -step
                if (best_len >= width) break;
                shr1<W>(Rlo);
                shr1<W>(Rhi);
                shr1_ones<W>(RN);
                nominate(Rlo, Rhi, RN);  // d = +step
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

// ---- warp-cooperative form (13 <= E <= 31) ----------------------------------------
// One warp owns 32 consecutive pairs and walks them one after the other; the
// lanes split the nomination instead of the pairs: lane l owns the diagonals
// with scan-order index o = l and o = l + 32 (o = 0, 1, 2, ... is
// d = 0, -1, +1, -2, +2, ...). The recursion is then uniform across the warp
// (one pair at a time: no divergence in the control flow), each lane builds
// its diagonals' mismatch vectors once per pair (a funnel shift by |d| < 32),
// and a nomination step is one longest_run per lane plus one warp max
// (redux.sync) over key = len*128 + (127 - o): the longest run wins and, among
// equal lengths, the smallest scan index — the reference's "strictly longer
// displaces" rule (magnet.cpp:41-52). The range stack lives in shared memory.
constexpr int kMagnetWarpNT = 128;

// One record row -> W plane words (bits 1/2/3 of the bytes), built by the warp:
// lane l converts columns 4l (+128 per chunk) and the words are assembled with
// shuffles; every lane ends with all W words.
template <int W>
__device__ __forceinline__ void warp_load_planes(const uint8_t* __restrict__ row, int m, int lane,
                                                 uint32_t (&lo)[W], uint32_t (&hi)[W],
                                                 uint32_t (&nn)[W]) {
    constexpr uint32_t K = (1u << 24) | (1u << 17) | (1u << 10) | (1u << 3);
#pragma unroll
    for (int i = 0; i < W; ++i) lo[i] = hi[i] = nn[i] = 0u;
#pragma unroll
    for (int c = 0; c < (W + 3) / 4; ++c) {  // 128 columns per chunk
        const int col = 128 * c + 4 * lane;
        uint32_t x = 0x41414141u;
        if (col < m) {
            x = *reinterpret_cast<const uint32_t*>(row + col);
            if (col + 4 > m) {
                const uint32_t keep = (1u << (8 * (m - col))) - 1u;
                x = (x & keep) | (0x41414141u & ~keep);
            }
        }
        uint32_t v[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            uint32_t nib = ((((x >> (k + 1)) & 0x01010101u) * K) >> 24) & 0xFu;
            nib <<= 4 * (lane & 7);
            nib |= __shfl_xor_sync(0xFFFFFFFFu, nib, 1);
            nib |= __shfl_xor_sync(0xFFFFFFFFu, nib, 2);
            nib |= __shfl_xor_sync(0xFFFFFFFFu, nib, 4);
            v[k] = nib;  // lanes 8q..8q+7 hold word 4c+q
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (4 * c + q < W) {
                lo[4 * c + q] = __shfl_sync(0xFFFFFFFFu, v[0], 8 * q);
                hi[4 * c + q] = __shfl_sync(0xFFFFFFFFu, v[1], 8 * q);
                nn[4 * c + q] = __shfl_sync(0xFFFFFFFFu, v[2], 8 * q);
            }
        }
    }
}

// Mismatch vector of diagonal d (|d| < 32): bit j = pattern[j+d] vs text[j];
// pattern columns outside [0, m) and N on either side mismatch.
template <int W>
__device__ __forceinline__ void diag_vector(int d, const uint32_t (&Plo)[W], const uint32_t (&Phi)[W],
                                            const uint32_t (&PNx)[W], const uint32_t (&Tlo)[W],
                                            const uint32_t (&Thi)[W], const uint32_t (&TN)[W],
                                            uint32_t (&D)[W]) {
    const int sft = d < 0 ? -d : d;
#pragma unroll
    for (int i = 0; i < W; ++i) {
        uint32_t slo, shi, sN;
        if (d >= 0) {  // bit j <- bit j + d: shift right, ones in at the top for N
            slo = __funnelshift_r(Plo[i], i + 1 < W ? Plo[i + 1] : 0u, sft);
            shi = __funnelshift_r(Phi[i], i + 1 < W ? Phi[i + 1] : 0u, sft);
            sN = __funnelshift_r(PNx[i], i + 1 < W ? PNx[i + 1] : ~0u, sft);
        } else {  // bit j <- bit j - |d|: shift left, ones in at column 0 for N
            slo = __funnelshift_l(i > 0 ? Plo[i - 1] : 0u, Plo[i], sft);
            shi = __funnelshift_l(i > 0 ? Phi[i - 1] : 0u, Phi[i], sft);
            sN = __funnelshift_l(i > 0 ? PNx[i - 1] : ~0u, PNx[i], sft);
        }
        D[i] = (slo ^ Tlo[i]) | (shi ^ Thi[i]) | sN | TN[i];
    }
}

// Up to 256 columns: 4 CTAs (16 warps) per SM at 128 registers (ptxas would
// take 168-190 and fit 2-3; the few spills cost less than the lost warps):
// m=150 E=15 83 -> 109, m=250 E=15 68 -> 90, E=25 37.6 -> 50.8 M pairs/s.
template <int W, class Src>
__global__ void __launch_bounds__(kMagnetWarpNT, (W <= 8 ? 4 : 1))
magnet_warp_kernel(Src src, long long n, int m, int e, uint32_t* __restrict__ accept,
                   uint32_t* __restrict__ estimates, uint64_t* __restrict__ bits) {
    constexpr int kStack = 16 * W + 4;
    __shared__ int16_t st_lo_all[kMagnetWarpNT / 32][kStack];
    __shared__ int16_t st_hi_all[kMagnetWarpNT / 32][kStack];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    int16_t* st_lo = st_lo_all[wib];
    int16_t* st_hi = st_hi_all[wib];
    const long long group = static_cast<long long>(blockIdx.x) * (kMagnetWarpNT / 32) + wib;
    const long long pair0 = group * 32;
    if (pair0 >= n) return;  // whole warp leaves together
    const int npairs = static_cast<int>(n - pair0 < 32 ? n - pair0 : 32);
    uint32_t valid[W];
#pragma unroll
    for (int i = 0; i < W; ++i) valid[i] = range_word(i, 0, m);
    // this lane's diagonals (scan order o -> d)
    const int o0 = lane, o1 = lane + 32;
    auto d_of = [](int o) { return o == 0 ? 0 : ((o & 1) ? -((o + 1) >> 1) : (o >> 1)); };
    const bool has0 = o0 <= 2 * e, has1 = o1 <= 2 * e;
    const int d0 = d_of(o0), d1 = d_of(o1);
    uint32_t acc_word = 0u;
    for (int k = 0; k < npairs; ++k) {
        const long long pair = pair0 + k;
        uint32_t D0[W], D1[W];
        {
            uint32_t Tlo[W], Thi[W], TN[W], Plo[W], Phi[W], PN[W];
            if constexpr (std::is_same_v<Src, AsciiSrc>) {
                // the warp converts the row together (lane l: columns 4l, +128, ...)
                warp_load_planes<W>(src.text + pair * src.pitch, m, lane, Tlo, Thi, TN);
                warp_load_planes<W>(src.pattern + pair * src.pitch, m, lane, Plo, Phi, PN);
            } else {
                // every lane decodes the record itself (same addresses: broadcast loads)
                src.template load<W>(pair, 0, m, Tlo, Thi, TN);
                src.template load<W>(pair, 1, m, Plo, Phi, PN);
            }
#pragma unroll
            for (int i = 0; i < W; ++i) PN[i] |= ~valid[i];
            if (has0) {
                diag_vector<W>(d0, Plo, Phi, PN, Tlo, Thi, TN, D0);
            } else {
#pragma unroll
                for (int i = 0; i < W; ++i) D0[i] = ~0u;
            }
            if (has1) {
                diag_vector<W>(d1, Plo, Phi, PN, Tlo, Thi, TN, D1);
            } else {
#pragma unroll
                for (int i = 0; i < W; ++i) D1[i] = ~0u;
            }
        }
        uint32_t bv[W];
#pragma unroll
        for (int i = 0; i < W; ++i) bv[i] = valid[i];
        if (lane == 0) {
            st_lo[0] = 0;
            st_hi[0] = static_cast<int16_t>(m - 1);
        }
        __syncwarp();
        int sp = 1;
        int budget = e + 1;
        while (sp > 0 && budget > 0) {
            --sp;
            const int lo = st_lo[sp], hi = st_hi[sp];
            __syncwarp();  // everyone has read the entry before it is overwritten
            if (lo > hi) continue;
            const int clo = max(lo, 0), chi = min(hi, m - 1);
            if (clo > chi) continue;
            uint32_t rng[W], z[W];
#pragma unroll
            for (int i = 0; i < W; ++i) rng[i] = range_word(i, clo, chi + 1);
#pragma unroll
            for (int i = 0; i < W; ++i) z[i] = ~D0[i] & rng[i];
            int s0 = 0, s1 = 0;
            const int l0 = longest_run<W>(z, &s0);
            int l1 = 0;
            if (has1) {
#pragma unroll
                for (int i = 0; i < W; ++i) z[i] = ~D1[i] & rng[i];
                l1 = longest_run<W>(z, &s1);
            }
            // this lane's best: longer first, then the smaller scan index (o0 < o1)
            const bool take1 = l1 > l0;
            const int len = take1 ? l1 : l0;
            const int st = take1 ? s1 : s0;
            const int o = take1 ? o1 : o0;
            const unsigned key = len > 0 ? (static_cast<unsigned>(len) << 7) | (127u - o) : 0u;
            const unsigned best = __reduce_max_sync(0xFFFFFFFFu, key);
            if (best == 0u) continue;
            const int winner = __ffs(__ballot_sync(0xFFFFFFFFu, key == best)) - 1;
            const int best_start = __shfl_sync(0xFFFFFFFFu, st, winner);
            const int best_len = static_cast<int>(best >> 7);
            --budget;
#pragma unroll
            for (int i = 0; i < W; ++i) bv[i] &= ~range_word(i, best_start, best_start + best_len);
            if (lane == 0 && sp + 2 <= kStack) {
                st_lo[sp] = static_cast<int16_t>(best_start + best_len + 1);
                st_hi[sp] = static_cast<int16_t>(hi);
                st_lo[sp + 1] = static_cast<int16_t>(lo);
                st_hi[sp + 1] = static_cast<int16_t>(best_start - 2);
            }
            sp += 2;
            __syncwarp();
        }
        int est = 0;
#pragma unroll
        for (int i = 0; i < W; ++i) est += __popc(bv[i]);
        if (est <= e) acc_word |= 1u << k;
        if (lane == 0 && estimates) estimates[pair] = static_cast<uint32_t>(est);
        if (bits) {
            const int wpp = (m + 63) / 64;
#pragma unroll
            for (int i = 0; i < W; i += 2) {
                if (lane == i / 2 && i / 2 < wpp) {
                    const uint64_t a = bv[i];
                    const uint64_t b = i + 1 < W ? bv[i + 1] : 0u;
                    bits[pair * wpp + i / 2] = a | (b << 32);
                }
            }
        }
    }
    if (lane == 0) accept[group] = acc_word;
}

template <int W, class Src>
cudaError_t launch_magnet_warp_w(const Src& src, long long n, int m, int e, uint32_t* accept,
                                 uint32_t* estimates, uint64_t* bits, cudaStream_t s) {
    const long long groups = (n + 31) / 32;
    constexpr int wpb = kMagnetWarpNT / 32;
    const unsigned grid = static_cast<unsigned>((groups + wpb - 1) / wpb);
    magnet_warp_kernel<W, Src><<<grid, kMagnetWarpNT, 0, s>>>(src, n, m, e, accept, estimates,
                                                              bits);
    count_launch();
    return cudaGetLastError();
}

bool magnet_warp_enabled() {
    static const bool v = [] {
        const char* env = std::getenv("PF_MAGNET_WARP");
        return !(env && env[0] == '0');
    }();
    return v;
}

template <int W, class Src>
cudaError_t launch_magnet_w(const Src& src, long long n, int m, int e, uint32_t* accept,
                            uint32_t* estimates, uint64_t* bits, cudaStream_t s) {
    const unsigned grid = static_cast<unsigned>((n + 127) / 128);
    magnet_kernel<W, Src><<<grid, 128, 0, s>>>(src, n, m, e, accept, estimates, bits);
    count_launch();
    return cudaGetLastError();
}

// Kernel choice by E and the register width W = ceil(m/32) (rounded to 1, 2, 4, 8, 16).
template <class Src>
cudaError_t launch_magnet_src(const Src& src, long long n, int m, int e, uint32_t* accept,
                              uint32_t* estimates, uint64_t* bits, cudaStream_t s) {
    // the warp form pays per-pair setup and a warp reduction per extraction; it
    // wins once most lanes own a diagonal (measured: m=250 E=15 68 vs 52 M pairs/s,
    // E=25 38 vs 23; m=100 E=10 219 vs 242, m=150 E=7 110 vs 194)
    if (e >= 13 && e <= 31 && magnet_warp_enabled()) {
        if (m <= 32) return launch_magnet_warp_w<1>(src, n, m, e, accept, estimates, bits, s);
        if (m <= 64) return launch_magnet_warp_w<2>(src, n, m, e, accept, estimates, bits, s);
        if (m <= 128) return launch_magnet_warp_w<4>(src, n, m, e, accept, estimates, bits, s);
        if (m <= 256) return launch_magnet_warp_w<8>(src, n, m, e, accept, estimates, bits, s);
        return launch_magnet_warp_w<16>(src, n, m, e, accept, estimates, bits, s);
    }
    if (m <= 32) return launch_magnet_w<1>(src, n, m, e, accept, estimates, bits, s);
    if (m <= 64) return launch_magnet_w<2>(src, n, m, e, accept, estimates, bits, s);
    if (m <= 128) return launch_magnet_w<4>(src, n, m, e, accept, estimates, bits, s);
    if (m <= 256) return launch_magnet_w<8>(src, n, m, e, accept, estimates, bits, s);
    return launch_magnet_w<16>(src, n, m, e, accept, estimates, bits, s);
}

}  // namespace

bool magnet_supported(int m) { return m >= 1 && m <= kMagnetMaxM; }

cudaError_t launch_magnet(const uint8_t* text, const uint8_t* pattern, size_t pitch, long long n,
                          int m, int e, uint32_t* accept, uint32_t* estimates, uint64_t* bits,
                          cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    if (!magnet_supported(m) || pitch % 4 != 0 || e < 0 || e >= m) return cudaErrorInvalidValue;
    return launch_magnet_src(AsciiSrc{text, pattern, pitch}, n, m, e, accept, estimates, bits, s);
}

cudaError_t launch_magnet_dibits(const uint8_t* text, const uint8_t* pattern, const uint8_t* ntext,
                                 const uint8_t* npattern, long long n, int m, int e,
                                 uint32_t* accept, uint32_t* estimates, uint64_t* bits,
                                 cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    if (!magnet_supported(m) || e < 0 || e >= m) return cudaErrorInvalidValue;
    return launch_magnet_src(DibitSrc{text, pattern, ntext, npattern}, n, m, e, accept, estimates,
                             bits, s);
}

}  // namespace sb
