// Blocked pair-sliced search for window widths other than 4 (3, 5, 6, 7, 8):
// the same structure as the width-4 kernel's D-rebuilding form (fused.cuh),
// generalised over the width W with a runtime threshold E.
//
// Reference: select_window / commit_window / shouji_filter
// (proj/src/shouji.cpp:17-58) with window_zero_table's width (:9-15).
//
// Per block of B = 4 windows j0..j0+3 the D columns j0 .. j0+W+2 are rebuilt
// for every diagonal (pattern columns in a register ring, the diagonal loop
// rolled in chunks of X steps); each window's candidate is the slice
// D[j..j+W-1] with key 2*ones + bit0 (ones by a hand-built carry-save adder),
// the strict first arg-min over d = -E..E is kept with explicit-LOP3 compare
// and select, and commit_window becomes the W-1-bit state machine: window j's
// last bit is always still 1, so "strictly more zeros than the incumbent" is
// ones(best) <= popcount(bv[j..j+W-2]).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "bitslice.cuh"
#include "fused.cuh"

namespace sb {

template <int W>
struct WPlanes {
    static constexpr int NO = W >= 8 ? 4 : (W >= 4 ? 3 : 2);       // ones in [0, W]
    static constexpr int NK = NO + 1;                               // key = bit0, ones
    static constexpr int NS = W - 1 >= 4 ? 3 : (W - 1 >= 2 ? 2 : 1);  // popcount of W-1 bits
};

__device__ __forceinline__ void full_add(uint32_t a, uint32_t b, uint32_t c, uint32_t& s,
                                         uint32_t& cy) {
    s = lop3<0x96>(a, b, c);   // a ^ b ^ c
    cy = lop3<0xE8>(a, b, c);  // majority
}

// Bit-sliced population count of N planes (N <= 8) into planes o[0..].
template <int N, int NO>
__device__ __forceinline__ void popcount_planes(const uint32_t* x, uint32_t (&o)[NO]) {
#pragma unroll
    for (int i = 0; i < NO; ++i) o[i] = 0u;
    if constexpr (N == 1) {
        o[0] = x[0];
    } else if constexpr (N == 2) {
        o[0] = x[0] ^ x[1];
        o[1] = x[0] & x[1];
    } else if constexpr (N == 3) {
        full_add(x[0], x[1], x[2], o[0], o[1]);
    } else if constexpr (N == 4) {
        uint32_t s1, c1;
        full_add(x[0], x[1], x[2], s1, c1);
        o[0] = s1 ^ x[3];
        o[1] = lop3<0x78>(c1, s1, x[3]);  // c1 ^ (s1 & x3)
        o[2] = lop3<0x80>(c1, s1, x[3]);  // c1 & s1 & x3
    } else if constexpr (N == 5) {
        uint32_t s1, c1, c2;
        full_add(x[0], x[1], x[2], s1, c1);
        full_add(s1, x[3], x[4], o[0], c2);
        o[1] = c1 ^ c2;
        o[2] = c1 & c2;
    } else if constexpr (N == 6) {
        uint32_t s1, c1, s2, c2, k;
        full_add(x[0], x[1], x[2], s1, c1);
        full_add(x[3], x[4], x[5], s2, c2);
        o[0] = s1 ^ s2;
        k = s1 & s2;
        full_add(c1, c2, k, o[1], o[2]);
    } else if constexpr (N == 7) {
        uint32_t s1, c1, s2, c2, k;
        full_add(x[0], x[1], x[2], s1, c1);
        full_add(x[3], x[4], x[5], s2, c2);
        full_add(s1, s2, x[6], o[0], k);
        full_add(c1, c2, k, o[1], o[2]);
    } else {
        static_assert(N == 8, "widths 3..8");
        uint32_t s1, c1, s2, c2, s3, k1, k2, t1, u1, v;
        full_add(x[0], x[1], x[2], s1, c1);
        full_add(x[3], x[4], x[5], s2, c2);
        full_add(s1, s2, x[6], s3, k1);
        o[0] = s3 ^ x[7];
        k2 = s3 & x[7];
        full_add(c1, c2, k1, t1, u1);
        o[1] = t1 ^ k2;
        v = t1 & k2;
        o[2] = u1 ^ v;
        o[3] = u1 & v;
    }
}

template <int W>
struct CandW {
    uint32_t k[WPlanes<W>::NK];  // k[0] = slice bit 0, k[1..] = ones
    uint32_t s[W - 1];           // slice bits 1 .. W-1
};

// NOPN: the warp's groups are N-free (N-presence flags): no N loads, and a
// 2-LOP3 map word in interior blocks (fused.cuh, load_rel / map_word).
template <int W, bool CHECK, bool NOPN = false>
__device__ __forceinline__ void wsearch_block(const uint32_t* __restrict__ tbase,
                                              const uint32_t* __restrict__ tnbase, int tcol0,
                                              const uint32_t* __restrict__ pbase,
                                              const uint32_t* __restrict__ pnbase, int pcol0,
                                              int m, int E, CandW<W> (&best)[4]) {
    constexpr int B = 4;
    constexpr int X = B + W - 1;
    constexpr int NK = WPlanes<W>::NK;
    constexpr int NO = WPlanes<W>::NO;
    uint32_t T[X][3];
#pragma unroll
    for (int x = 0; x < X; ++x) load_rel<CHECK, true, NOPN>(tbase, tnbase, x, tcol0, m, T[x]);
    uint32_t P[X][3];
#pragma unroll
    for (int x = 0; x < X; ++x) load_rel<CHECK, true, NOPN>(pbase, pnbase, x, pcol0, m, P[x]);
    auto step = [&](const int rot, bool first) {
        uint32_t sv[X];
#pragma unroll
        for (int x = 0; x < X; ++x) {
            sv[x] = map_word<NOPN && !CHECK>(P[(rot + x) % X], T[x]);
        }
#pragma unroll
        for (int b = 0; b < B; ++b) {
            CandW<W> cd;
            uint32_t ones[NO];
            popcount_planes<W, NO>(sv + b, ones);
            cd.k[0] = sv[b];
#pragma unroll
            for (int i = 0; i < NO; ++i) cd.k[i + 1] = ones[i];
#pragma unroll
            for (int i = 0; i < W - 1; ++i) cd.s[i] = sv[b + 1 + i];
            if (first) {
                best[b] = cd;
            } else {
                uint32_t lt = 0u;
#pragma unroll
                for (int i = 0; i < NK; ++i) lt = lop3<0x8E>(cd.k[i], best[b].k[i], lt);
#pragma unroll
                for (int i = 0; i < NK; ++i) best[b].k[i] = lop3<0xE4>(cd.k[i], best[b].k[i], lt);
#pragma unroll
                for (int i = 0; i < W - 1; ++i) best[b].s[i] = lop3<0xE4>(cd.s[i], best[b].s[i], lt);
            }
        }
    };
    step(0, true);  // d = -E
#pragma unroll 1
    for (int d0 = 1; d0 <= 2 * E; d0 += X) {
#pragma unroll
        for (int u = 0; u < X; ++u) {
            const int di = d0 + u;
            if (di > 2 * E) break;
            load_rel<CHECK, true, NOPN>(pbase, pnbase, di + X - 1, pcol0, m, P[u]);
            step((1 + u) % X, false);
        }
    }
}

// commit_window for width W as a state machine over S = bv[j .. j+W-2].
template <int W>
__device__ __forceinline__ uint32_t fsm_step_w(const CandW<W>& best, uint32_t (&S)[W - 1]) {
    constexpr int NO = WPlanes<W>::NO;
    constexpr int NS = WPlanes<W>::NS;
    uint32_t ps[NS];
    popcount_planes<W - 1, NS>(S, ps);
    uint32_t ones[NO];
#pragma unroll
    for (int i = 0; i < NO; ++i) ones[i] = best.k[i + 1];
    const uint32_t commit = ~bs_less(ps, ones);  // ones(best) <= popcount(S)
    const uint32_t out = lop3<0xE4>(best.k[0], S[0], commit);
#pragma unroll
    for (int i = 0; i < W - 2; ++i) S[i] = lop3<0xE4>(best.s[i], S[i + 1], commit);
    S[W - 2] = best.s[W - 2] | ~commit;
    return out;
}

// The whole sweep for group g (32 pairs): NB blocks of 4 windows.
// NOPN / zero / tzero / pzero: as search_group (fused.cuh).
template <int W, int NC, bool NOPN = false>
__device__ __forceinline__ void wsearch_group(const uint32_t* __restrict__ planes, long long g,
                                              long long n, int m, int E,
                                              uint32_t* __restrict__ accept,
                                              uint32_t* __restrict__ estimates,
                                              uint32_t* __restrict__ outplanes,
                                              const uint32_t* __restrict__ zero = nullptr,
                                              bool tzero = false, bool pzero = false) {
    constexpr int B = 4;
    constexpr int X = B + W - 1;
    const long long row0 = g * 32;
    if (row0 >= n) return;
    const long long ngroups = (n + 31) / 32;
    const long long nblocks = (n + kPackPairs - 1) / kPackPairs;
    const int mc = plane_cols(m);
    const uint32_t* const tb = planes + lohi_index(0, g, 0, 0, nblocks, mc);
    const uint32_t* const pb = planes + lohi_index(1, g, 0, 0, nblocks, mc);
    const uint32_t* const tnb = tzero ? zero + g % kPackGroups : planes + nplane_index(0, g, 0, nblocks, mc);
    const uint32_t* const pnb = pzero ? zero + g % kPackGroups : planes + nplane_index(1, g, 0, nblocks, mc);
    uint32_t S[W - 1];
#pragma unroll
    for (int i = 0; i < W - 1; ++i) S[i] = ~0u;  // bitvector bv(m, true) (shouji.cpp:52)
    uint32_t cnt[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) cnt[i] = 0u;
    const int NB = (m + B - 1) / B;
#pragma unroll 1
    for (int blk = 0; blk < NB; ++blk) {
        const int j0 = blk * B;
        const int pcol0 = j0 - E;
        const bool interior = pcol0 >= 0 && j0 + X + E <= m;
        const uint32_t* tbase = tb + static_cast<long long>(j0) * kLhColWords;
        const uint32_t* pbase = pb + static_cast<long long>(pcol0) * kLhColWords;
        const uint32_t* tnbase = tnb + static_cast<long long>(j0) * kNColWords;
        const uint32_t* pnbase = pnb + static_cast<long long>(pcol0) * kNColWords;
        CandW<W> best[B];
        if (interior)
            wsearch_block<W, false, NOPN>(tbase, tnbase, j0, pbase, pnbase, pcol0, m, E, best);
        else
            wsearch_block<W, true, NOPN>(tbase, tnbase, j0, pbase, pnbase, pcol0, m, E, best);
        uint32_t outs[B];
#pragma unroll
        for (int b = 0; b < B; ++b) {
            const int j = j0 + b;
            outs[b] = 0u;
            if (j < m) {
                outs[b] = fsm_step_w<W>(best[b], S);
                if (outplanes) outplanes[static_cast<long long>(j) * ngroups + g] = outs[b];
            }
        }
        uint32_t v[3];
        popcount_planes<4, 3>(outs, v);
        bs_add(cnt, v);
    }
    const long long valid = n - row0;
    const uint32_t vmask = valid >= 32 ? ~0u : ((1u << valid) - 1u);
    accept[g] = bs_le_const(cnt, static_cast<uint32_t>(E)) & vmask;
    if (estimates) {
#pragma unroll 1
        for (int b = 0; b < 32 && b < valid; ++b) {
            uint32_t est = 0;
#pragma unroll
            for (int i = 0; i < NC; ++i) est |= ((cnt[i] >> b) & 1u) << i;
            estimates[row0 + b] = est;
        }
    }
}

template <int W, int NC>
__global__ void __launch_bounds__(128)
shouji_wsearch(const uint32_t* __restrict__ planes, long long n, int m, int E,
               uint32_t* __restrict__ accept, uint32_t* __restrict__ estimates,
               uint32_t* __restrict__ outplanes, const uint32_t* __restrict__ nflags) {
    const long long g = static_cast<long long>(blockIdx.x) * 128 + threadIdx.x;
    if (nflags != nullptr) {  // as shouji_search_w4 (fused.cuh)
        const long long nblocks = (n + kPackPairs - 1) / kPackPairs;
        const bool live = g * 32 < n;
        const bool tz = !live || nflags[nflag_index(0, g, nblocks)] == 0u;
        const bool pz = !live || nflags[nflag_index(1, g, nblocks)] == 0u;
        if (__all_sync(~0u, tz && pz)) {
            wsearch_group<W, NC, true>(planes, g, n, m, E, accept, estimates, outplanes);
            return;
        }
        wsearch_group<W, NC, false>(planes, g, n, m, E, accept, estimates, outplanes,
                                    nflags + nflag_words(n), tz, pz);
        return;
    }
    wsearch_group<W, NC>(planes, g, n, m, E, accept, estimates, outplanes);
}

}  // namespace sb
