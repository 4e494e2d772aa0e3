// Fused width-4 Shouji kernel, specialised on the edit threshold E.
//
// Reference: shouji_filter (proj/src/shouji.cpp:41-58): build the 2E+1
// diagonal mismatch vectors (neighborhood.cpp:41-79), then for j = 0..m-1
// select_window (shouji.cpp:17-31) and commit_window (shouji.cpp:33-39), and
// finally accept iff popcount(bv) <= E (shouji.cpp:56-57).
//
// One thread owns one group of 32 consecutive pairs and reads the group's
// pair-sliced planes (written by the pack kernel, pack.cuh) column by column.
// Per block of four windows:
//   * the diagonal loop d = -E..+E is fully unrolled and scanned in reference
//     order; each new pattern column is one load per plane (8 threads share
//     one fully used 32-byte sector), kept in a sliding register window;
//   * D_d for the block's columns is (Plo^Tlo)|(Phi^Thi)|PN|TN;
//   * the window key is 2*ones + bit0 (windows 0,1 and 2,3 of a block share
//     the popcount of their three common columns) and the winner is the strict first
//     minimum — exactly select_window's "more zeros, or equal zeros and a
//     leading zero replacing a leading one" rule;
//   * commit_window becomes a 3-bit state machine (fsm_step4): bit j+3 is
//     always still 1 when window j is examined, so "strictly more zeros than
//     the incumbent" is ones(best) <= popcount(bv[j..j+2]).
//   * the final tally bits are summed in a bit-sliced counter; accept and the
//     estimate fall out of it.
// CARRY (E <= 12): the last three D columns of each diagonal are carried to
// the next block in registers (3 new map words per window and diagonal).
// Otherwise D is rebuilt over the block's 7 columns (fewer registers).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "bitslice.cuh"
#include "kernels.cuh"
#include "pack.cuh"
#include "pack_tile.cuh"
#include "phase_a.cuh"

namespace sb {

// A window's candidate. select_window orders candidates by key = 2*ones + s0
// (more zeros first, then a leading zero); only 8 (ones, s0) combinations
// exist — ones = 0 forces s0 = 0 and ones = 4 forces s0 = 1 — so the key is
// held as its 3-bit rank among them:
//   (ones, s0): (0,0) (1,0) (1,1) (2,0) (2,1) (3,0) (3,1) (4,1)
//   rank:         0     1     2     3     4     5     6     7
// which keeps the order (strict first minimum of the rank == of the key) with
// one plane less to compare and select. The slice is (s0, s1, s2, s3): s0
// and the parity of ones decode from the rank, s1 and s2 are carried, and s3
// is implied by the parity — all recovered once per window at commit.
struct Cand4 {
    uint32_t r[3];  // rank planes, LSB first
    uint32_t s[2];  // slice bits 1..2
};

// The four windows of a block over D columns sv[0..6] (window b = sv[b..b+3]).
// Window b's rank from s0 = sv[b] and u = sv[b+1] + sv[b+2] + sv[b+3]
// (u0 = xor, u1 = majority):
//   s0 = 0: rank = 2u - [u >= 1]   -> r0 = u1|u0, r1 = u1&~u0, r2 = u1&u0
//   s0 = 1: rank = 2u + 2 - [u==3] -> r0 = u1&u0, r1 = u1|~u0, r2 = u1|u0
// i.e. one LOP3 per rank plane: 5 LOP3 per window.
__device__ __forceinline__ void make_block_cands(const uint32_t (&sv)[7], Cand4 (&cd)[4]) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const uint32_t a = sv[b + 1], c = sv[b + 2], d = sv[b + 3];
        const uint32_t u0 = lop3<0x96>(a, c, d);  // a ^ c ^ d
        const uint32_t u1 = lop3<0xE8>(a, c, d);  // majority
        cd[b].r[0] = lop3<0x8E>(sv[b], u1, u0);  // s0 ? u1&u0 : u1|u0
        cd[b].r[1] = lop3<0xD4>(sv[b], u1, u0);  // s0 ? u1|~u0 : u1&~u0
        cd[b].r[2] = lop3<0xE8>(sv[b], u1, u0);  // s0 ? u1|u0 : u1&u0 (majority)
        cd[b].s[0] = a;
        cd[b].s[1] = c;
    }
}

// best = c if rank(c) < rank(best): 3 LOP3 for the strict compare (LSB first:
// lt = ~c&b | ~(c^b)&lt, table 0x8E) and 5 for the select (lt ? c : best,
// table 0xE4) — 8 per candidate, pinned with explicit lop3.
__device__ __forceinline__ void update_best4(const Cand4& c, Cand4& best) {
    uint32_t lt = lop3<0x8E>(c.r[0], best.r[0], 0u);
    lt = lop3<0x8E>(c.r[1], best.r[1], lt);
    lt = lop3<0x8E>(c.r[2], best.r[2], lt);
#pragma unroll
    for (int i = 0; i < 3; ++i) best.r[i] = lop3<0xE4>(c.r[i], best.r[i], lt);
#pragma unroll
    for (int i = 0; i < 2; ++i) best.s[i] = lop3<0xE4>(c.s[i], best.s[i], lt);
}

// commit_window as a state machine over S = tally bits (j, j+1, j+2). Bit j+3
// is still 1, so "more zeros than the incumbent" is ones(best) <= p with
// p = S0+S1+S2, i.e. rank(best) <= 2p (the largest rank with ones = p).
__device__ __forceinline__ uint32_t fsm_step4(const Cand4& best, uint32_t (&S)[3]) {
    const uint32_t r0 = best.r[0], r1 = best.r[1], r2 = best.r[2];
    const uint32_t s0 = lop3<0xD4>(r2, r1, r0);          // rank in {2,4,6,7}
    const uint32_t g = lop3<0xB2>(r2, r1, r0);           // parity(ones) ^ s0 = r0^r1^s0
    const uint32_t s3 = lop3<0x96>(g, best.s[0], best.s[1]);
    const uint32_t p0 = lop3<0x96>(S[0], S[1], S[2]);
    const uint32_t p1 = lop3<0xE8>(S[0], S[1], S[2]);
    const uint32_t le1 = lop3<0x4D>(r1, p0, r0);          // (r1 r0) <= (p0 0)
    const uint32_t commit = lop3<0x8E>(r2, p1, le1);      // (r2 r1 r0) <= (p1 p0 0)
    const uint32_t out = lop3<0xE4>(s0, S[0], commit);
    S[0] = lop3<0xE4>(best.s[0], S[1], commit);
    S[1] = lop3<0xE4>(best.s[1], S[2], commit);
    S[2] = s3 | ~commit;
    return out;
}

template <int E>
struct SearchCfg {
    // measured: the carried form at 8 <= E <= 12 beats the rebuilding form
    // (4 CTAs/SM) by 3-6% despite its register pressure
    static constexpr bool CARRY = E <= 12;
    static constexpr int B = 4;  // windows per block
    static constexpr int NT = 128;
    // 4 CTAs (16 warps) per SM where the carried D columns still fit 128
    // registers without spilling (E <= 7); 3 CTAs for 8 <= E <= 12 (168
    // registers instead of 190-242 at 2 CTAs: +2-3.5%; 4 CTAs spill and lose);
    // the rebuilding form (E > 12) fits 4 CTAs on its own.
    static constexpr int MINB = E <= 7 ? 4 : (E <= 12 ? 3 : 1);
};

// Column loads relative to per-block base pointers: lo/hi word (x*2 + k) * 8
// of base and N word x * 8 of nbase (pack.cuh layout), x counted from the
// block's first column `col0`. CHECK: the block touches columns outside
// [0, m), which read as N.
// NC: the planes are read-only while the search kernel runs (the pack kernel
// wrote them in an earlier launch), so the non-coherent path may serve them.
// NOPN: the warp's groups are all N-free (N-presence flags, pack.cuh): the N
// word is 0 and never loaded. (An N-free group in a mixed warp reads an
// all-zero column image through nbase instead.)
template <bool CHECK, bool NC = true, bool NOPN = false>
__device__ __forceinline__ void load_rel(const uint32_t* __restrict__ base,
                                         const uint32_t* __restrict__ nbase, int x, int col0, int m,
                                         uint32_t (&v)[3]) {
    if (!CHECK || static_cast<unsigned>(col0 + x) < static_cast<unsigned>(m)) {
        if constexpr (NC) {
            v[0] = __ldg(base + (x * 2 + 0) * kPackGroups);
            v[1] = __ldg(base + (x * 2 + 1) * kPackGroups);
            v[2] = NOPN ? 0u : __ldg(nbase + x * kNColWords);
        } else {
            v[0] = base[(x * 2 + 0) * kPackGroups];
            v[1] = base[(x * 2 + 1) * kPackGroups];
            v[2] = NOPN ? 0u : nbase[x * kNColWords];
        }
    } else {
        v[0] = 0u;
        v[1] = 0u;
        v[2] = ~0u;
    }
}

__device__ __forceinline__ void prefetch_l1(const uint32_t* p) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// One mismatch-map word D = !bases_match for a (pattern, text) column pair.
// FAST: both N words are known zero (N-free warp, interior block): 2 LOP3.
template <bool FAST>
__device__ __forceinline__ uint32_t map_word(const uint32_t (&p)[3], const uint32_t (&t)[3]) {
    if constexpr (FAST)
        return (p[0] ^ t[0]) | (p[1] ^ t[1]);
    else
        return (p[0] ^ t[0]) | (p[1] ^ t[1]) | p[2] | t[2];
}

// Best candidate of each window of one block (windows j0 .. j0+B-1).
// tcol0/pcol0: first text / pattern column the block reads; tbase/pbase point
// at those columns (pointers may be out of range when CHECK masks the load).
template <int E, bool CHECK, bool NC, bool NOPN = false>
__device__ __forceinline__ void search_block(const uint32_t* __restrict__ tbase,
                                             const uint32_t* __restrict__ tnbase, int tcol0,
                                             const uint32_t* __restrict__ pbase,
                                             const uint32_t* __restrict__ pnbase, int pcol0, int m,
                                             uint32_t (*Dc)[3], Cand4 (&best)[SearchCfg<E>::B]) {
    constexpr int B = SearchCfg<E>::B;
    constexpr bool FAST = NOPN && !CHECK;
    if constexpr (SearchCfg<E>::CARRY) {
        // new D columns tcol0 .. tcol0+B-1; pattern column = that + d, pcol0 = tcol0 - E
        uint32_t T[B][3];
#pragma unroll
        for (int b = 0; b < B; ++b) load_rel<CHECK, NC, NOPN>(tbase, tnbase, b, tcol0, m, T[b]);
        uint32_t P[B][3];
#pragma unroll
        for (int di = 0; di <= 2 * E; ++di) {
            if (di == 0) {
#pragma unroll
                for (int b = 0; b < B; ++b) load_rel<CHECK, NC, NOPN>(pbase, pnbase, b, pcol0, m, P[b]);
            } else {
#pragma unroll
                for (int b = 0; b < B - 1; ++b) {
                    P[b][0] = P[b + 1][0];
                    P[b][1] = P[b + 1][1];
                    P[b][2] = P[b + 1][2];
                }
                load_rel<CHECK, NC, NOPN>(pbase, pnbase, B - 1 + di, pcol0, m, P[B - 1]);
            }
            uint32_t s[B + 3];
            s[0] = Dc[di][0];
            s[1] = Dc[di][1];
            s[2] = Dc[di][2];
#pragma unroll
            for (int b = 0; b < B; ++b)
                s[3 + b] = map_word<FAST>(P[b], T[b]);
            Cand4 cd[B];
            make_block_cands(s, cd);
#pragma unroll
            for (int b = 0; b < B; ++b) {
                if (di == 0)
                    best[b] = cd[b];
                else
                    update_best4(cd[b], best[b]);
            }
            Dc[di][0] = s[B];
            Dc[di][1] = s[B + 1];
            Dc[di][2] = s[B + 2];
        }
    } else {
        // D over columns tcol0 .. tcol0+B+2 rebuilt per block, pcol0 = tcol0 - E.
        // The pattern columns of diagonal di are pcol0+di .. pcol0+di+X-1, held in
        // a register ring: column pcol0+c sits in slot c % X. The diagonal loop
        // runs in rolled chunks of X fully unrolled steps (slot indices stay
        // compile-time, no register shuffling), so large E does not unroll into
        // hundreds of hoisted loads.
        constexpr int X = B + 3;
        uint32_t T[X][3];
#pragma unroll
        for (int x = 0; x < X; ++x) load_rel<CHECK, NC, NOPN>(tbase, tnbase, x, tcol0, m, T[x]);
        uint32_t P[X][3];
#pragma unroll
        for (int x = 0; x < X; ++x) load_rel<CHECK, NC, NOPN>(pbase, pnbase, x, pcol0, m, P[x]);
        auto step = [&](const int rot, bool first) {
            // rot = di % X: slot of pattern column pcol0 + di + x is (rot + x) % X
            uint32_t sv[X];
#pragma unroll
            for (int x = 0; x < X; ++x) {
                sv[x] = map_word<FAST>(P[(rot + x) % X], T[x]);
            }
            Cand4 cd[B];
            make_block_cands(sv, cd);
#pragma unroll
            for (int b = 0; b < B; ++b) {
                if (first)
                    best[b] = cd[b];
                else
                    update_best4(cd[b], best[b]);
            }
        };
        step(0, true);  // di = 0
#pragma unroll 1
        for (int d0 = 1; d0 <= 2 * E; d0 += X) {
#pragma unroll
            for (int u = 0; u < X; ++u) {
                const int di = d0 + u;
                if (di > 2 * E) break;
                // new column pcol0 + di + X - 1 replaces pcol0 + di - 1 in slot (di - 1) % X = u
                load_rel<CHECK, NC, NOPN>(pbase, pnbase, di + X - 1, pcol0, m, P[u]);
                step((1 + u) % X, false);
            }
        }
    }
}

// The commit chain over one block's windows (column order) and the tally
// counter update: fsm_step4 per window, then the block's 4 tally bits are
// added to the bit-sliced estimate counter.
template <int B, int NC>
__device__ __forceinline__ void commit_block(const Cand4 (&best)[B], uint32_t (&S)[3], int j0,
                                             int m, long long g, long long ngroups,
                                             uint32_t* __restrict__ outplanes,
                                             uint32_t (&cnt)[NC]) {
    static_assert(B == 4, "the tally adder below is written for 4 windows per block");
    uint32_t outs[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
        const int j = j0 + b;
        outs[b] = 0u;
        if (j >= 0 && j < m) {
            outs[b] = fsm_step4(best[b], S);
            if (outplanes) outplanes[static_cast<long long>(j) * ngroups + g] = outs[b];
        }
    }
    uint32_t v[3];
    const uint32_t s1 = outs[0] ^ outs[1] ^ outs[2];
    const uint32_t c1 = (outs[0] & outs[1]) | (outs[0] & outs[2]) | (outs[1] & outs[2]);
    v[0] = s1 ^ outs[3];
    v[1] = c1 ^ (s1 & outs[3]);
    v[2] = c1 & s1 & outs[3];
    bs_add(cnt, v);
}

// accept = ones <= e (shouji.cpp:56-57); bits of pairs past n are 0.
template <int E, int NC>
__device__ __forceinline__ void finish_group(const uint32_t (&cnt)[NC], long long row0, long long n,
                                             long long g, uint32_t* __restrict__ accept,
                                             uint32_t* __restrict__ estimates) {
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

// The whole Shouji sweep for group g (32 pairs) from its planes.
// NC: bit planes of the estimate counter (8: m <= 255, 12: m <= 4095).
// NOPN: see load_rel. tzero / pzero: the group's text / pattern N planes are
// not stored (N-presence flags): read the all-zero column image `zero` instead.
template <int E, bool NCLOAD, int NC = 8, bool NOPN = false>
__device__ __forceinline__ void search_group(const uint32_t* __restrict__ planes, long long g,
                                             long long n, int m, uint32_t* __restrict__ accept,
                                             uint32_t* __restrict__ estimates,
                                             uint32_t* __restrict__ outplanes,
                                             const uint32_t* __restrict__ zero = nullptr,
                                             bool tzero = false, bool pzero = false) {
    using Cfg = SearchCfg<E>;
    constexpr int B = Cfg::B;
    constexpr bool CARRY = Cfg::CARRY;
    const long long row0 = g * 32;
    if (row0 >= n) return;
    const long long ngroups = (n + 31) / 32;
    const long long nblocks = (n + kPackPairs - 1) / kPackPairs;
    const int mc = plane_cols(m);
    const uint32_t* const tb = planes + lohi_index(0, g, 0, 0, nblocks, mc);
    const uint32_t* const pb = planes + lohi_index(1, g, 0, 0, nblocks, mc);
    const uint32_t* const tnb = tzero ? zero + g % kPackGroups : planes + nplane_index(0, g, 0, nblocks, mc);
    const uint32_t* const pnb = pzero ? zero + g % kPackGroups : planes + nplane_index(1, g, 0, nblocks, mc);

    constexpr int DCN = CARRY ? 2 * E + 1 : 1;
    uint32_t Dc[DCN][3];
#pragma unroll
    for (int di = 0; di < DCN; ++di) Dc[di][0] = Dc[di][1] = Dc[di][2] = ~0u;
    uint32_t S[3] = {~0u, ~0u, ~0u};  // bitvector bv(m, true) (shouji.cpp:52)
    uint32_t cnt[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) cnt[i] = 0u;

    // Block blk covers windows j0 = blk*B-3 .. j0+B-1. It reads text columns
    // [tcol0, tcol0 + TW) and pattern columns [tcol0 - E, tcol0 + TW + E).
    constexpr int TOFF = CARRY ? 3 : 0;   // tcol0 = j0 + TOFF
    constexpr int TW = CARRY ? B : B + 3;
    const int NB = (m + 3 + B - 1) / B;  // blocks: windows must reach m-1
#pragma unroll 1
    for (int blk = 0; blk < NB; ++blk) {
        const int j0 = blk * B - 3;
        const int tcol0 = j0 + TOFF;
        const int pcol0 = tcol0 - E;
        const bool interior = tcol0 >= 0 && pcol0 >= 0 && tcol0 + TW + E <= m;
        Cand4 best[B];
        // pointers may point outside the group's planes; CHECK masks those loads
        const uint32_t* tbase = tb + static_cast<long long>(tcol0) * kLhColWords;
        const uint32_t* pbase = pb + static_cast<long long>(pcol0) * kLhColWords;
        const uint32_t* tnbase = tnb + static_cast<long long>(tcol0) * kNColWords;
        const uint32_t* pnbase = pnb + static_cast<long long>(pcol0) * kNColWords;
#ifndef SB_PF_DIST
#define SB_PF_DIST 2
#endif
        if (blk + SB_PF_DIST < NB) {
            // pull the first-touch columns of block blk + SB_PF_DIST (text
            // tcol0+TW.., pattern pcol0+TW+2E.., 4 each, shifted by the distance)
            // towards the SM now: their loads then wait on L2 instead of DRAM
            // (lo/hi words of a column are 64 contiguous bytes of the pair block;
            // these 4 columns span <= 3 lines)
            const int nt = tcol0 + TW + B * (SB_PF_DIST - 1), np = pcol0 + TW + 2 * E + B * (SB_PF_DIST - 1);
            const uint32_t* tn = tb + static_cast<long long>(max(nt, 0)) * kLhColWords;
            const uint32_t* pn = pb + static_cast<long long>(max(np, 0)) * kLhColWords;
            if (nt + B <= m) {
                prefetch_l1(tn);
                prefetch_l1(tn + 2 * kLhColWords);
            }
            if (np + B <= m) {
                prefetch_l1(pn);
                prefetch_l1(pn + 2 * kLhColWords);
                prefetch_l1(pn + 3 * kLhColWords);
            }
        }
        if (interior)
            search_block<E, false, NCLOAD, NOPN>(tbase, tnbase, tcol0, pbase, pnbase, pcol0, m, Dc,
                                                 best);
        else
            search_block<E, true, NCLOAD, NOPN>(tbase, tnbase, tcol0, pbase, pnbase, pcol0, m, Dc,
                                                best);
        commit_block(best, S, j0, m, g, ngroups, outplanes, cnt);
    }
    finish_group<E>(cnt, row0, n, g, accept, estimates);
}

// ---- prefetching form (CARRY, used for 8 <= E <= 12) ---------------------------
// The same sweep, but the planes a block needs arrive one block ahead with
// cp.async into a per-thread shared-memory region: a double-buffered text
// slot (4 columns x 3 planes) and a pattern ring of R = 2E+8 columns (block
// blk reads pattern columns [4blk-E, 4blk+4+E) while the 4 columns of block
// blk+1 stream in). Each pattern column is fetched once (the direct form
// reloads it (4+2E)/4 times from L1/L2) and the search reads shared memory
// (~30-cycle latency) instead of waiting on global loads. Columns outside
// [0, m) are written as N planes directly, so the search needs no bounds
// checks. Per-thread regions have an odd word stride: the 32 lanes of a warp
// reading the same offset hit 32 banks.
__device__ __forceinline__ void cp_async4(uint32_t* dst, const uint32_t* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait1() {
    asm volatile("cp.async.wait_group 1;" ::: "memory");
}

template <int E>
struct PfCfg {
    static constexpr int R = 2 * E + 8;            // pattern ring columns
    static constexpr int TEXT = 0;                 // [2][4][3] words
    static constexpr int RING = 24;                // [R][3] words
    static constexpr int WORDS = (24 + 3 * R) | 1;  // per-thread stride (odd)
};

// Column `col` of sequence planes `base` (the group's plane words, pack.cuh
// layout) into dst[0..2]: cp.async in range, N planes outside.
__device__ __forceinline__ void fetch_col(uint32_t* dst, const uint32_t* __restrict__ base,
                                          const uint32_t* __restrict__ nbase, int col, int m) {
    if (static_cast<unsigned>(col) < static_cast<unsigned>(m)) {
        const uint32_t* src = base + static_cast<long long>(col) * kLhColWords;
        cp_async4(dst + 0, src);
        cp_async4(dst + 1, src + kPackGroups);
        cp_async4(dst + 2, nbase + static_cast<long long>(col) * kNColWords);
    } else {
        dst[0] = 0u;
        dst[1] = 0u;
        dst[2] = ~0u;
    }
}

template <int E, int NC = 8>
__device__ __forceinline__ void search_group_pf(const uint32_t* __restrict__ planes, long long g,
                                                long long n, int m, uint32_t* __restrict__ accept,
                                                uint32_t* __restrict__ estimates,
                                                uint32_t* __restrict__ outplanes,
                                                uint32_t* __restrict__ region) {
    using P = PfCfg<E>;
    constexpr int B = 4;
    constexpr int R = P::R;
    const long long row0 = g * 32;
    const long long ngroups = (n + 31) / 32;
    const long long nblocks = (n + kPackPairs - 1) / kPackPairs;
    const int mc = plane_cols(m);
    const bool live = row0 < n;
    // dead threads still walk the blocks (uniform cp.async groups), on group 0's planes
    const long long gg = live ? g : 0;
    const uint32_t* const tb = planes + lohi_index(0, gg, 0, 0, nblocks, mc);
    const uint32_t* const pb = planes + lohi_index(1, gg, 0, 0, nblocks, mc);
    const uint32_t* const tnb = planes + nplane_index(0, gg, 0, nblocks, mc);
    const uint32_t* const pnb = planes + nplane_index(1, gg, 0, nblocks, mc);
    uint32_t* const text = region + P::TEXT;
    uint32_t* const ring = region + P::RING;
    auto ring_slot = [&](int col) { return ring + ((col + E) % R) * 3; };

    uint32_t Dc[2 * E + 1][3];
#pragma unroll
    for (int di = 0; di <= 2 * E; ++di) Dc[di][0] = Dc[di][1] = Dc[di][2] = ~0u;
    uint32_t S[3] = {~0u, ~0u, ~0u};
    uint32_t cnt[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) cnt[i] = 0u;

    const int NB = (m + 3 + B - 1) / B;
    // prologue: block 0 (text columns 0..3, pattern columns [-E, 4+E))
#pragma unroll
    for (int b = 0; b < B; ++b) fetch_col(text + b * 3, tb, tnb, b, m);
#pragma unroll 1
    for (int c = -E; c < B + E; ++c) fetch_col(ring_slot(c), pb, pnb, c, m);
    cp_async_commit();
#pragma unroll 1
    for (int blk = 0; blk < NB; ++blk) {
        const int tcol0 = B * blk;
        if (blk + 1 < NB) {
            uint32_t* tn = text + ((blk + 1) & 1) * 12;
#pragma unroll
            for (int b = 0; b < B; ++b) fetch_col(tn + b * 3, tb, tnb, tcol0 + B + b, m);
#pragma unroll
            for (int b = 0; b < B; ++b) {
                const int c = tcol0 + B + E + b;
                fetch_col(ring_slot(c), pb, pnb, c, m);
            }
        }
        cp_async_commit();
        cp_async_wait1();  // block blk's columns have landed
        const uint32_t* tc = text + (blk & 1) * 12;
        uint32_t T[B][3];
#pragma unroll
        for (int b = 0; b < B; ++b) {
            T[b][0] = tc[b * 3 + 0];
            T[b][1] = tc[b * 3 + 1];
            T[b][2] = tc[b * 3 + 2];
        }
        // pattern column tcol0 - E + x lives in ring slot (tcol0 + x) % R
        const int base = tcol0 % R;
        const int split = R - base;  // x >= split wraps to the ring's start
        const uint32_t* lo = ring + base * 3;
        const uint32_t* hi = ring + (base - R) * 3;
        auto pcol = [&](int x, uint32_t (&v)[3]) {
            const uint32_t* q = (x < split ? lo : hi) + x * 3;
            v[0] = q[0];
            v[1] = q[1];
            v[2] = q[2];
        };
        Cand4 best[B];
        uint32_t P4[B][3];
#pragma unroll
        for (int di = 0; di <= 2 * E; ++di) {
            if (di == 0) {
#pragma unroll
                for (int b = 0; b < B; ++b) pcol(b, P4[b]);
            } else {
#pragma unroll
                for (int b = 0; b < B - 1; ++b) {
                    P4[b][0] = P4[b + 1][0];
                    P4[b][1] = P4[b + 1][1];
                    P4[b][2] = P4[b + 1][2];
                }
                pcol(B - 1 + di, P4[B - 1]);
            }
            uint32_t sv[B + 3];
            sv[0] = Dc[di][0];
            sv[1] = Dc[di][1];
            sv[2] = Dc[di][2];
#pragma unroll
            for (int b = 0; b < B; ++b)
                sv[3 + b] = (P4[b][0] ^ T[b][0]) | (P4[b][1] ^ T[b][1]) | P4[b][2] | T[b][2];
            Cand4 cd[B];
            make_block_cands(sv, cd);
#pragma unroll
            for (int b = 0; b < B; ++b) {
                if (di == 0)
                    best[b] = cd[b];
                else
                    update_best4(cd[b], best[b]);
            }
            Dc[di][0] = sv[B];
            Dc[di][1] = sv[B + 1];
            Dc[di][2] = sv[B + 2];
        }
        commit_block(best, S, tcol0 - 3, m, g, ngroups, live ? outplanes : nullptr, cnt);
    }
    if (live) finish_group<E>(cnt, row0, n, g, accept, estimates);
}

template <int E, int NC>
__global__ void __launch_bounds__(SearchCfg<E>::NT, SearchCfg<E>::MINB)
shouji_search_w4_pf(const uint32_t* __restrict__ planes, long long n, int m,
                    uint32_t* __restrict__ accept, uint32_t* __restrict__ estimates,
                    uint32_t* __restrict__ outplanes) {
    extern __shared__ uint32_t pf_smem[];
    const long long g = static_cast<long long>(blockIdx.x) * SearchCfg<E>::NT + threadIdx.x;
    search_group_pf<E, NC>(planes, g, n, m, accept, estimates, outplanes,
                           pf_smem + threadIdx.x * PfCfg<E>::WORDS);
}

bool search_prefetch_enabled();

// nflags: N-presence flags (pack.cuh) or null. A warp whose 32 groups are all
// N-free (the usual case) runs the N-free instantiation: no N-plane loads and
// a 2-LOP3 mismatch map in interior blocks; in a mixed warp the N-free groups
// read the all-zero column image after the flags.
template <int E, int NC>
__global__ void __launch_bounds__(SearchCfg<E>::NT, SearchCfg<E>::MINB)
shouji_search_w4(const uint32_t* __restrict__ planes, long long n, int m,
                 uint32_t* __restrict__ accept, uint32_t* __restrict__ estimates,
                 uint32_t* __restrict__ outplanes, const uint32_t* __restrict__ nflags) {
    const long long g = static_cast<long long>(blockIdx.x) * SearchCfg<E>::NT + threadIdx.x;
    if (nflags != nullptr) {
        const long long nblocks = (n + kPackPairs - 1) / kPackPairs;
        const bool live = g * 32 < n;
        const bool tz = !live || nflags[nflag_index(0, g, nblocks)] == 0u;
        const bool pz = !live || nflags[nflag_index(1, g, nblocks)] == 0u;
        if (__all_sync(~0u, tz && pz)) {
            search_group<E, true, NC, true>(planes, g, n, m, accept, estimates, outplanes);
            return;
        }
        search_group<E, true, NC, false>(planes, g, n, m, accept, estimates, outplanes,
                                         nflags + nflag_words(n), tz, pz);
        return;
    }
    search_group<E, true, NC, false>(planes, g, n, m, accept, estimates, outplanes);
}

template <int E, int NC>
cudaError_t launch_search_nc(const FilterArgs& a, cudaStream_t s) {
    using Cfg = SearchCfg<E>;
    const long long ngroups = (a.n + 31) / 32;
    const unsigned grid = static_cast<unsigned>((ngroups + Cfg::NT - 1) / Cfg::NT);
    // measured on B200 (tools/exp_e_sweep.py, m=100): the prefetching form wins
    // from E = 8 (+5%) to E = 12 (+7% at E = 10), ties at E = 7 and loses below
    // (its per-block fetch bookkeeping outweighs the hidden latency when there
    // are few diagonals)
    if constexpr (Cfg::CARRY && E >= 8) {
        if (search_prefetch_enabled() && a.nflags == nullptr) {
            const size_t smem = static_cast<size_t>(Cfg::NT) * PfCfg<E>::WORDS * 4;
            const cudaError_t st =
                ensure_smem_attr<shouji_search_w4_pf<E, NC>>(static_cast<int>(smem));
            if (st != cudaSuccess) return st;
            shouji_search_w4_pf<E, NC><<<grid, Cfg::NT, smem, s>>>(a.planes, a.n, a.m, a.accept,
                                                                  a.estimates, a.outplanes);
            count_launch();
            return cudaGetLastError();
        }
    }
    shouji_search_w4<E, NC><<<grid, Cfg::NT, 0, s>>>(a.planes, a.n, a.m, a.accept, a.estimates,
                                                      a.outplanes, a.nflags);
    count_launch();
    return cudaGetLastError();
}

// The counter width follows m: 8 planes up to m = 255 (the common case, fewer
// live registers), 12 planes up to 4095.
template <int E>
cudaError_t launch_search_e(const FilterArgs& a, cudaStream_t s) {
    return a.m <= 255 ? launch_search_nc<E, 8>(a, s) : launch_search_nc<E, 12>(a, s);
}

}  // namespace sb

// Explicit instantiation helper for the fused_e*.cu units.
#define SB_INSTANTIATE_FUSED(E)                                                      \
    template cudaError_t sb::launch_search_e<E>(const sb::FilterArgs&, cudaStream_t);
