// Phase A of the pair-sliced Shouji kernels: ASCII records -> bit planes.
//
// Reference: packed_sequence::from_string (proj/src/packed_sequence.cpp:7-34)
// packs A/C/G/T into two code planes plus an N plane and throws on any other
// byte. Here one thread converts a 16-column x 32-pair tile of one sequence
// into 16 column words per plane, where bit b of a column word belongs to
// pair row0+b ("pair-sliced" layout).
//
// Encoding: ASCII bits 1/2/3 of A,C,G,T,N are (lo,hi,N) = 000,100,110,010,111.
// A,C,G,T get distinct (bit1,bit2) codes and only N sets bit 3, so
//   mismatch = (Plo^Tlo) | (Phi^Thi) | PN | TN
// is exactly !bases_match (packed_sequence.hpp:58-61; N matches nothing,
// itself included). Columns outside [0, m) are forced to N: that realises both
// boundary rules of the reference — a pattern index outside [0,m) is a
// mismatch (neighborhood.cpp:71-76) and window reads past the text read as 1
// (bitvector.hpp:88-91) — with no special cases in phase B.
//
// Validation is exact and costs no extra pass: a byte is in {A,C,G,T,N} iff
// bits 7..5 are 010 and, given (b3,b2,b1) in {000,001,011,010,111},
// b0 == ~b3&(~b2|b1) and b4 == b2&~b1&~b3. gather_chunk_smem (the shared-memory
// tile path) checks all eight bits on its transposed bit planes; gather_chunk
// (global-memory path) checks bits 7..5 with OR/AND accumulators over the
// loaded words and bits 0..4 on its gathered planes. Any failure only raises a
// flag; the host then runs a locator kernel for the reference's exact error
// (lowest pair, text before pattern, lowest position).
#pragma once
#include <cstdint>

#include "bitslice.cuh"

namespace sb {

constexpr int CH = 16;  // columns per chunk (one 128-bit load per row)

// Compile-time rotate for mask constants (s may be negative).
__host__ __device__ constexpr uint32_t crotl(uint32_t x, int s) {
    return ((s % 32) + 32) % 32 == 0
               ? x
               : (x << (((s % 32) + 32) % 32)) | (x >> (32 - ((s % 32) + 32) % 32));
}

// Load 16 bytes of a record row: one 128-bit load when rows are 16-byte
// aligned, four 32-bit loads when they are only 4-byte aligned (pitch % 4).
template <int ALIGN>
__device__ __forceinline__ uint4 load_row16(const uint8_t* p) {
    if constexpr (ALIGN == 16) {
        return *reinterpret_cast<const uint4*>(p);
    } else {
        const uint32_t* q = reinterpret_cast<const uint32_t*>(p);
        return make_uint4(q[0], q[1], q[2], q[3]);
    }
}

// The same for the chunk straddling m: only the row's own words (byte offset <
// pitch) are loaded — the last record's bytes past its pitch may be past the end
// of the caller's array — and the rest read as "AAAA" (masked off anyway).
__device__ __forceinline__ uint4 load_row16_lim(const uint8_t* p, int nwords) {
    const uint32_t* q = reinterpret_cast<const uint32_t*>(p);
    return make_uint4(nwords > 0 ? q[0] : 0x41414141u, nwords > 1 ? q[1] : 0x41414141u,
                      nwords > 2 ? q[2] : 0x41414141u, nwords > 3 ? q[3] : 0x41414141u);
}

// Gather columns [col0, col0 + 4*NCG) of rows [row0, row0+32) into plane words:
// dst[(col*2 + k) * dstride], k = 0 lo, 1 hi, and ndst[col * dstride] (N). Returns nonzero on any
// illegal byte. EDGE: the chunk straddles m (bytes at columns >= m are
// ignored; only columns < m are stored). NCG: column groups of 4 processed
// (fewer than 4 only for the chunk straddling m). ALIGN: row alignment (16/4).
//
// Bit k of byte q of row i's word lands at bit 8q+i of the plane-k
// accumulator by a per-plane shift (left for i >= k, right otherwise) — a
// multiply or a high multiply, so the shifts issue on the FMA pipe and the
// ALU pipe only sees the masked ORs.
//
// DEFER_N: the N-plane words are not stored but returned in nout[0..4*NCG)
// (0 for columns >= m), for pack kernels that write them only for groups that
// hold an N (pack.cuh, N-presence flags).
template <bool EDGE, bool CHECK_ROWS = true, int NCG = 4, int ALIGN = 16, bool DEFER_N = false>
__device__ __forceinline__ uint32_t gather_chunk(const uint8_t* __restrict__ seq, size_t pitch,
                                                 long long row0, long long n, int col0, int m,
                                                 uint32_t* __restrict__ dst,
                                                 uint32_t* __restrict__ ndst, int dstride,
                                                 uint32_t* __restrict__ nout = nullptr) {
    uint32_t O[NCG][3][4];  // [column group][plane][column in group] -> column words
#pragma unroll
    for (int cg = 0; cg < NCG; ++cg)
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int q = 0; q < 4; ++q) O[cg][k][q] = 0u;
    uint32_t orr = 0u, andd = ~0u, err = 0u;
    uint32_t cm[NCG];
    // words of the row at/after col0 that lie within its pitch (EDGE loads only)
    const long long row_words = (static_cast<long long>(pitch) - col0) / 4;
    const int edge_words = row_words < 4 ? static_cast<int>(row_words) : 4;
    if (EDGE) {
#pragma unroll
        for (int cg = 0; cg < NCG; ++cg) {
            uint32_t mask = 0u;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (col0 + 4 * cg + q < m) mask |= 0xFFu << (8 * q);
            cm[cg] = mask;
        }
    }
    // Rows are consumed in groups of 8 (one byte lane of 8 pairs per column);
    // the loop stays rolled so at most 8 row loads are in flight per thread.
#pragma unroll 1
    for (int g8 = 0; g8 < 4; ++g8) {
        uint4 v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const long long row = row0 + 8 * g8 + i;
            if (!CHECK_ROWS || row < n)
                v[i] = EDGE ? load_row16_lim(seq + row * pitch + col0, edge_words)
                            : load_row16<ALIGN>(seq + row * pitch + col0);  // global or shared
            else
                v[i] = make_uint4(0x41414141u, 0x41414141u, 0x41414141u, 0x41414141u);
        }
        uint32_t acc[5][NCG];
#pragma unroll
        for (int k = 0; k < 5; ++k)
#pragma unroll
            for (int cg = 0; cg < NCG; ++cg) acc[k][cg] = 0u;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint32_t wv[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
            for (int cg = 0; cg < NCG; ++cg) {
                uint32_t w = wv[cg];
                if (EDGE) w = (w & cm[cg]) | (0x41414141u & ~cm[cg]);
                orr |= w;
                andd &= w;
#pragma unroll
                for (int k = 0; k < 5; ++k) {
                    const uint32_t u = i >= k ? w * (1u << (i - k)) : __umulhi(w, 1u << (32 - (k - i)));
                    acc[k][cg] |= u & (0x01010101u << i);
                }
            }
        }
#pragma unroll
        for (int cg = 0; cg < NCG; ++cg) {
            // bit (8q+i) of acc[k] = bit k of (row 8*g8+i, column 4cg+q)
            const uint32_t p0 = acc[0][cg], p1 = acc[1][cg], p2 = acc[2][cg];
            const uint32_t p3 = acc[3][cg], p4 = acc[4][cg];
            const uint32_t g0 = ~p3 & (~p2 | p1);
            const uint32_t gg4 = p2 & ~p1 & ~p3;
            err |= (p0 ^ g0) | (p4 ^ gg4) | (p3 & ~(p2 & p1));
            const uint32_t P[3] = {p1, p2, p3};
            // byte q of P (column 4cg+q, pairs 8g8..8g8+7) becomes byte g8 of the
            // column word: shift the word down one byte and insert at the top.
#pragma unroll
            for (int k = 0; k < 3; ++k)
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    O[cg][k][q] = __byte_perm(O[cg][k][q], P[k], 0x0321 | ((4 + q) << 12));
        }
    }
    err |= (orr & 0xA0A0A0A0u) | (~andd & 0x40404040u);
#pragma unroll
    for (int cg = 0; cg < NCG; ++cg)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int col = 4 * cg + q;
            if constexpr (DEFER_N) nout[col] = O[cg][2][q];  // columns >= m read as 'A': 0
            if (EDGE && col0 + col >= m) continue;  // never read: columns >= m are N
            dst[(col * 2 + 0) * dstride] = O[cg][0][q];
            dst[(col * 2 + 1) * dstride] = O[cg][1][q];
            if constexpr (!DEFER_N) ndst[col * dstride] = O[cg][2][q];
        }
    return err;
}

// 8x8 bit transpose inside every byte lane of w[0..7]: afterwards bit i of
// byte q of w[k] is bit k of byte q of the input w[i]. Three delta-swap stages
// (4-, 2-, 1-bit blocks); each pair exchange is two shifts, issued as a
// multiply / high multiply on the FMA pipe, and two LOP3 selects:
//   a' = (a & lo) | (b << S & ~lo),   b' = (a >> S & lo) | (b & ~lo).
// No bit crosses a byte: the masks keep only bits that moved inside it.
__device__ __forceinline__ void transpose8_bytes(uint32_t (&w)[8]) {
    auto xchg = [](uint32_t& a, uint32_t& b, uint32_t lo, int s) {
        const uint32_t x = b * (1u << s);               // b << s
        const uint32_t y = __umulhi(a, 1u << (32 - s));  // a >> s
        a = lop3<0xE4>(a, x, lo);                       // lo ? a : x
        b = lop3<0xE4>(y, b, lo);                       // lo ? y : b
    };
#pragma unroll
    for (int i = 0; i < 4; ++i) xchg(w[i], w[i + 4], 0x0F0F0F0Fu, 4);
    xchg(w[0], w[2], 0x33333333u, 2);
    xchg(w[1], w[3], 0x33333333u, 2);
    xchg(w[4], w[6], 0x33333333u, 2);
    xchg(w[5], w[7], 0x33333333u, 2);
#pragma unroll
    for (int i = 0; i < 8; i += 2) xchg(w[i], w[i + 1], 0x55555555u, 1);
}

// Bytes [4*mis, 4*mis + 4*NCG) of two 16-byte-aligned shared-memory chunks at
// p - 4*mis, i.e. the NCG words at p (mis = p's word offset past a 16-byte
// boundary, a compile-time constant once the caller's row loop is unrolled).
// One LDS.128 (two when the words straddle the boundary) instead of NCG
// LDS.32 that would hit only 8 distinct 16-byte bank groups per warp.
template <int NCG>
__device__ __forceinline__ void lds_words(const uint8_t* p, int mis, uint32_t (&x)[4]) {
    const uint4* a = reinterpret_cast<const uint4*>(p - 4 * mis);
    const uint4 c0 = a[0];
    uint32_t t[8] = {c0.x, c0.y, c0.z, c0.w, 0u, 0u, 0u, 0u};
    if (mis + NCG > 4) {
        const uint4 c1 = a[1];
        t[4] = c1.x;
        t[5] = c1.y;
        t[6] = c1.z;
        t[7] = c1.w;
    }
#pragma unroll
    for (int k = 0; k < NCG; ++k) x[k] = t[(mis + k) & 7];
}

// gather_chunk for records staged in shared memory (pack_one_tile): same
// contract as gather_chunk with CHECK_ROWS = false, rows 0..31 of seq. PM =
// (pitch / 4) % 4, so row i starts (i * PM) % 4 words past a 16-byte boundary
// (group bases and col0 are 16-byte aligned). Per 8 rows and 4 columns: one
// 8x8 byte-lane transpose (24 FMA + 24 LOP3) turns the 8 row words into the 8
// bit planes of the ASCII bytes; bits 1/2/3 are the lo/hi/N planes and all
// eight check the alphabet (7 LOP3, see the header).
// The gather itself: O[cg][k][q] = plane k (lo, hi, N) column word of column
// col0 + 4cg + q (columns >= m read as 'A' when EDGE); returns nonzero on an
// illegal byte. Shared by the store-to-planes form below and the select-in-pack
// kernel (select_pack.cu), which keeps the words in registers.
template <bool EDGE, int NCG, int PM>
__device__ __forceinline__ uint32_t gather_core_smem(const uint8_t* __restrict__ seq, size_t pitch,
                                                     int col0, int m, uint32_t (&O)[NCG][3][4]) {
#pragma unroll
    for (int cg = 0; cg < NCG; ++cg)
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int q = 0; q < 4; ++q) O[cg][k][q] = 0u;
    uint32_t err = 0u;
    uint32_t cm[NCG];
    if (EDGE) {
#pragma unroll
        for (int cg = 0; cg < NCG; ++cg) {
            uint32_t mask = 0u;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (col0 + 4 * cg + q < m) mask |= 0xFFu << (8 * q);
            cm[cg] = mask;
        }
    }
#pragma unroll 1
    for (int g8 = 0; g8 < 4; ++g8) {
        uint32_t v[8][4];
        const uint8_t* base = seq + static_cast<size_t>(8 * g8) * pitch + col0;
#pragma unroll
        for (int i = 0; i < 8; ++i) lds_words<NCG>(base + i * pitch, (i * PM) & 3, v[i]);
#pragma unroll
        for (int cg = 0; cg < NCG; ++cg) {
            uint32_t w[8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
                w[i] = EDGE ? lop3<0xE4>(v[i][cg], 0x41414141u, cm[cg]) : v[i][cg];
            transpose8_bytes(w);
            // bit i of byte q of w[k] = bit k of (row 8*g8+i, column 4cg+q)
            const uint32_t e0 = lop3<0xFB>(w[5], w[6], w[7]);   // b5 | ~b6 | b7
            const uint32_t t1 = lop3<0x51>(w[1], w[2], w[3]);   // ~b3 & (~b2 | b1)
            const uint32_t t2 = lop3<0x04>(w[1], w[2], w[3]);   // b2 & ~b1 & ~b3
            const uint32_t t3 = lop3<0x2A>(w[1], w[2], w[3]);   // b3 & ~(b2 & b1)
            const uint32_t r1 = lop3<0xBE>(w[0], t1, e0);       // (b0 ^ t1) | e0
            const uint32_t r2 = lop3<0xBE>(w[4], t2, r1);       // (b4 ^ t2) | r1
            err = lop3<0xFE>(err, r2, t3);
#pragma unroll
            for (int k = 0; k < 3; ++k)
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    O[cg][k][q] = __byte_perm(O[cg][k][q], w[k + 1], 0x0321 | ((4 + q) << 12));
        }
    }
    return err;
}

template <bool EDGE, int NCG, int PM, bool DEFER_N = false>
__device__ __forceinline__ uint32_t gather_chunk_smem(const uint8_t* __restrict__ seq, size_t pitch,
                                                      int col0, int m, uint32_t* __restrict__ dst,
                                                      uint32_t* __restrict__ ndst, int dstride,
                                                      uint32_t* __restrict__ nout = nullptr) {
    uint32_t O[NCG][3][4];
    const uint32_t err = gather_core_smem<EDGE, NCG, PM>(seq, pitch, col0, m, O);
#pragma unroll
    for (int cg = 0; cg < NCG; ++cg)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int col = 4 * cg + q;
            if constexpr (DEFER_N) nout[col] = O[cg][2][q];  // columns >= m read as 'A': 0
            if (EDGE && col0 + col >= m) continue;  // never read: columns >= m are N
            dst[(col * 2 + 0) * dstride] = O[cg][0][q];
            dst[(col * 2 + 1) * dstride] = O[cg][1][q];
            if constexpr (!DEFER_N) ndst[col * dstride] = O[cg][2][q];
        }
    return err;
}

// gather_chunk for nibble records (pack.cuh nibble format, validated on the
// host): a 16-column chunk is two words per row; column group cg (4 columns)
// is word cg/2, low nibbles for even cg, high nibbles for odd cg, so ASCII bit
// k of column 4cg+q sits at bit 8q + 4(cg&1) + k of the word and reaches bit
// 8q+i of the plane-k accumulator by one shift, as in gather_chunk.
template <bool EDGE, int NCG, bool DEFER_N = false>
__device__ __forceinline__ void gather_chunk_nib(const uint8_t* __restrict__ seq, size_t pitch,
                                                 int col0, int m, uint32_t* __restrict__ dst,
                                                 uint32_t* __restrict__ ndst, int dstride,
                                                 uint32_t* __restrict__ nout = nullptr) {
    constexpr int NW = (NCG + 1) / 2;
    uint32_t O[NCG][3][4];
#pragma unroll
    for (int cg = 0; cg < NCG; ++cg)
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int q = 0; q < 4; ++q) O[cg][k][q] = 0u;
#pragma unroll 1
    for (int g8 = 0; g8 < 4; ++g8) {
        uint32_t v[8][NW];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint32_t* q =
                reinterpret_cast<const uint32_t*>(seq + (8 * g8 + i) * pitch + col0 / 2);
#pragma unroll
            for (int w = 0; w < NW; ++w) v[i][w] = q[w];
        }
        uint32_t acc[3][NCG];
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int cg = 0; cg < NCG; ++cg) acc[k][cg] = 0u;
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int cg = 0; cg < NCG; ++cg) {
                const uint32_t w = v[i][cg / 2];
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const int s = i - (k + 1) - 4 * (cg & 1);
                    const uint32_t u = s >= 0 ? w * (1u << s) : __umulhi(w, 1u << (32 + s));
                    acc[k][cg] |= u & (0x01010101u << i);
                }
            }
#pragma unroll
        for (int cg = 0; cg < NCG; ++cg)
#pragma unroll
            for (int k = 0; k < 3; ++k)
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    O[cg][k][q] = __byte_perm(O[cg][k][q], acc[k][cg], 0x0321 | ((4 + q) << 12));
    }
#pragma unroll
    for (int cg = 0; cg < NCG; ++cg)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int col = 4 * cg + q;
            if constexpr (DEFER_N) nout[col] = O[cg][2][q];  // columns >= m are zero nibbles
            if (EDGE && col0 + col >= m) continue;
            dst[(col * 2 + 0) * dstride] = O[cg][0][q];
            dst[(col * 2 + 1) * dstride] = O[cg][1][q];
            if constexpr (!DEFER_N) ndst[col * dstride] = O[cg][2][q];
        }
}

// gather_chunk for dibit records (pack.cuh dibit format, validated by the
// host): a 16-column chunk is one word per row; column 4t+q of the chunk sits
// in byte q at bits 2t (lo) and 2t+1 (hi), so plane k of column group t
// reaches bit 8q+i of the accumulator by one shift. The N plane comes from the
// optional N-plane rows (bit c = column c); without them every column is
// N-free.
// SKIP_N (only without HAS_N): the all-zero N plane is not stored (the
// group's N-presence flag says so, pack.cuh).
template <bool EDGE, int NCG, bool HAS_N, bool SKIP_N = false>
__device__ __forceinline__ void gather_chunk_dib(const uint8_t* __restrict__ seq, size_t pitch,
                                                 const uint8_t* __restrict__ nseq, size_t npitch,
                                                 int col0, int m, uint32_t* __restrict__ dst,
                                                 uint32_t* __restrict__ ndst, int dstride) {
    static_assert(!(HAS_N && SKIP_N), "N planes with N data are always stored");
    uint32_t O[NCG][3][4];
#pragma unroll
    for (int cg = 0; cg < NCG; ++cg)
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int q = 0; q < 4; ++q) O[cg][k][q] = 0u;
#pragma unroll 1
    for (int g8 = 0; g8 < 4; ++g8) {
        uint32_t v[8], nv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            v[i] = *reinterpret_cast<const uint32_t*>(seq + (8 * g8 + i) * pitch + col0 / 4);
            if constexpr (HAS_N) {
                const uint32_t w = *reinterpret_cast<const uint32_t*>(
                    nseq + (8 * g8 + i) * npitch + (col0 / 32) * 4);
                nv[i] = w >> (col0 & 31);  // the chunk's 16 N bits at bits 0..15
            }
        }
        uint32_t acc[3][NCG];
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int cg = 0; cg < NCG; ++cg) acc[k][cg] = 0u;
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int cg = 0; cg < NCG; ++cg) {
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const int s = i - (2 * cg + k);
                    const uint32_t u =
                        s >= 0 ? v[i] * (1u << s) : __umulhi(v[i], 1u << (32 + s));
                    acc[k][cg] |= u & (0x01010101u << i);
                }
                if constexpr (HAS_N) {
                    // bits 4cg..4cg+3 of the N word -> bit 8q (x * (1 + 2^7 + 2^14 + 2^21)) -> 8q+i
                    const uint32_t x = (nv[i] >> (4 * cg)) & 0xFu;
                    acc[2][cg] |= ((x * 0x00204081u) & 0x01010101u) << i;
                }
            }
#pragma unroll
        for (int cg = 0; cg < NCG; ++cg)
#pragma unroll
            for (int k = 0; k < (HAS_N ? 3 : 2); ++k)
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    O[cg][k][q] = __byte_perm(O[cg][k][q], acc[k][cg], 0x0321 | ((4 + q) << 12));
    }
#pragma unroll
    for (int cg = 0; cg < NCG; ++cg)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int col = 4 * cg + q;
            if (EDGE && col0 + col >= m) continue;
            dst[(col * 2 + 0) * dstride] = O[cg][0][q];
            dst[(col * 2 + 1) * dstride] = O[cg][1][q];
            if constexpr (!SKIP_N) ndst[col * dstride] = O[cg][2][q];
        }
}

// A chunk entirely outside [0, m): every column is N.
__device__ __forceinline__ void fill_oob_chunk(uint32_t* __restrict__ dst,
                                               uint32_t* __restrict__ ndst, int dstride) {
#pragma unroll
    for (int col = 0; col < CH; ++col) {
        dst[(col * 2 + 0) * dstride] = 0u;
        dst[(col * 2 + 1) * dstride] = 0u;
        ndst[col * dstride] = ~0u;
    }
}

// One chunk straight from global memory (long-record path): rows need only be
// 4-byte aligned.
__device__ __forceinline__ uint32_t produce_chunk(const uint8_t* __restrict__ seq, size_t pitch,
                                                  long long row0, long long n, int chunk, int m,
                                                  uint32_t* __restrict__ dst,
                                                  uint32_t* __restrict__ ndst, int dstride) {
    const int col0 = chunk * CH;
    if (chunk < 0 || col0 >= m) {
        fill_oob_chunk(dst, ndst, dstride);
        return 0u;
    }
    if (col0 + CH <= m)
        return gather_chunk<false, true, 4, 4>(seq, pitch, row0, n, col0, m, dst, ndst, dstride);
    return gather_chunk<true, true, 4, 4>(seq, pitch, row0, n, col0, m, dst, ndst, dstride);
}

}  // namespace sb
