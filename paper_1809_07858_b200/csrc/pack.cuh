// Stage 1 of the Shouji pipeline: ASCII records -> pair-sliced bit planes.
//
// Reference: packed_sequence::from_string (proj/src/packed_sequence.cpp:7-34),
// applied to every text and pattern of the batch before any filtering, as
// load_pairs / generate_pairs do (proj/src/dataset.cpp:28-30,86-87).
//
// Memory shape. One CTA owns a PAIR BLOCK of 256 consecutive pairs (8 groups
// of 32). Its records are two contiguous byte ranges (256 rows x pitch), so
// they arrive with two TMA bulk copies (cp.async.bulk, completion on an
// mbarrier) at full sector efficiency. Threads then bit-transpose 16-column x
// 32-pair tiles out of shared memory (gather_chunk, phase_a.cuh) and the CTA
// writes its planes back as one contiguous range per sequence:
//
//   planes [s][pair_block][col][lo, hi][8 groups]     (uint32 words)
//   nplanes[s][pair_block][col][8 groups]              (after all lo/hi planes)
//
// so the filter kernel, whose thread owns one group and walks columns, reads
// one fully used 32-byte sector per (column, plane) per 8 threads. The N
// planes live in their own region so that N-free pair blocks (the usual case)
// neither write nor read them: whole lines are skipped, not single sectors
// inside lines that are written anyway (which saves no DRAM traffic).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace sb {

constexpr int kPackPairs = 256;                 // pairs per pair block (CTA)
constexpr int kPackGroups = kPackPairs / 32;    // groups per pair block
constexpr int kPackNT = 128;                    // threads per pack CTA

// Column stride of the planes layout: exactly m (only columns < m are ever
// written or read).
__host__ __device__ inline int plane_cols(int m) { return m; }

// Words of plane storage for n pairs of length m (both sequences, lo/hi + N).
inline size_t plane_words(long long n, int m) {
    const long long blocks = (n + kPackPairs - 1) / kPackPairs;
    return static_cast<size_t>(2 * blocks * plane_cols(m) * 3 * kPackGroups);
}

constexpr int kLhColWords = 2 * kPackGroups;  // lo/hi words per column of a pair block
constexpr int kNColWords = kPackGroups;       // N words per column of a pair block

// Offset (in words) of plane word (s, group g, col, k in {0 lo, 1 hi}); the
// group's 8-lane slot is g % 8.
__host__ __device__ inline size_t lohi_index(int s, long long g, int col, int k, long long nblocks,
                                             int mc) {
    const long long blk = g / kPackGroups;
    return ((static_cast<size_t>(s) * nblocks + blk) * mc + col) * kLhColWords + k * kPackGroups +
           (g % kPackGroups);
}

// Offset (in words) of N-plane word (s, group g, col).
__host__ __device__ inline size_t nplane_index(int s, long long g, int col, long long nblocks,
                                               int mc) {
    const long long blk = g / kPackGroups;
    return static_cast<size_t>(2 * nblocks) * mc * kLhColWords +
           ((static_cast<size_t>(s) * nblocks + blk) * mc + col) * kNColWords + (g % kPackGroups);
}

// N-presence flags, stored after the plane words: one uint32 per (sequence,
// group), nonzero iff the N planes of that group were stored. A pack kernel
// that writes flags stores the N planes of a tile's sequence only when one of
// its records holds an N, and a search that reads flags points N-free groups
// at an all-zero column image (after the flags, plane_cols(m) x 8 words) or,
// for a warp of N-free groups, drops the N terms altogether.
__host__ __device__ inline size_t nflag_words(long long n) {
    return static_cast<size_t>(2 * ((n + kPackPairs - 1) / kPackPairs) * kPackGroups);
}
__host__ __device__ inline size_t nflag_index(int s, long long g, long long nblocks) {
    return static_cast<size_t>(s) * nblocks * kPackGroups + g;
}
__host__ __device__ inline size_t nzero_words(int m) {
    return static_cast<size_t>(plane_cols(m)) * kNColWords;
}

// Nibble records: the upload format of host-packed batches (host_pack.cpp).
// A record of m columns is ceil(m/8) little-endian uint32 words; byte q of
// word w holds the low nibbles of columns 8w+q (bits 0-3) and 8w+q+4 (bits
// 4-7); columns >= m are zero. Bits 1-3 of a nibble are bits 1-3 of the ASCII
// byte (lo, hi, N), so the device gather needs only a different shift per
// column. Validation happens on the host, which packs.
__host__ __device__ inline size_t nibble_pitch(int m) { return 4 * static_cast<size_t>((m + 7) / 8); }

// Dibit records: the compact upload format (host_pack.cpp). A record of m
// columns is ceil(m/16) little-endian uint32 words; byte q of word w holds the
// 2-bit codes (ASCII bits 1-2: lo, hi) of columns 16w+q, 16w+q+4, 16w+q+8 and
// 16w+q+12 at bits 0-1, 2-3, 4-5, 6-7; columns >= m are zero. N is carried
// separately: N-plane records of ceil(m/32) uint32 words (bit c = column c is
// 'N'), sent only for chunks that contain an N.
__host__ __device__ inline size_t dibit_pitch(int m) { return 4 * static_cast<size_t>((m + 15) / 16); }
__host__ __device__ inline size_t nplane_pitch(int m) { return 4 * static_cast<size_t>((m + 31) / 32); }

}  // namespace sb
