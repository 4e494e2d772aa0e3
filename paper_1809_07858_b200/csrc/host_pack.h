// Host packing stage: ASCII records -> nibble records on the CPU (see host_pack.cpp).
#pragma once
#include <cstddef>
#include <cstdint>

namespace sb {

// First illegal byte seen, in the reference's order: lowest pair, text (field
// 0) before pattern (field 1), lowest position.
struct HostBad {
    bool any = false;
    uint64_t pair = 0;
    int field = 0;
    int pos = 0;
    uint8_t byte = 0;
    void offer(uint64_t p, int f, int q, uint8_t b) {
        if (!any || p < pair || (p == pair && (f < field || (f == field && q < pos)))) {
            any = true;
            pair = p;
            field = f;
            pos = q;
            byte = b;
        }
    }
};

// Pack pairs [lo, hi) of a batch into nibble records (pack.cuh nibble format,
// row pitch nibble_pitch(m)); out_text/out_pattern point at the batch's row 0.
// Thread-safe for disjoint pair ranges.
void host_pack_nibbles(const uint8_t* text, const uint8_t* pattern, size_t stride, int m,
                       long long lo, long long hi, uint8_t* out_text, uint8_t* out_pattern,
                       HostBad* bad, bool allow_simd = true);

// All n pairs on the process-wide worker pool (threads = 0: all hardware
// threads). bad receives the first illegal byte in pair order.
void host_pack_nibbles_parallel(const uint8_t* text, const uint8_t* pattern, size_t stride,
                                long long n, int m, uint8_t* out_text, uint8_t* out_pattern,
                                HostBad* bad, unsigned threads = 0, bool allow_simd = true);
unsigned host_pack_threads();

// All n pairs into dibit records (pack.cuh) on the worker pool. has_n reports
// whether any base is 'N'; only then are the N-plane records (n_text,
// n_pattern; nplane_pitch(m) bytes per record) written.
void host_pack_dibits_parallel(const uint8_t* text, const uint8_t* pattern, size_t stride,
                               long long n, int m, uint8_t* out_text, uint8_t* out_pattern,
                               uint8_t* n_text, uint8_t* n_pattern, HostBad* bad, bool* has_n,
                               bool allow_simd = true);

// Alphabet check only (packed_sequence::from_string's byte rule) over n pairs
// on the worker pool: bad receives the first illegal byte in pair order.
void host_validate_parallel(const uint8_t* text, const uint8_t* pattern, size_t stride,
                            long long n, int m, HostBad* bad);

// memcpy on the same worker pool (pageable -> pinned staging copies).
void host_copy_parallel(void* dst, const void* src, size_t bytes);

// Stream-read bandwidth of the host cores over buf (GB/s, `passes` timed passes
// after one warm pass), with the host pack's access pattern on its worker pool.
double host_read_gbs(const uint8_t* buf, size_t bytes, int passes);

// True when the AVX-512 (BW/VBMI) path is used on this host.
bool host_pack_uses_simd();

}  // namespace sb
