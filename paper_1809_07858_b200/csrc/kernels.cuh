// Internal launch interface between the C ABI (capi.cpp) and the sm_100a
// kernels (kernels.cu). Not installed; not part of the public boundary.
#pragma once
#include <cstddef>
#include <atomic>
#include <cstdint>

#include <cuda_runtime.h>

namespace sb {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device):
// the attribute belongs to the device's context, so a context spanning several
// devices must set it on each (one bit per device ordinal).
template <auto Kernel>
cudaError_t ensure_smem_attr(int bytes) {
    static std::atomic<unsigned long long> done{0};
    int dev = 0;
    cudaError_t st = cudaGetDevice(&dev);
    if (st != cudaSuccess) return st;
    const unsigned long long bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    st = cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (st == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
    return st;
}

// Largest E served by the fused, E-specialised width-4 kernel; larger E and
// widths other than 4 run the two-kernel generic path.
constexpr int kFusedMaxE = 31;

struct FilterArgs {
    const uint8_t* text;     // device, [n][pitch]
    const uint8_t* pattern;  // device, [n][pitch]
    size_t pitch;
    long long n;
    int m;
    uint32_t e;
    uint32_t width;
    uint32_t* accept;      // device, ceil(n/32) words
    uint32_t* estimates;   // device, n, may be null
    uint32_t* outplanes;   // device scratch [m][ngroups] or null (tally dump)
    uint32_t* err_flag;    // device, 1 word, zeroed by the caller
    uint32_t* planes;      // device scratch for the pair-sliced planes (pack.cuh)
    size_t planes_words;   // available words in planes
    bool nibbles;          // text/pattern are host-packed nibble records (pitch unused)
    bool dibits;           // text/pattern are dibit records (pack.cuh; pitch unused)
    const uint8_t* ntext;     // dibits: N-plane records, or null when the batch has no N
    const uint8_t* npattern;
    cudaEvent_t stage_event;   // non-null: recorded between the pack and the search kernel
    const uint64_t* packed_text;     // non-null: pre-packed planes input (pack_planes.cu);
    const uint64_t* packed_pattern;  //   text/pattern/pitch unused
    uint32_t* nflags;  // set by launch_filter: N-presence flags (pack.cuh) shared by the
                       // pack and search kernels, or null (N planes always stored and read)
};

// Scratch words the filter needs for n pairs of length m.
size_t planes_scratch_words(long long n, int m);
bool use_fused(uint32_t width, uint32_t e, int m);

// Stage 1: records -> planes (planes may be null: validation only).
// nflags (optional): write N-presence flags and skip N-free groups' N planes
// (requires pack_writes_nflags).
cudaError_t launch_pack(const uint8_t* text, const uint8_t* pattern, size_t pitch, long long n,
                        int m, uint32_t* planes, uint32_t* err_flag, cudaStream_t s,
                        uint32_t* nflags = nullptr);
bool pack_writes_nflags(const FilterArgs& a);
// Stage 1 from nibble records (pack.cuh nibble format; no validation).
bool nibble_pack_fits(int m);
cudaError_t launch_pack_nibbles(const uint8_t* text, const uint8_t* pattern, long long n, int m,
                                uint32_t* planes, cudaStream_t s, uint32_t* nflags = nullptr);
// Blocked search for any width 3..8 and any E (wsearch.cuh), m <= 4095.
bool wsearch_applies(const FilterArgs& a);
cudaError_t launch_wsearch(const FilterArgs& a, cudaStream_t s);
// Stage 1 from dibit records (+ optional N-plane records; pack.cuh).
bool dibit_pack_fits(int m);
cudaError_t launch_pack_dibits(const uint8_t* text, const uint8_t* pattern, const uint8_t* ntext,
                               const uint8_t* npattern, long long n, int m, uint32_t* planes,
                               cudaStream_t s,
                               uint32_t* nflags = nullptr);
// Stage 1 from packed_sequence planes ([n][3][ceil(m/64)] u64 per sequence).
// packed_sequence planes (16-byte aligned, ceil(m/64) <= 8) can also write the
// N-presence flags (pack.cuh).
bool pack_planes_writes_nflags(const uint64_t* text, const uint64_t* pattern, int m);
cudaError_t launch_pack_planes(const uint64_t* text, const uint64_t* pattern, long long n, int m,
                               uint32_t* planes, cudaStream_t s,
                               uint32_t* nflags = nullptr);
// Launch the filter (pack + width-4 search, or pack + generic). Returns a cudaError_t.
cudaError_t launch_filter(const FilterArgs& a, cudaStream_t s);
// One stage of launch_filter on its own stream: 1 = pack into a.planes, 2 = search
// from them (same FilterArgs for both; the caller orders stage 2 after stage 1).
cudaError_t launch_filter_stage(const FilterArgs& a, cudaStream_t s, int stage);
// Validation only (for e >= m or an invalid width): sets *err_flag on any illegal byte.
cudaError_t launch_validate(const FilterArgs& a, cudaStream_t s);
// First illegal byte: key = ((pair*2+field) << 24) | pos into *d_key (pre-set to ~0).
cudaError_t launch_locate(const uint8_t* text, const uint8_t* pattern, size_t pitch, long long n,
                          int m, unsigned long long* d_key, cudaStream_t s);
// [m][ngroups] tally plane words -> per-pair bitvector words.
cudaError_t launch_bits_transpose(const uint32_t* outplanes, long long n, int m, uint64_t* bits,
                                  cudaStream_t s);
// Copy n rows of m bytes from a device buffer with any row stride into the
// tight round4(m)-pitched layout the filter kernels read.
cudaError_t launch_repitch(const uint8_t* src, size_t src_stride, uint8_t* dst, size_t dst_pitch,
                           long long n, int m, cudaStream_t s);
// Exact Levenshtein distance per pair (Myers bit-vector); out[i] = d <= e ? d : -1.
// The same from dibit records (+ optional N rows), the host-pack upload format.
cudaError_t launch_edit_distance_dibits(const uint8_t* text, const uint8_t* pattern,
                                        const uint8_t* ntext, const uint8_t* npattern, long long n,
                                        int m, int e, int32_t* out, cudaStream_t s);
cudaError_t launch_edit_distance(const uint8_t* text, const uint8_t* pattern, size_t pitch,
                                 long long n, int m, int e, int32_t* out, cudaStream_t s);
// MAGNET (magnet.cu): one thread per pair, validated ASCII records, 0 <= e < m,
// m <= kMagnetMaxM. Writes the accept bitmap, optional u32 estimates and
// optional tally bits [n][ceil(m/64)] u64.
constexpr int kMagnetMaxM = 512;
bool magnet_supported(int m);
cudaError_t launch_magnet(const uint8_t* text, const uint8_t* pattern, size_t pitch, long long n,
                          int m, int e, uint32_t* accept, uint32_t* estimates, uint64_t* bits,
                          cudaStream_t s);
// MAGNET from dibit records (+ optional N-plane rows), as produced by the host pack.
cudaError_t launch_magnet_dibits(const uint8_t* text, const uint8_t* pattern, const uint8_t* ntext,
                                 const uint8_t* npattern, long long n, int m, int e,
                                 uint32_t* accept, uint32_t* estimates, uint64_t* bits,
                                 cudaStream_t s);
// Latency form for small batches (small.cu): one CTA per pair, windows over the
// threads. ASCII records (text/pattern/stride; validated, first illegal byte into
// *bad_key as launch_locate encodes it) or packed_sequence planes (tplanes/pplanes,
// [n][3][ceil(m/64)] u64). accept: one byte per pair (0/1); est and bits may be
// null. Any pointer may be a mapped pinned host alias.
constexpr int kSmallMaxM = 2048;
constexpr long long kSmallMaxN = 64;
struct SmallArgs {
    const uint8_t* text;
    const uint8_t* pattern;
    size_t stride;
    const uint64_t* tplanes;
    const uint64_t* pplanes;
    int n;
    int m;
    uint32_t e;
    int w;
    uint8_t* accept;
    uint32_t* est;
    uint64_t* bits;
    unsigned long long* bad_key;
    unsigned* counter;         // device word, 0 between launches (null: no done flag)
    volatile unsigned* done;   // receives seq when every CTA has finished
    unsigned seq;
};
size_t small_smem_bytes(int m, uint32_t e);
cudaError_t launch_small(const SmallArgs& a, cudaStream_t s);

// e >= m short-circuit outputs.
cudaError_t launch_accept_all(long long n, int m, uint32_t* accept, uint32_t* estimates,
                              uint64_t* bits, cudaStream_t s);
cudaError_t launch_generate(int kind, uint64_t seed, uint32_t param, uint8_t* text,
                            uint8_t* pattern, size_t pitch, long long n, int m, cudaStream_t s);

// Integer pipe microbenchmark (diagnostic): lane-ops per second for op
// 0 LOP3, 1 SHF (funnel), 2 PRMT, 3 IMAD.
cudaError_t measure_int_peak(int op, cudaStream_t s, double* ops_per_second);

uint64_t launch_count();
void count_launch(int k = 1);

}  // namespace sb
