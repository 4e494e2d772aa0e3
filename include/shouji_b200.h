/*
 * shouji_b200 — C ABI of the B200-native Shouji pre-alignment filter.
 *
 * This is the drop-in boundary for the reference's hot path
 *
 *   prefilter::shouji_filter(const packed_sequence& pattern,
 *                            const packed_sequence& text,
 *                            std::uint32_t e, unsigned width = 4)
 *       proj/include/prefilter/shouji.hpp:57-59, proj/src/shouji.cpp:41-58
 *
 * and of its batch callers (run_filter proj/src/evaluate.cpp:13-21 driven by
 * parallel_for_pairs proj/src/evaluate.cpp:23-48, run_bench
 * proj/src/bench.cpp:11-42). Plain pointers and sizes only; no C++ or torch
 * types cross it. All compute runs in hand-written sm_100a kernels; there is
 * no CPU fallback: without a usable CUDA device every compute entry point
 * returns PF_ERR_NO_DEVICE.
 *
 * Input records are ASCII (A/C/G/T/N, upper case only — lower case is an
 * illegal character exactly as in packed_sequence::from_string,
 * proj/src/packed_sequence.cpp:19-29). Pair i's text (reference segment) is
 * at text + i*stride and its pattern (read) at pattern + i*stride, m bytes
 * each. Argument order follows the reference: the PATTERN is the read, the
 * TEXT the reference segment; swapping them changes results.
 *
 * Outputs: accept_bitmap is LSB-first, bit i%32 of word i/32 is pair i's
 * accept (ceil(n/32) words; bits past n are zero). estimates[i] is the
 * filter_decision::edit_estimate (popcount of the tally vector,
 * proj/include/prefilter/filter_decision.hpp:12-16). bits, when requested,
 * holds the tally vector of pair i as ceil(m/64) LSB-first uint64 words at
 * bits + i*ceil(m/64) (bitvector word layout, bitvector.hpp:16-31).
 */
#ifndef SHOUJI_B200_H
#define SHOUJI_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes map 1:1 onto the reference exception classes
 * (proj/include/prefilter/errors.hpp:11-84). */
typedef enum pf_status {
    PF_OK = 0,
    PF_ERR_EMPTY_SEQUENCE = 1,      /* empty_sequence_error      errors.hpp:17-20 */
    PF_ERR_ILLEGAL_CHARACTER = 2,   /* illegal_character_error   errors.hpp:23-37 */
    PF_ERR_LENGTH_MISMATCH = 3,     /* length_mismatch_error     errors.hpp:40-48 */
    PF_ERR_THRESHOLD_TOO_LARGE = 4, /* threshold_too_large_error errors.hpp:52-57 */
    PF_ERR_OUT_OF_BAND = 5,         /* out_of_band_error         errors.hpp:60-65 */
    PF_ERR_PARSE = 6,               /* parse_error               errors.hpp:68-77 */
    PF_ERR_INVALID_PARAMETERS = 7,  /* invalid_parameters_error  errors.hpp:81-84 */
    PF_ERR_NO_DEVICE = 100,         /* no usable sm_100 CUDA device */
    PF_ERR_CUDA = 101,              /* a CUDA runtime call failed */
    PF_ERR_OUT_OF_MEMORY = 102,
    PF_ERR_NULL_ARGUMENT = 103
} pf_status;

/* Where an error was found. For PF_ERR_ILLEGAL_CHARACTER: the lowest pair
 * index holding an illegal byte, text (field 0) checked before pattern
 * (field 1) as load_pairs does (proj/src/dataset.cpp:28-30), and the first
 * offending offset within that sequence (packed_sequence.cpp:27-28). */
typedef struct pf_error {
    int32_t status;
    uint32_t field;    /* 0 = text, 1 = pattern */
    uint64_t pair;
    uint64_t position;
    uint32_t byte;
    int32_t cuda_error; /* cudaError_t when status == PF_ERR_CUDA */
    uint64_t line;      /* 1-based input line for PF_ERR_PARSE / dataset length errors */
    char message[160];
} pf_error;

typedef struct pf_ctx pf_ctx;

/* Library / device information. */
const char* pf_status_string(int status);
const char* pf_version(void);
/* Number of CUDA devices usable by this build (0 when none). */
int pf_device_count(void);

/* Context over a set of devices (one stream, pinned staging and device
 * buffers per device; all library-owned). A batch is split into contiguous
 * pair ranges, 32-pair aligned, one per device — the static chunking of
 * parallel_for_pairs (evaluate.cpp:36-37) — and gathered on the host; there
 * is no device-to-device traffic. devices == NULL / count == 0 means device 0.
 * A context is internally serialised; use one per host thread for concurrency. */
int pf_ctx_create(const int* devices, int count, pf_ctx** out);
void pf_ctx_destroy(pf_ctx* ctx);
int pf_ctx_device_count(const pf_ctx* ctx);
/* How host batches are spread over the ctx's devices: chunk_pairs = 0 (default)
 * cuts each batch into one contiguous 32-pair-aligned shard per device (the
 * n*t/T split of parallel_for_pairs, proj/src/evaluate.cpp:36-37); > 0 deals
 * consecutive chunks of that many pairs (rounded up to 32) round-robin, chunk c
 * to device c mod N — BASELINE config 4's streaming layout (1Mi-pair chunks over
 * 8 GPUs). Results are identical either way. */
int pf_ctx_set_shard_chunk(pf_ctx* ctx, size_t chunk_pairs);

/* Batched Shouji over caller-owned HOST buffers (pinned or pageable; pinned
 * buffers are DMA'd directly). Synchronous. Checks, in the reference's order:
 *   m == 0 with n > 0                  -> PF_ERR_EMPTY_SEQUENCE
 *   any illegal byte                   -> PF_ERR_ILLEGAL_CHARACTER (+ err)
 *   width outside [3, 8]               -> PF_ERR_INVALID_PARAMETERS
 *   e >= m                             -> every pair accepted, estimate 0,
 *                                         all-zero bits (shouji.cpp:48-49)
 * estimates and bits may be NULL. stride >= m. */
int pf_shouji_filter_batch(pf_ctx* ctx, const uint8_t* text, const uint8_t* pattern,
                           size_t stride, size_t n, uint32_t m, uint32_t e, uint32_t width,
                           uint32_t* accept_bitmap, uint32_t* estimates, uint64_t* bits,
                           pf_error* err);

/* Same over DEVICE-resident records on the ctx's first device, asynchronous
 * on `stream` (a cudaStream_t; NULL = the legacy default stream) except that an error
 * check forces a stream synchronisation at the end. Records need a pitch that
 * is a multiple of 4 and >= m (pf_device_pitch(m) = round4(m) is the tight
 * layout) and 16-byte aligned bases; bytes in [m, pitch) are ignored, but they are
 * read: each record array must span n*pitch bytes (the last record included; its
 * padding is loaded by the tile copies and never used). Output pointers
 * are device pointers (accept_bitmap ceil(n/32) words; estimates/bits as for
 * the host call, may be NULL). */
int pf_shouji_filter_device(pf_ctx* ctx, const uint8_t* d_text, const uint8_t* d_pattern,
                            size_t pitch, size_t n, uint32_t m, uint32_t e, uint32_t width,
                            uint32_t* d_accept_bitmap, uint32_t* d_estimates, uint64_t* d_bits,
                            void* stream, pf_error* err);

/* Same as pf_shouji_filter_device but fully asynchronous: no host sync and no
 * error location. Any illegal byte ORs 1 into *d_err_flag (a device word the
 * caller zeroes); call pf_shouji_filter_device to locate it. Used for
 * back-to-back device-resident throughput runs. e < m and 3 <= width <= 8
 * are required (the short-circuit / width errors need the synchronous call). */
int pf_shouji_filter_device_async(pf_ctx* ctx, const uint8_t* d_text, const uint8_t* d_pattern,
                                  size_t pitch, size_t n, uint32_t m, uint32_t e, uint32_t width,
                                  uint32_t* d_accept_bitmap, uint32_t* d_estimates,
                                  uint32_t* d_err_flag, void* stream);

/* Diagnostic: pf_shouji_filter_device_async's two stages timed separately
 * with CUDA events on the context's stream (pack = records -> planes, search =
 * map + select + commit + accept), averaged over reps synchronous runs. */
int pf_shouji_profile_stages(pf_ctx* ctx, const uint8_t* d_text, const uint8_t* d_pattern,
                             size_t pitch, size_t n, uint32_t m, uint32_t e, uint32_t width,
                             uint32_t* d_accept_bitmap, uint32_t* d_err_flag, int reps,
                             float* pack_ms, float* search_ms);

/* Measured integer pipe throughput on the ctx's first device (diagnostic for
 * the INT roofline): op 0 = LOP3, 1 = funnel shift, 2 = PRMT, 3 = IMAD.
 * Writes lane-operations per second. */
int pf_int_peak(pf_ctx* ctx, int op, double* ops_per_second);

/* ---- Split stages (advanced callers) -------------------------------------
 * The host batch call's upload stage, exposed on its own. pf_host_pack_nibbles
 * packs ASCII records on the host's cores into nibble records (4 bits per
 * base, pf_nibble_pitch(m) bytes per record: byte q of 32-bit word w holds the
 * low nibbles of columns 8w+q and 8w+q+4), validating every byte like
 * packed_sequence::from_string (proj/src/packed_sequence.cpp:19-29: first
 * illegal byte in pair order, text before pattern). simd = 0 forces the
 * portable path. pf_shouji_filter_nibbles_device filters nibble records
 * already in device memory (stream-ordered, no validation: the host did it).
 * pf_shouji_filter_batch packs large batches this way (PF_HOST_PACK=0 turns
 * it off, =1 forces it). */
size_t pf_nibble_pitch(uint32_t m);
int pf_host_pack_nibbles(const uint8_t* text, const uint8_t* pattern, size_t stride, size_t n,
                         uint32_t m, uint8_t* out_text, uint8_t* out_pattern, int simd,
                         pf_error* err);
int pf_shouji_filter_nibbles_device(pf_ctx* ctx, const uint8_t* d_text, const uint8_t* d_pattern,
                                    size_t n, uint32_t m, uint32_t e, uint32_t width,
                                    uint32_t* d_accept_bitmap, uint32_t* d_estimates, void* stream,
                                    pf_error* err);

/* Tight device row pitch for length-m records: round4(m). */
size_t pf_device_pitch(uint32_t m);

/* Exact alignment oracle / verification step on the GPU:
 * banded_edit_distance(pattern, text, e) (proj/src/edit_distance.cpp:26-70)
 * for every pair of host records: out[i] = distance if <= e, else -1 (the
 * reference's std::nullopt). N matches nothing. Same validation and error
 * reporting as pf_shouji_filter_batch; m <= 1024. */
int pf_banded_edit_distance_batch(pf_ctx* ctx, const uint8_t* text, const uint8_t* pattern,
                                  size_t stride, size_t n, uint32_t m, uint32_t e, int32_t* out,
                                  pf_error* err);

/* Per-pair compatibility entry (a batch of one), reference argument order:
 * shouji_filter(pattern, text, e, width). Lengths may differ (->
 * PF_ERR_LENGTH_MISMATCH, checked before the width, shouji.cpp:44-47).
 * bits may be NULL (else ceil(text_len/64) words). */
int pf_shouji_filter_one(pf_ctx* ctx, const char* pattern, size_t pattern_len, const char* text,
                         size_t text_len, uint32_t e, uint32_t width, int* accept,
                         uint32_t* estimate, uint64_t* bits, pf_error* err);

/* Dibit records: the default upload format of the host-pack path (2 bits per
 * base; pf_dibit_pitch(m) = 4*ceil(m/16) bytes per record: byte q of 32-bit
 * word w holds the codes (ASCII bits 1-2) of columns 16w+q, +4, +8, +12 at
 * bits 0-1, 2-3, 4-5, 6-7). N is carried in N-plane records
 * (pf_nplane_pitch(m) = 4*ceil(m/32) bytes, bit c = column c is 'N'), written
 * by pf_host_pack_dibits only when *has_n comes back 1 (both N arrays may be
 * NULL when the caller knows there is no N). pf_shouji_filter_dibits_device
 * filters dibit records on the device; pass NULL N arrays for N-free batches.
 * PF_HOST_FORMAT=nibble makes pf_shouji_filter_batch upload nibbles instead. */
size_t pf_dibit_pitch(uint32_t m);
size_t pf_nplane_pitch(uint32_t m);
int pf_host_pack_dibits(const uint8_t* text, const uint8_t* pattern, size_t stride, size_t n,
                        uint32_t m, uint8_t* out_text, uint8_t* out_pattern, uint8_t* n_text,
                        uint8_t* n_pattern, int* has_n, int simd, pf_error* err);
int pf_shouji_filter_dibits_device(pf_ctx* ctx, const uint8_t* d_text, const uint8_t* d_pattern,
                                   const uint8_t* d_ntext, const uint8_t* d_npattern, size_t n,
                                   uint32_t m, uint32_t e, uint32_t width,
                                   uint32_t* d_accept_bitmap, uint32_t* d_estimates, void* stream,
                                   pf_error* err);

/* ---- Packed-planes variant --------------------------------
 * Pairs the caller already packed with packed_sequence::from_string
 * (proj/src/packed_sequence.cpp:7-34), passed in that class's own storage:
 * per pair and sequence pf_packed_words(m) = 3 * ceil(m/64) uint64 words,
 * low_plane then high_plane then n_plane (packed_sequence.hpp:50-53), each
 * LSB-first (bit j of word w = base 64w+j; bits >= m ignored):
 *   text_planes[i * pf_packed_words(m) + k * ceil(m/64) + w]
 * This is the input run_bench times (pairs pre-packed, bench.cpp:24-25). No
 * validation is needed (packing validated); the width check and the e >= m
 * short-circuit follow shouji.cpp:47-49. Host arrays may be pinned (DMA'd in
 * place) or pageable (staged through pinned buffers in 1Mi-pair chunks). */
size_t pf_packed_words(uint32_t m);
int pf_shouji_filter_packed_batch(pf_ctx* ctx, const uint64_t* text_planes,
                                  const uint64_t* pattern_planes, size_t n, uint32_t m, uint32_t e,
                                  uint32_t width, uint32_t* accept_bitmap, uint32_t* estimates,
                                  uint64_t* bits, pf_error* err);
/* Same on device-resident plane arrays (8-byte aligned), stream-ordered. */
int pf_shouji_filter_packed_device(pf_ctx* ctx, const uint64_t* d_text_planes,
                                   const uint64_t* d_pattern_planes, size_t n, uint32_t m,
                                   uint32_t e, uint32_t width, uint32_t* d_accept_bitmap,
                                   uint32_t* d_estimates, uint64_t* d_bits, void* stream,
                                   pf_error* err);

/* ---- MAGNET (proj/src/magnet.cpp) --------------------------
 * magnet_filter(pattern, text, e) (magnet.cpp:77-87) over a batch: e+1
 * extract-and-encapsulate steps over the 2e+1 diagonals; estimate =
 * popcount(bits), accept = estimate <= e; e >= m accepts with estimate 0 and
 * all-zero bits. Same validation, error order, outputs and sharding as
 * pf_shouji_filter_batch (no width). One GPU thread per pair; m <= 512.
 * Replaces run_filter(filter_algo::magnet, ...) (evaluate.cpp:13-21). */
int pf_magnet_filter_batch(pf_ctx* ctx, const uint8_t* text, const uint8_t* pattern, size_t stride,
                           size_t n, uint32_t m, uint32_t e, uint32_t* accept_bitmap,
                           uint32_t* estimates, uint64_t* bits, pf_error* err);
/* Device-resident records (same layout rules as pf_shouji_filter_device),
 * synchronous validation, results stream-ordered on `stream`. */
int pf_magnet_filter_device(pf_ctx* ctx, const uint8_t* d_text, const uint8_t* d_pattern,
                            size_t pitch, size_t n, uint32_t m, uint32_t e,
                            uint32_t* d_accept_bitmap, uint32_t* d_estimates, uint64_t* d_bits,
                            void* stream, pf_error* err);
/* Per-pair magnet_filter(pattern, text, e) (a batch of one). */
int pf_magnet_filter_one(pf_ctx* ctx, const char* pattern, size_t pattern_len, const char* text,
                         size_t text_len, uint32_t e, int* accept, uint32_t* estimate,
                         uint64_t* bits, pf_error* err);

/* Pinned host allocation helpers (cudaHostAlloc on the ctx's first device). */
void* pf_host_alloc(size_t bytes);
void pf_host_free(void* p);

/* Seeded synthetic pair generator on the device (bench / test workloads; see
 * DESIGN.md "Synthetic configs"). Writes n records of length m with the
 * given pitch into d_text / d_pattern. kind: 1..4 = BASELINE.json configs 1..4
 * (param = E for configs 1 and 3, ignored otherwise). Deterministic in
 * (kind, seed, param, pair index). */
int pf_generate_device(pf_ctx* ctx, int kind, uint64_t seed, uint32_t param, uint8_t* d_text,
                       uint8_t* d_pattern, size_t pitch, size_t n, uint32_t m, void* stream);

/* ---- Pair datasets: the caller side of the path (dataset.hpp / dataset.cpp) ----
 * A dataset holds n equal-length ASCII pairs as fixed-stride records (stride =
 * m, pinned host memory when available), ready for pf_shouji_filter_batch. */
typedef struct pf_dataset pf_dataset;

/* load_pairs (proj/src/dataset.cpp:13-44): one TEXT '\t' PATTERN pair per
 * line. The scan and the byte validation run on the host cores (ctx is not
 * used and may be NULL; the records are then filtered on a ctx's GPUs by the
 * batch calls); errors are the ones the
 * reference's line-by-line loader throws first: PF_ERR_PARSE with err->line for
 * a wrong field count, an empty field or an illegal byte (err->position/byte),
 * PF_ERR_LENGTH_MISMATCH with err->line for unequal lengths, PF_ERR_PARSE line
 * 1 for an input without pairs. */
int pf_dataset_load_tsv(pf_ctx* ctx, const char* data, size_t len, const char* source_name,
                        pf_dataset** out, pf_error* err);
int pf_dataset_load_tsv_file(pf_ctx* ctx, const char* path, pf_dataset** out, pf_error* err);
/* generate_pairs({seed, count, length, {lo, hi}}) (dataset.cpp:71-126), byte-identical. */
int pf_dataset_generate(uint64_t seed, size_t count, uint32_t length, uint32_t lo, uint32_t hi,
                        pf_dataset** out, pf_error* err);
/* Copy caller records (stride >= m) into a dataset. */
int pf_dataset_from_records(const uint8_t* text, const uint8_t* pattern, size_t stride, size_t n,
                            uint32_t m, const char* source_name, pf_dataset** out);
size_t pf_dataset_size(const pf_dataset* ds);
uint32_t pf_dataset_length(const pf_dataset* ds);
const uint8_t* pf_dataset_text(const pf_dataset* ds);
const uint8_t* pf_dataset_pattern(const pf_dataset* ds);
const char* pf_dataset_source(const pf_dataset* ds);
/* write_pairs (dataset.cpp:53-56); path "-" = stdout. */
int pf_dataset_write_tsv(const pf_dataset* ds, const char* path);
void pf_dataset_free(pf_dataset* ds);

/* Number of kernel launches issued by this process so far (all contexts);
 * bench.py reports the delta over its timed region. */
uint64_t pf_launch_count(void);

/* Bytes copied host->device and device->host by the host entry points
 * (pf_shouji_filter_batch and friends) so far in this process; bench.py
 * reports the per-step delta as the e2e transfer volume. Either may be NULL. */
void pf_transfer_bytes(uint64_t* h2d, uint64_t* d2h);

/* Diagnostic: how fast this host's cores stream-read `bytes` of the caller's
 * buffer (GB/s; the host pack's AVX-512 loads and prefetch, all pool threads,
 * `passes` timed passes after a warm one). Every host entry point must read
 * each record byte once, so this is the ceiling of the host-records e2e path:
 * pairs/s <= gbs * 1e9 / (2 * m). Returns 0 for buffers under 1 MiB. No GPU. */
double pf_host_read_bandwidth(const void* buf, size_t bytes, int passes);

#ifdef __cplusplus
}
#endif

#endif /* SHOUJI_B200_H */
