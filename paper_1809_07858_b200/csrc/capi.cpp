// C ABI of the B200-native Shouji filter (declared in include/shouji_b200.h).
//
// Host side of the boundary: argument checks in the reference's order
// (proj/src/shouji.cpp:44-49, packed_sequence.cpp:8,27-28), device buffer and
// pinned-staging management, the 32-pair-aligned static split across devices
// (the contiguous chunking of parallel_for_pairs, proj/src/evaluate.cpp:36-37)
// and the gather of per-device bitmaps. Every filter decision is computed by
// the sm_100a kernels; the only host-side processing is the host-pack upload
// stage (host_pack.cpp: records packed to 2-bit form and validated on the CPU
// cores before they cross PCIe). Without a device the calls fail with
// PF_ERR_NO_DEVICE.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/shouji_b200.h"
#include "host_pack.h"
#include "kernels.cuh"
#include "pack.cuh"
#include "split.h"

namespace {

constexpr size_t kStageBytes = size_t(64) << 20;  // per-sequence H2D staging chunk

size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct DeviceState {
    int device = 0;
    cudaStream_t stream = nullptr;
    uint8_t* d_text = nullptr;
    uint8_t* d_pattern = nullptr;
    size_t in_bytes = 0;
    size_t in_pattern_bytes = 0;
    uint32_t* d_accept = nullptr;
    size_t accept_words = 0;
    uint32_t* d_est = nullptr;
    size_t est_n = 0;
    uint64_t* d_bits = nullptr;
    size_t bits_words = 0;
    uint32_t* d_outplanes = nullptr;
    size_t outplanes_words = 0;
    uint32_t* d_scratch = nullptr;
    size_t scratch_words = 0;
    uint32_t* d_flag = nullptr;
    unsigned long long* d_key = nullptr;
    uint8_t* d_stage = nullptr;  // device staging for non-pitched host rows
    size_t d_stage_bytes = 0;
    uint8_t* h_stage[2] = {nullptr, nullptr};
    size_t stage_bytes = 0;
    cudaEvent_t stage_ev[2] = {nullptr, nullptr};
    // host-pack upload path: pinned nibble buffers, device nibble buffers, events
    uint8_t* h_nib[2] = {nullptr, nullptr};
    size_t h_nib_bytes = 0;
    uint8_t* d_nib[2] = {nullptr, nullptr};
    size_t d_nib_bytes[2] = {0, 0};
    cudaEvent_t nib_ev[2] = {nullptr, nullptr};
    // host-pack path: a copy stream for the chunk uploads, so chunk i+1's DMA
    // overlaps chunk i's kernels; kern_ev[b]: the kernels that read device
    // buffer b are done (before the next upload into it); up_ev: ordering point
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t kern_ev[2] = {nullptr, nullptr};
    cudaEvent_t up_ev = nullptr;
    uint8_t* h_nrow[2] = {nullptr, nullptr};  // dibit path: pinned N-plane rows
    size_t h_nrow_bytes = 0;
    uint8_t* d_nrow[2] = {nullptr, nullptr};
    size_t d_nrow_bytes[2] = {0, 0};
    // packed-planes input: device chunk buffers (text, pattern) and pinned staging
    uint64_t* d_pk[2] = {nullptr, nullptr};
    size_t d_pk_words[2] = {0, 0};
    uint64_t* h_pk[2] = {nullptr, nullptr};
    size_t h_pk_words = 0;
    cudaEvent_t pk_ev[2] = {nullptr, nullptr};
    // last use of the plane scratch (d_scratch) on any stream:
    // device calls on caller streams and host batches on `stream` share them
    cudaEvent_t scratch_ev = nullptr;
    // latency path (small.cu): mapped pinned staging, host pointer + device alias
    uint8_t* h_small_in = nullptr;
    uint8_t* d_small_in = nullptr;
    size_t small_in_bytes = 0;
    uint8_t* h_small_out = nullptr;
    uint8_t* d_small_out = nullptr;
    size_t small_out_bytes = 0;
    unsigned* d_small_counter = nullptr;  // CTA completion count (device)
    unsigned small_seq = 0;
    // hybrid upload (raw ASCII chunks DMA'd from pinned records alongside the
    // host-pack route): its stream, double-buffered device records, events,
    // plane scratch and validation flag
    cudaStream_t raw_stream = nullptr;
    uint8_t* d_raw[2] = {nullptr, nullptr};
    size_t d_raw_bytes[2] = {0, 0};
    cudaEvent_t raw_ev[2] = {nullptr, nullptr};
    cudaEvent_t raw_done = nullptr;
    uint32_t* d_raw_scratch = nullptr;
    size_t raw_scratch_words = 0;
    uint32_t* d_raw_flag = nullptr;
    // SM-partitioned pack | search pipeline (split.cpp), created on first use
    sb::SplitPipe* split = nullptr;
    int split_sms = 0;  // PF_SPLIT setting the pipe was built for (0: none tried)
};

}  // namespace

struct pf_ctx {
    std::vector<DeviceState> devs;
    std::mutex mu;
    // host batches: 0 = one contiguous 32-aligned shard per device (parallel_for_pairs'
    // split); > 0 = chunks of this many pairs dealt round-robin (chunk c -> device
    // c mod N), the streamed layout of BASELINE config 4
    size_t shard_chunk = 0;
};

namespace {

void set_err(pf_error* err, int status, const char* msg, cudaError_t ce = cudaSuccess) {
    if (!err) return;
    err->status = status;
    err->cuda_error = static_cast<int32_t>(ce);
    if (msg) {
        std::snprintf(err->message, sizeof(err->message), "%s%s%s", msg,
                      ce != cudaSuccess ? ": " : "", ce != cudaSuccess ? cudaGetErrorString(ce) : "");
    }
}

#define PF_CUDA(call)                                                  \
    do {                                                               \
        cudaError_t ce_ = (call);                                      \
        if (ce_ != cudaSuccess) {                                      \
            set_err(err, ce_ == cudaErrorMemoryAllocation ? PF_ERR_OUT_OF_MEMORY : PF_ERR_CUDA, \
                    #call, ce_);                                       \
            return ce_ == cudaErrorMemoryAllocation ? PF_ERR_OUT_OF_MEMORY : PF_ERR_CUDA; \
        }                                                              \
    } while (0)

template <typename T>
cudaError_t grow(T*& p, size_t& have, size_t need) {
    if (need <= have && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    have = 0;
    const size_t n = std::max<size_t>(need, 1);
    cudaError_t st = cudaMalloc(&p, n * sizeof(T));
    if (st == cudaSuccess) have = n;
    return st;
}

// Allocate plane scratch and launch pack + search.
// Order every use of the plane scratch after the previous one, whatever stream
// each runs on (a device call on a caller stream may still be reading it when
// the next call arrives on another stream).
cudaError_t scratch_acquire(DeviceState& d, cudaStream_t s) {
    if (!d.scratch_ev) {
        const cudaError_t st = cudaEventCreateWithFlags(&d.scratch_ev, cudaEventDisableTiming);
        if (st != cudaSuccess) return st;
        return cudaSuccess;  // never recorded yet: nothing to wait for
    }
    return cudaStreamWaitEvent(s, d.scratch_ev, 0);
}
cudaError_t scratch_release(DeviceState& d, cudaStream_t s) {
    return cudaEventRecord(d.scratch_ev, s);
}

cudaError_t launch_any_unordered(DeviceState& d, sb::FilterArgs a, cudaStream_t s);

cudaError_t launch_any(DeviceState& d, sb::FilterArgs a, cudaStream_t s) {
    cudaError_t st = scratch_acquire(d, s);
    if (st == cudaSuccess) st = launch_any_unordered(d, a, s);
    if (st == cudaSuccess) st = scratch_release(d, s);
    return st;
}

// Pack | search on disjoint SM partitions (split.cpp) for device-resident ASCII
// records with the width-4 search: PF_SPLIT = pack SMs (0 = off), PF_SPLIT_CHUNK =
// pairs per chunk. Read per call so that A/B sweeps can change them in-process.
int split_pack_sms_setting() {
    const char* e = std::getenv("PF_SPLIT");
    return e ? std::atoi(e) : 0;
}
long long split_chunk_setting() {
    const char* e = std::getenv("PF_SPLIT_CHUNK");
    const long long v = e ? std::atoll(e) : 0;
    return v > 0 ? v : (3ll << 20);
}

bool split_applies(const sb::FilterArgs& a) {
    return !a.nibbles && !a.dibits && !a.packed_text && a.stage_event == nullptr &&
           a.outplanes == nullptr && sb::use_fused(a.width, a.e, a.m) &&
           a.n >= 2 * split_chunk_setting();
}

sb::SplitPipe* split_pipe(DeviceState& d) {
    const int want = split_pack_sms_setting();  // < 0: shared mode (split.cpp)
    if (want == 0) return nullptr;
    if (d.split_sms != want) {
        sb::split_destroy(d.split);
        std::string why;
        d.split = sb::split_create(d.device, want, &why);
        d.split_sms = want;
        if (!d.split && std::getenv("PF_SPLIT_VERBOSE"))
            std::fprintf(stderr, "pf: SM split unavailable (%s); serial pack + search\n", why.c_str());
    }
    return d.split;
}

cudaError_t launch_any_unordered(DeviceState& d, sb::FilterArgs a, cudaStream_t s) {
    if (split_applies(a)) {
        if (sb::SplitPipe* sp = split_pipe(d)) return sb::split_launch(sp, a, s, split_chunk_setting());
    }
    const cudaError_t st = grow(d.d_scratch, d.scratch_words, sb::planes_scratch_words(a.n, a.m));
    if (st != cudaSuccess) return st;
    a.planes = d.d_scratch;
    a.planes_words = d.scratch_words;
    return sb::launch_filter(a, s);
}

// Bytes moved between host and device by the host entry points (bench.py
// reports them per step; pf_transfer_bytes).
std::atomic<uint64_t> g_h2d{0}, g_d2h{0};

cudaError_t xfer(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, cudaStream_t s) {
    (kind == cudaMemcpyHostToDevice ? g_h2d : g_d2h).fetch_add(bytes, std::memory_order_relaxed);
    return cudaMemcpyAsync(dst, src, bytes, kind, s);
}

bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// Host packing upload path: PF_HOST_PACK=0 disables it, =1 forces it for any
// batch size (A/B runs, tests); unset, batches of kHostPackMin pairs or more use it.
int host_pack_mode() {
    static const int v = [] {
        const char* e = std::getenv("PF_HOST_PACK");
        return e ? (e[0] == '0' ? 0 : 1) : -1;
    }();
    return v;
}
constexpr long long kHostPackMin = 1ll << 16;

// Upload format of the host-pack path: dibit records (2 bits per base, N
// planes only for chunks that contain an N; default) or nibble records
// (4 bits per base). PF_HOST_FORMAT=nibble selects the latter.
bool host_format_dibit() {
    static const bool v = [] {
        const char* e = std::getenv("PF_HOST_FORMAT");
        return !(e && std::strcmp(e, "nibble") == 0);
    }();
    return v;
}

// Pairs per host-pack chunk (PF_HOST_CHUNK overrides; multiple of 256).
long long host_chunk() {
    static const long long v = [] {
        const char* e = std::getenv("PF_HOST_CHUNK");
        long long c = e ? std::atoll(e) : (1ll << 18);
        c = std::max(256ll, c);
        return (c + 255) / 256 * 256;
    }();
    return v;
}

// Hybrid upload: when the host records are pinned, a second route DMAs raw
// ASCII chunks straight from them (200 B/pair of PCIe, no host CPU, device-side
// validation + pack) while the host cores pack the other chunks to dibits; the
// two routes take chunks from one counter, so each runs at its own pace.
// PF_HYBRID=1 turns it on (read per call; A/B runs).
bool hybrid_enabled() {
    const char* e = std::getenv("PF_HYBRID");
    return e && e[0] == '1';
}

void set_illegal(pf_error* err, uint64_t pair, uint32_t field, uint64_t pos, uint8_t byte) {
    if (!err) return;
    err->status = PF_ERR_ILLEGAL_CHARACTER;
    err->pair = pair;
    err->field = field;
    err->position = pos;
    err->byte = byte;
    std::snprintf(err->message, sizeof(err->message),
                  "illegal character '%c' at position %llu of %s %llu",
                  (byte >= 32 && byte < 127) ? byte : '?', (unsigned long long)pos,
                  field == 0 ? "text" : "pattern", (unsigned long long)pair);
}

// Decode the locator key and fill err (the byte is read from the records).
void decode_illegal(unsigned long long key, long long pair_base, const uint8_t* text,
                    const uint8_t* pattern, size_t stride, bool host_records, pf_error* err) {
    const unsigned long long pf = key >> 24;
    const uint64_t pair = pf / 2;
    const uint32_t field = static_cast<uint32_t>(pf % 2);
    const uint64_t pos = key & 0xFFFFFFull;
    uint8_t byte = 0;
    const uint8_t* src = (field == 0 ? text : pattern) + pair * stride + pos;
    if (host_records)
        byte = *src;
    else
        cudaMemcpy(&byte, src, 1, cudaMemcpyDeviceToHost);
    set_illegal(err, pair + static_cast<uint64_t>(pair_base), field, pos, byte);
}

struct ShardResult {
    int status = PF_OK;
    pf_error err{};
};

// Filter pairs [p0, p1) of host records on one device. With `dist` set the
// shard computes exact banded edit distances instead (validation, then the
// Myers kernel; accept/estimates/bits unused).
void run_host_shard(DeviceState& d, const uint8_t* text, const uint8_t* pattern, size_t stride,
                    size_t p0, size_t p1, uint32_t m, uint32_t e, uint32_t width,
                    uint32_t* accept_bitmap, uint32_t* estimates, uint64_t* bits, int32_t* dist,
                    bool magnet, ShardResult* res) {
    pf_error* err = &res->err;
    auto fail = [&](int st) { res->status = st; };
    const size_t n = p1 - p0;
    if (n == 0) return;
    if (cudaSetDevice(d.device) != cudaSuccess) return fail(PF_ERR_NO_DEVICE);
    // Pinned records whose stride is a multiple of 4 are used in place (one DMA
    // per sequence); anything else is re-pitched on the device to round4(m).
    const bool pinned = is_pinned(text) && is_pinned(pattern);
    const size_t pitch = (pinned && stride % 4 == 0) ? stride : pf_device_pitch(m);
    auto cu = [&](cudaError_t ce, const char* what) {
        if (ce == cudaSuccess) return true;
        set_err(err, ce == cudaErrorMemoryAllocation ? PF_ERR_OUT_OF_MEMORY : PF_ERR_CUDA, what, ce);
        fail(ce == cudaErrorMemoryAllocation ? PF_ERR_OUT_OF_MEMORY : PF_ERR_CUDA);
        return false;
    };
    const int hp_mode = host_pack_mode();
    // MAGNET reads the dibit records directly (no pack kernel), so it only
    // needs the dibit format and its own length limit.
    // The edit distance reads the dibit records directly too (m <= 1024).
    const bool shape_ok =
        dist     ? host_format_dibit() && m <= 1024
        : magnet ? host_format_dibit() && sb::magnet_supported(static_cast<int>(m))
                 : width >= 3 && width <= 8 && !bits &&
                       (host_format_dibit() ? sb::dibit_pack_fits(static_cast<int>(m))
                                            : sb::nibble_pack_fits(static_cast<int>(m)));
    const bool host_pack = hp_mode != 0 && e < m && shape_ok &&
                           (hp_mode == 1 || (static_cast<long long>(n) >= kHostPackMin &&
                                             // the portable packer is slower than PCIe
                                             sb::host_pack_uses_simd()));
    if (!host_pack) {
        if (!cu(grow(d.d_text, d.in_bytes, n * pitch), "alloc text")) return;
        if (!cu(grow(d.d_pattern, d.in_pattern_bytes, n * pitch), "alloc pattern")) return;
    }
    const size_t ngroups = (n + 31) / 32;
    if (!cu(grow(d.d_accept, d.accept_words, ngroups), "alloc accept")) return;
    if ((estimates || dist) && !cu(grow(d.d_est, d.est_n, n), "alloc estimates")) return;
    const size_t wpp = (m + 63) / 64;
    if (bits) {
        if (!cu(grow(d.d_bits, d.bits_words, n * wpp), "alloc bits")) return;
        if (!magnet &&
            !cu(grow(d.d_outplanes, d.outplanes_words, size_t(m) * ngroups), "alloc tally planes"))
            return;
    }
    if (!d.d_flag) {
        if (!cu(cudaMalloc(&d.d_flag, sizeof(uint32_t)), "alloc flag")) return;
        if (!cu(cudaMalloc(&d.d_key, sizeof(unsigned long long)), "alloc key")) return;
    }

    // ---- host packing upload path ---------------------------------------------
    // The host's cores pack records into dibit (or nibble) records
    // (host_pack.cpp) chunk by chunk into pinned buffers; chunk i's DMA, device
    // pack and search (or the MAGNET kernel, straight from the dibit records)
    // run on the stream while the cores pack chunk i+1.
    if (host_pack) {
        const bool dib = host_format_dibit();
        // pairs per chunk; a multiple of 256 so the pattern rows (at chunk * rp)
        // stay 16-byte aligned for the pack kernels' bulk copies
        const long long chunk =
            std::min<long long>((static_cast<long long>(n) + 255) / 256 * 256, host_chunk());
        const size_t rp = dib ? sb::dibit_pitch(static_cast<int>(m)) : sb::nibble_pitch(static_cast<int>(m));
        const size_t npr = sb::nplane_pitch(static_cast<int>(m));
        const size_t cbytes = 2 * static_cast<size_t>(chunk) * rp;  // text rows, then pattern rows
        const size_t nbytes = dib ? 2 * static_cast<size_t>(chunk) * npr : 0;
        if (d.h_nib_bytes < cbytes) {
            for (int b = 0; b < 2; ++b) {
                if (d.h_nib[b]) cudaFreeHost(d.h_nib[b]);
                d.h_nib[b] = nullptr;
            }
            d.h_nib_bytes = 0;
            for (int b = 0; b < 2; ++b)
                if (!cu(cudaHostAlloc(&d.h_nib[b], cbytes, cudaHostAllocPortable), "alloc host records"))
                    return;
            d.h_nib_bytes = cbytes;
        }
        if (d.h_nrow_bytes < nbytes) {
            for (int b = 0; b < 2; ++b) {
                if (d.h_nrow[b]) cudaFreeHost(d.h_nrow[b]);
                d.h_nrow[b] = nullptr;
            }
            d.h_nrow_bytes = 0;
            for (int b = 0; b < 2; ++b)
                if (!cu(cudaHostAlloc(&d.h_nrow[b], nbytes, cudaHostAllocPortable), "alloc host N rows"))
                    return;
            d.h_nrow_bytes = nbytes;
        }
        for (int b = 0; b < 2; ++b) {
            if (!cu(grow(d.d_nib[b], d.d_nib_bytes[b], cbytes), "alloc device records")) return;
            if (dib && !cu(grow(d.d_nrow[b], d.d_nrow_bytes[b], nbytes), "alloc device N rows")) return;
            if (!d.nib_ev[b] &&
                !cu(cudaEventCreateWithFlags(&d.nib_ev[b], cudaEventDisableTiming), "event"))
                return;
            if (!d.kern_ev[b] &&
                !cu(cudaEventCreateWithFlags(&d.kern_ev[b], cudaEventDisableTiming), "event"))
                return;
        }
        if (!d.copy_stream &&
            !cu(cudaStreamCreateWithFlags(&d.copy_stream, cudaStreamNonBlocking), "copy stream"))
            return;
        if (!d.up_ev && !cu(cudaEventCreateWithFlags(&d.up_ev, cudaEventDisableTiming), "event"))
            return;
        // uploads start after everything already queued on the device stream
        // (earlier batches' kernels may still read the device record buffers)
        if (!cu(cudaEventRecord(d.up_ev, d.stream), "record event") ||
            !cu(cudaStreamWaitEvent(d.copy_stream, d.up_ev, 0), "copy stream order"))
            return;
        if (!magnet && !dist &&
            !cu(grow(d.d_scratch, d.scratch_words, sb::planes_scratch_words(chunk, m)),
                "alloc planes"))
            return;
        const uint8_t* tsrc0 = text + p0 * stride;
        const uint8_t* psrc0 = pattern + p0 * stride;
        if (!cu(scratch_acquire(d, d.stream), "scratch order")) return;
        const long long nchunks = (static_cast<long long>(n) + chunk - 1) / chunk;
        // ---- hybrid: the raw-ASCII route on its own thread and stream ----------------
        const bool hybrid = !magnet && !dist && pinned && stride % 4 == 0 && nchunks >= 2 &&
                            hybrid_enabled() && sb::use_fused(width, e, static_cast<int>(m));
        std::atomic<long long> next_chunk{0};
        std::atomic<bool> stop{false};
        cudaError_t raw_err = cudaSuccess;
        std::thread raw_thread;
        if (hybrid) {
            const size_t rbytes = 2 * static_cast<size_t>(chunk) * stride;
            for (int b = 0; b < 2; ++b) {
                if (!cu(grow(d.d_raw[b], d.d_raw_bytes[b], rbytes), "alloc raw records")) return;
                if (!d.raw_ev[b] &&
                    !cu(cudaEventCreateWithFlags(&d.raw_ev[b], cudaEventDisableTiming), "event"))
                    return;
            }
            if (!d.raw_stream &&
                !cu(cudaStreamCreateWithFlags(&d.raw_stream, cudaStreamNonBlocking), "raw stream"))
                return;
            if (!d.raw_done &&
                !cu(cudaEventCreateWithFlags(&d.raw_done, cudaEventDisableTiming), "event"))
                return;
            if (!cu(grow(d.d_raw_scratch, d.raw_scratch_words, sb::planes_scratch_words(chunk, m)),
                    "alloc raw planes"))
                return;
            if (!d.d_raw_flag && !cu(cudaMalloc(&d.d_raw_flag, sizeof(uint32_t)), "alloc flag"))
                return;
            if (!cu(cudaStreamWaitEvent(d.raw_stream, d.up_ev, 0), "raw stream order") ||
                !cu(cudaMemsetAsync(d.d_raw_flag, 0, sizeof(uint32_t), d.raw_stream), "memset flag"))
                return;
            raw_thread = std::thread([&] {
                cudaError_t st = cudaSetDevice(d.device);
                for (long long k = 0; st == cudaSuccess && !stop.load(); ++k) {
                    const int b = static_cast<int>(k & 1);
                    // device buffer b is free once the kernels of this route's chunk k-2 are done
                    if (k >= 2 && (st = cudaEventSynchronize(d.raw_ev[b])) != cudaSuccess) break;
                    const long long i = next_chunk.fetch_add(1);
                    if (i >= nchunks) break;
                    const long long lo = i * chunk;
                    const long long cn = std::min<long long>(chunk, static_cast<long long>(n) - lo);
                    uint8_t* dt = d.d_raw[b];
                    uint8_t* dq = d.d_raw[b] + static_cast<size_t>(chunk) * stride;
                    const size_t bytes = static_cast<size_t>(cn - 1) * stride + m;
                    if ((st = xfer(dt, tsrc0 + lo * stride, bytes, cudaMemcpyHostToDevice,
                                   d.raw_stream)) != cudaSuccess ||
                        (st = xfer(dq, psrc0 + lo * stride, bytes, cudaMemcpyHostToDevice,
                                   d.raw_stream)) != cudaSuccess)
                        break;
                    if (stride > m &&  // the last record's padding is read, never used
                        ((st = cudaMemsetAsync(dt + bytes, 'A', stride - m, d.raw_stream)) != cudaSuccess ||
                         (st = cudaMemsetAsync(dq + bytes, 'A', stride - m, d.raw_stream)) != cudaSuccess))
                        break;
                    sb::FilterArgs ra{};
                    ra.text = dt;
                    ra.pattern = dq;
                    ra.pitch = stride;
                    ra.n = cn;
                    ra.m = static_cast<int>(m);
                    ra.e = e;
                    ra.width = width;
                    ra.accept = d.d_accept + lo / 32;
                    ra.estimates = estimates ? d.d_est + lo : nullptr;
                    ra.err_flag = d.d_raw_flag;
                    ra.planes = d.d_raw_scratch;
                    ra.planes_words = d.raw_scratch_words;
                    if ((st = sb::launch_filter(ra, d.raw_stream)) != cudaSuccess ||
                        (st = cudaEventRecord(d.raw_ev[b], d.raw_stream)) != cudaSuccess)
                        break;
                }
                if (st == cudaSuccess) st = cudaEventRecord(d.raw_done, d.raw_stream);
                raw_err = st;
            });
        }
        // The first illegal byte in pair order, whichever route met it: the host's
        // exact check over the whole shard (errors only).
        auto report_first_bad = [&]() {
            stop.store(true);
            if (raw_thread.joinable()) raw_thread.join();
            cudaStreamSynchronize(d.stream);
            if (d.raw_stream) cudaStreamSynchronize(d.raw_stream);
            sb::HostBad bad;
            sb::host_validate_parallel(tsrc0, psrc0, stride, static_cast<long long>(n),
                                       static_cast<int>(m), &bad);
            if (bad.any)
                set_illegal(err, p0 + bad.pair, static_cast<uint32_t>(bad.field),
                            static_cast<uint64_t>(bad.pos), bad.byte);
            fail(PF_ERR_ILLEGAL_CHARACTER);
        };
        struct JoinGuard {  // never leave the raw thread running on an early return
            std::thread& t;
            std::atomic<bool>& stop;
            ~JoinGuard() {
                stop.store(true);
                if (t.joinable()) t.join();
            }
        } join_guard{raw_thread, stop};
        for (long long k = 0;; ++k) {
            const long long i = hybrid ? next_chunk.fetch_add(1) : k;
            if (i >= nchunks) break;
            const int b = static_cast<int>(k & 1);
            const long long lo = i * chunk;
            const long long cn = std::min<long long>(chunk, static_cast<long long>(n) - lo);
            // the DMA that last read these pinned buffers (chunk k-2 of this route) must be done
            if (k >= 2 && !cu(cudaEventSynchronize(d.nib_ev[b]), "record buffer wait")) return;
            uint8_t* ht = d.h_nib[b];
            uint8_t* hq = ht + static_cast<size_t>(chunk) * rp;
            uint8_t* hnt = dib ? d.h_nrow[b] : nullptr;
            uint8_t* hnq = dib ? d.h_nrow[b] + static_cast<size_t>(chunk) * npr : nullptr;
            sb::HostBad bad;
            bool has_n = false;
            if (dib)
                sb::host_pack_dibits_parallel(tsrc0 + lo * stride, psrc0 + lo * stride, stride, cn,
                                              static_cast<int>(m), ht, hq, hnt, hnq, &bad, &has_n);
            else
                sb::host_pack_nibbles_parallel(tsrc0 + lo * stride, psrc0 + lo * stride, stride, cn,
                                               static_cast<int>(m), ht, hq, &bad);
            if (bad.any) {
                if (hybrid) return report_first_bad();  // the other route may hold an earlier one
                // one route: chunks run in pair order, the first chunk with a bad byte wins
                cu(cudaStreamSynchronize(d.stream), "sync");
                set_illegal(err, p0 + lo + bad.pair, static_cast<uint32_t>(bad.field),
                            static_cast<uint64_t>(bad.pos), bad.byte);
                return fail(PF_ERR_ILLEGAL_CHARACTER);
            }
            const size_t cb = static_cast<size_t>(cn) * rp;
            // device buffer b is free once chunk k-2's kernels (which read it) are done
            if (k >= 2 && !cu(cudaStreamWaitEvent(d.copy_stream, d.kern_ev[b], 0), "buffer order"))
                return;
            if (!cu(xfer(d.d_nib[b], ht, cb, cudaMemcpyHostToDevice, d.copy_stream), "H2D records"))
                return;
            if (!cu(xfer(d.d_nib[b] + static_cast<size_t>(chunk) * rp, hq, cb,
                         cudaMemcpyHostToDevice, d.copy_stream), "H2D records"))
                return;
            if (has_n) {
                const size_t nb = static_cast<size_t>(cn) * npr;
                if (!cu(xfer(d.d_nrow[b], hnt, nb, cudaMemcpyHostToDevice, d.copy_stream),
                        "H2D N rows"))
                    return;
                if (!cu(xfer(d.d_nrow[b] + static_cast<size_t>(chunk) * npr, hnq, nb,
                             cudaMemcpyHostToDevice, d.copy_stream), "H2D N rows"))
                    return;
            }
            // nib_ev[b]: this upload is done (host buffer b reusable; kernels may read)
            if (!cu(cudaEventRecord(d.nib_ev[b], d.copy_stream), "record event") ||
                !cu(cudaStreamWaitEvent(d.stream, d.nib_ev[b], 0), "upload order"))
                return;
            if (dist) {
                if (!cu(sb::launch_edit_distance_dibits(
                            d.d_nib[b], d.d_nib[b] + static_cast<size_t>(chunk) * rp,
                            has_n ? d.d_nrow[b] : nullptr,
                            has_n ? d.d_nrow[b] + static_cast<size_t>(chunk) * npr : nullptr, cn,
                            static_cast<int>(m), static_cast<int>(std::min<uint32_t>(e, 1u << 30)),
                            reinterpret_cast<int32_t*>(d.d_est) + lo, d.stream),
                        "edit distance kernel"))
                    return;
                if (!cu(cudaEventRecord(d.kern_ev[b], d.stream), "record event")) return;
                continue;
            }
            if (magnet) {
                if (!cu(sb::launch_magnet_dibits(
                            d.d_nib[b], d.d_nib[b] + static_cast<size_t>(chunk) * rp,
                            has_n ? d.d_nrow[b] : nullptr,
                            has_n ? d.d_nrow[b] + static_cast<size_t>(chunk) * npr : nullptr, cn,
                            static_cast<int>(m), static_cast<int>(e), d.d_accept + lo / 32,
                            estimates ? d.d_est + lo : nullptr,
                            bits ? d.d_bits + static_cast<size_t>(lo) * wpp : nullptr, d.stream),
                        "magnet kernel"))
                    return;
                if (!cu(cudaEventRecord(d.kern_ev[b], d.stream), "record event")) return;
                continue;
            }
            sb::FilterArgs a{};
            a.text = d.d_nib[b];
            a.pattern = d.d_nib[b] + static_cast<size_t>(chunk) * rp;
            a.pitch = rp;
            a.nibbles = !dib;
            a.dibits = dib;
            a.ntext = has_n ? d.d_nrow[b] : nullptr;
            a.npattern = has_n ? d.d_nrow[b] + static_cast<size_t>(chunk) * npr : nullptr;
            a.n = cn;
            a.m = static_cast<int>(m);
            a.e = e;
            a.width = width;
            a.accept = d.d_accept + lo / 32;
            a.estimates = estimates ? d.d_est + lo : nullptr;
            a.planes = d.d_scratch;
            a.planes_words = d.scratch_words;
            if (!cu(sb::launch_filter(a, d.stream), "filter kernel")) return;
            if (!cu(cudaEventRecord(d.kern_ev[b], d.stream), "record event")) return;
        }
        if (hybrid) {
            stop.store(false);
            raw_thread.join();
            if (!cu(raw_err, "raw route")) return;
            uint32_t raw_flag = 0;
            if (!cu(cudaMemcpyAsync(&raw_flag, d.d_raw_flag, sizeof(raw_flag),
                                    cudaMemcpyDeviceToHost, d.raw_stream), "D2H flag") ||
                !cu(cudaStreamSynchronize(d.raw_stream), "sync"))
                return;
            if (raw_flag) return report_first_bad();
            if (!cu(cudaStreamWaitEvent(d.stream, d.raw_done, 0), "raw route order")) return;
        }
        if (!cu(scratch_release(d, d.stream), "scratch order")) return;
        if (dist) {
            if (!cu(xfer(dist + p0, d.d_est, n * sizeof(int32_t), cudaMemcpyDeviceToHost, d.stream),
                    "D2H distances"))
                return;
            cu(cudaStreamSynchronize(d.stream), "sync");
            return;
        }
        if (!cu(xfer(accept_bitmap + p0 / 32, d.d_accept, ngroups * sizeof(uint32_t),
                                cudaMemcpyDeviceToHost, d.stream), "D2H accept"))
            return;
        if (estimates &&
            !cu(xfer(estimates + p0, d.d_est, n * sizeof(uint32_t),
                                cudaMemcpyDeviceToHost, d.stream), "D2H estimates"))
            return;
        if (bits && !cu(xfer(bits + p0 * wpp, d.d_bits, n * wpp * sizeof(uint64_t),
                             cudaMemcpyDeviceToHost, d.stream), "D2H bits"))
            return;
        cu(cudaStreamSynchronize(d.stream), "sync");
        return;
    }

    // ---- host -> device ----------------------------------------------------
    // Records land in the device layout (pitch = round4(m), or the caller's
    // 4-byte-multiple stride for pinned buffers). Pinned records already in that
    // layout are one DMA per sequence; other pinned strides are DMA'd
    // contiguously into a device staging slot and re-pitched by a kernel.
    // Pageable records are copied row by row into double-buffered pinned
    // staging at the device pitch (the host copy of chunk i+1 overlaps the DMA
    // of chunk i) and DMA'd straight into place.
    const uint8_t* tsrc = text + p0 * stride;
    const uint8_t* psrc = pattern + p0 * stride;
    if (pinned && stride == pitch) {
        const size_t bytes = (n - 1) * pitch + m;
        if (!cu(xfer(d.d_text, tsrc, bytes, cudaMemcpyHostToDevice, d.stream), "H2D text"))
            return;
        if (!cu(xfer(d.d_pattern, psrc, bytes, cudaMemcpyHostToDevice, d.stream),
                "H2D pattern"))
            return;
    } else if (pinned) {
        const size_t rows = std::max<size_t>(1, std::min(n, kStageBytes / stride));
        if (!cu(grow(d.d_stage, d.d_stage_bytes, 2 * rows * stride), "alloc device stage")) return;
        for (size_t r0 = 0; r0 < n; r0 += rows) {
            const size_t nr = std::min(rows, n - r0);
            const size_t bytes = (nr - 1) * stride + m;
            uint8_t* dt = d.d_stage;
            uint8_t* dp = d.d_stage + rows * stride;
            if (!cu(xfer(dt, tsrc + r0 * stride, bytes, cudaMemcpyHostToDevice, d.stream),
                    "H2D text"))
                return;
            if (!cu(xfer(dp, psrc + r0 * stride, bytes, cudaMemcpyHostToDevice, d.stream),
                    "H2D pattern"))
                return;
            if (!cu(sb::launch_repitch(dt, stride, d.d_text + r0 * pitch, pitch,
                                       static_cast<long long>(nr), static_cast<int>(m), d.stream),
                    "repitch text"))
                return;
            if (!cu(sb::launch_repitch(dp, stride, d.d_pattern + r0 * pitch, pitch,
                                       static_cast<long long>(nr), static_cast<int>(m), d.stream),
                    "repitch pattern"))
                return;
        }
    } else {
        const size_t rows = std::max<size_t>(1, std::min(n, kStageBytes / pitch));
        const size_t need = rows * pitch * 2;
        if (d.stage_bytes < need) {
            for (int b = 0; b < 2; ++b) {
                if (d.h_stage[b]) cudaFreeHost(d.h_stage[b]);
                d.h_stage[b] = nullptr;
                if (!cu(cudaHostAlloc(&d.h_stage[b], need, cudaHostAllocPortable), "alloc stage"))
                    return;
                if (!d.stage_ev[b] &&
                    !cu(cudaEventCreateWithFlags(&d.stage_ev[b], cudaEventDisableTiming), "event"))
                    return;
            }
            d.stage_bytes = need;
        }
        int buf = 0;
        for (size_t r0 = 0; r0 < n; r0 += rows, buf ^= 1) {
            const size_t nr = std::min(rows, n - r0);
            if (!cu(cudaEventSynchronize(d.stage_ev[buf]), "stage wait")) return;
            uint8_t* ht = d.h_stage[buf];
            uint8_t* hp = ht + rows * pitch;
            for (size_t r = 0; r < nr; ++r) {
                std::memcpy(ht + r * pitch, tsrc + (r0 + r) * stride, m);
                std::memcpy(hp + r * pitch, psrc + (r0 + r) * stride, m);
            }
            const size_t bytes = (nr - 1) * pitch + m;
            if (!cu(xfer(d.d_text + r0 * pitch, ht, bytes, cudaMemcpyHostToDevice, d.stream),
                    "H2D text"))
                return;
            if (!cu(xfer(d.d_pattern + r0 * pitch, hp, bytes, cudaMemcpyHostToDevice, d.stream),
                    "H2D pattern"))
                return;
            if (!cu(cudaEventRecord(d.stage_ev[buf], d.stream), "stage record")) return;
        }
    }
    if (pitch > m) {
        // the last record's padding is read by the tile copies (never used): define it
        const size_t tail = (n - 1) * pitch + m;
        if (!cu(cudaMemsetAsync(d.d_text + tail, 'A', pitch - m, d.stream), "pad text") ||
            !cu(cudaMemsetAsync(d.d_pattern + tail, 'A', pitch - m, d.stream), "pad pattern"))
            return;
    }

    // ---- kernels -----------------------------------------------------------
    if (!cu(cudaMemsetAsync(d.d_flag, 0, sizeof(uint32_t), d.stream), "memset flag")) return;
    sb::FilterArgs a{};
    a.text = d.d_text;
    a.pattern = d.d_pattern;
    a.pitch = pitch;
    a.n = static_cast<long long>(n);
    a.m = static_cast<int>(m);
    a.e = e;
    a.width = width;
    a.accept = d.d_accept;
    a.estimates = estimates ? d.d_est : nullptr;
    a.outplanes = bits && !magnet ? d.d_outplanes : nullptr;
    a.err_flag = d.d_flag;
    a.planes = d.d_scratch;
    a.planes_words = d.scratch_words;
    const bool short_circuit = e >= m;
    const bool bad_width = !dist && !magnet && (width < 3 || width > 8);
    auto report_illegal = [&]() {
        // the key is reset on the stream the locate kernel runs on (a legacy-stream
        // cudaMemcpy is not ordered with a non-blocking stream)
        if (!cu(cudaMemsetAsync(d.d_key, 0xFF, sizeof(unsigned long long), d.stream), "key init"))
            return;
        if (!cu(sb::launch_locate(d.d_text, d.d_pattern, pitch, a.n, a.m, d.d_key, d.stream),
                "locate"))
            return;
        unsigned long long key = 0;
        if (!cu(xfer(&key, d.d_key, sizeof(key), cudaMemcpyDeviceToHost, d.stream), "D2H key"))
            return;
        if (!cu(cudaStreamSynchronize(d.stream), "sync")) return;
        decode_illegal(key, static_cast<long long>(p0), tsrc, psrc, stride, true, err);
        fail(PF_ERR_ILLEGAL_CHARACTER);
    };
    if (!(short_circuit || bad_width || dist || magnet)) {
        // the filter itself: kernels, error flag and results in one round trip;
        // on an illegal byte the results are discarded and the byte located
        if (!cu(launch_any(d, a, d.stream), "filter kernel")) return;
        if (bits &&
            !cu(sb::launch_bits_transpose(d.d_outplanes, a.n, a.m, d.d_bits, d.stream), "bits"))
            return;
        uint32_t flag = 0;
        if (!cu(xfer(&flag, d.d_flag, sizeof(flag), cudaMemcpyDeviceToHost, d.stream), "D2H flag"))
            return;
        if (!cu(xfer(accept_bitmap + p0 / 32, d.d_accept, ngroups * sizeof(uint32_t),
                     cudaMemcpyDeviceToHost, d.stream), "D2H accept"))
            return;
        if (estimates && !cu(xfer(estimates + p0, d.d_est, n * sizeof(uint32_t),
                                  cudaMemcpyDeviceToHost, d.stream), "D2H estimates"))
            return;
        if (bits && !cu(xfer(bits + p0 * wpp, d.d_bits, n * wpp * sizeof(uint64_t),
                             cudaMemcpyDeviceToHost, d.stream), "D2H bits"))
            return;
        if (!cu(cudaStreamSynchronize(d.stream), "sync")) return;
        if (flag) report_illegal();
        return;
    }
    if (!cu(sb::launch_validate(a, d.stream), "validate")) return;
    uint32_t flag = 0;
    if (!cu(xfer(&flag, d.d_flag, sizeof(flag), cudaMemcpyDeviceToHost, d.stream),
            "D2H flag"))
        return;
    if (!cu(cudaStreamSynchronize(d.stream), "sync")) return;
    if (flag) return report_illegal();
    if (bad_width) return;  // caller reports invalid parameters after all shards validated
    if (dist) {
        int32_t* dd = reinterpret_cast<int32_t*>(d.d_est);
        if (!cu(sb::launch_edit_distance(d.d_text, d.d_pattern, pitch, a.n, a.m,
                                         static_cast<int>(std::min<uint32_t>(e, 1u << 30)), dd,
                                         d.stream),
                "edit distance kernel"))
            return;
        if (!cu(xfer(dist + p0, dd, n * sizeof(int32_t), cudaMemcpyDeviceToHost,
                                d.stream), "D2H distances"))
            return;
        cu(cudaStreamSynchronize(d.stream), "sync");
        return;
    }
    if (short_circuit) {
        if (!cu(sb::launch_accept_all(a.n, a.m, d.d_accept, estimates ? d.d_est : nullptr,
                                      bits ? d.d_bits : nullptr, d.stream),
                "accept_all"))
            return;
    } else if (magnet) {
        if (!cu(sb::launch_magnet(d.d_text, d.d_pattern, pitch, a.n, a.m, static_cast<int>(e),
                                  d.d_accept, estimates ? d.d_est : nullptr,
                                  bits ? d.d_bits : nullptr, d.stream),
                "magnet kernel"))
            return;
    }

    // ---- device -> host ------------------------------------------------------
    if (!cu(xfer(accept_bitmap + p0 / 32, d.d_accept, ngroups * sizeof(uint32_t),
                            cudaMemcpyDeviceToHost, d.stream), "D2H accept"))
        return;
    if (estimates &&
        !cu(xfer(estimates + p0, d.d_est, n * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                            d.stream), "D2H estimates"))
        return;
    if (bits &&
        !cu(xfer(bits + p0 * wpp, d.d_bits, n * wpp * sizeof(uint64_t),
                            cudaMemcpyDeviceToHost, d.stream), "D2H bits"))
        return;
    cu(cudaStreamSynchronize(d.stream), "sync");
}

const char* kStatusNames[] = {"ok", "empty sequence", "illegal character", "length mismatch",
                              "threshold too large", "out of band", "parse error",
                              "invalid parameters"};

}  // namespace

extern "C" {

const char* pf_status_string(int status) {
    if (status >= 0 && status <= 7) return kStatusNames[status];
    switch (status) {
        case PF_ERR_NO_DEVICE: return "no usable CUDA device";
        case PF_ERR_CUDA: return "CUDA error";
        case PF_ERR_OUT_OF_MEMORY: return "out of memory";
        case PF_ERR_NULL_ARGUMENT: return "null argument";
        default: return "unknown status";
    }
}

const char* pf_version(void) { return "shouji_b200 0.1 (sm_100a)"; }

int pf_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

size_t pf_device_pitch(uint32_t m) { return round_up(std::max<uint32_t>(m, 1), 4); }

uint64_t pf_launch_count(void) { return sb::launch_count(); }

void pf_transfer_bytes(uint64_t* h2d, uint64_t* d2h) {
    if (h2d) *h2d = g_h2d.load();
    if (d2h) *d2h = g_d2h.load();
}

double pf_host_read_bandwidth(const void* buf, size_t bytes, int passes) {
    return sb::host_read_gbs(static_cast<const uint8_t*>(buf), bytes, passes);
}

size_t pf_nibble_pitch(uint32_t m) { return sb::nibble_pitch(static_cast<int>(std::max<uint32_t>(m, 1))); }

int pf_host_pack_nibbles(const uint8_t* text, const uint8_t* pattern, size_t stride, size_t n,
                         uint32_t m, uint8_t* out_text, uint8_t* out_pattern, int simd,
                         pf_error* err) {
    if (err) std::memset(err, 0, sizeof(*err));
    if (n == 0) return PF_OK;
    if (!text || !pattern || !out_text || !out_pattern) return PF_ERR_NULL_ARGUMENT;
    if (m == 0) {
        set_err(err, PF_ERR_EMPTY_SEQUENCE, "empty sequence");
        return PF_ERR_EMPTY_SEQUENCE;
    }
    if (stride < m) {
        set_err(err, PF_ERR_INVALID_PARAMETERS, "stride < m");
        return PF_ERR_INVALID_PARAMETERS;
    }
    sb::HostBad bad;
    sb::host_pack_nibbles_parallel(text, pattern, stride, static_cast<long long>(n),
                                   static_cast<int>(m), out_text, out_pattern, &bad, 0, simd != 0);
    if (bad.any) {
        set_illegal(err, bad.pair, static_cast<uint32_t>(bad.field), static_cast<uint64_t>(bad.pos),
                    bad.byte);
        return PF_ERR_ILLEGAL_CHARACTER;
    }
    return PF_OK;
}

int pf_shouji_filter_nibbles_device(pf_ctx* ctx, const uint8_t* d_text, const uint8_t* d_pattern,
                                    size_t n, uint32_t m, uint32_t e, uint32_t width,
                                    uint32_t* d_accept_bitmap, uint32_t* d_estimates, void* stream,
                                    pf_error* err) {
    if (err) std::memset(err, 0, sizeof(*err));
    if (!ctx) return PF_ERR_NULL_ARGUMENT;
    if (n == 0) return PF_OK;
    if (!d_text || !d_pattern || !d_accept_bitmap) return PF_ERR_NULL_ARGUMENT;
    if (m == 0 || e >= m || width < 3 || width > 8 || !sb::nibble_pack_fits(static_cast<int>(m)) ||
        reinterpret_cast<uintptr_t>(d_text) % 16 || reinterpret_cast<uintptr_t>(d_pattern) % 16) {
        set_err(err, PF_ERR_INVALID_PARAMETERS,
                "nibble path needs e < m, 3 <= width <= 8, a record that fits a pack tile and "
                "16-byte aligned record arrays");
        return PF_ERR_INVALID_PARAMETERS;
    }
    std::lock_guard<std::mutex> lock(ctx->mu);
    DeviceState& d = ctx->devs[0];
    PF_CUDA(cudaSetDevice(d.device));
    PF_CUDA(grow(d.d_scratch, d.scratch_words,
                 sb::planes_scratch_words(static_cast<long long>(n), static_cast<int>(m))));
    sb::FilterArgs a{};
    a.text = d_text;
    a.pattern = d_pattern;
    a.pitch = sb::nibble_pitch(static_cast<int>(m));
    a.nibbles = true;
    a.n = static_cast<long long>(n);
    a.m = static_cast<int>(m);
    a.e = e;
    a.width = width;
    a.accept = d_accept_bitmap;
    a.estimates = d_estimates;
    a.planes = d.d_scratch;
    a.planes_words = d.scratch_words;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    PF_CUDA(scratch_acquire(d, s));
    PF_CUDA(sb::launch_filter(a, s));
    PF_CUDA(scratch_release(d, s));
    return PF_OK;
}

size_t pf_dibit_pitch(uint32_t m) { return sb::dibit_pitch(static_cast<int>(std::max<uint32_t>(m, 1))); }
size_t pf_nplane_pitch(uint32_t m) { return sb::nplane_pitch(static_cast<int>(std::max<uint32_t>(m, 1))); }

int pf_host_pack_dibits(const uint8_t* text, const uint8_t* pattern, size_t stride, size_t n,
                        uint32_t m, uint8_t* out_text, uint8_t* out_pattern, uint8_t* n_text,
                        uint8_t* n_pattern, int* has_n, int simd, pf_error* err) {
    if (err) std::memset(err, 0, sizeof(*err));
    if (has_n) *has_n = 0;
    if (n == 0) return PF_OK;
    if (!text || !pattern || !out_text || !out_pattern || !has_n) return PF_ERR_NULL_ARGUMENT;
    if (m == 0) {
        set_err(err, PF_ERR_EMPTY_SEQUENCE, "empty sequence");
        return PF_ERR_EMPTY_SEQUENCE;
    }
    if (stride < m) {
        set_err(err, PF_ERR_INVALID_PARAMETERS, "stride < m");
        return PF_ERR_INVALID_PARAMETERS;
    }
    sb::HostBad bad;
    bool any = false;
    sb::host_pack_dibits_parallel(text, pattern, stride, static_cast<long long>(n),
                                  static_cast<int>(m), out_text, out_pattern, n_text, n_pattern,
                                  &bad, &any, simd != 0);
    if (bad.any) {
        set_illegal(err, bad.pair, static_cast<uint32_t>(bad.field), static_cast<uint64_t>(bad.pos),
                    bad.byte);
        return PF_ERR_ILLEGAL_CHARACTER;
    }
    *has_n = any ? 1 : 0;
    return PF_OK;
}

int pf_shouji_filter_dibits_device(pf_ctx* ctx, const uint8_t* d_text, const uint8_t* d_pattern,
                                   const uint8_t* d_ntext, const uint8_t* d_npattern, size_t n,
                                   uint32_t m, uint32_t e, uint32_t width,
                                   uint32_t* d_accept_bitmap, uint32_t* d_estimates, void* stream,
                                   pf_error* err) {
    if (err) std::memset(err, 0, sizeof(*err));
    if (!ctx) return PF_ERR_NULL_ARGUMENT;
    if (n == 0) return PF_OK;
    if (!d_text || !d_pattern || !d_accept_bitmap || (!d_ntext != !d_npattern))
        return PF_ERR_NULL_ARGUMENT;
    const uintptr_t al = reinterpret_cast<uintptr_t>(d_text) | reinterpret_cast<uintptr_t>(d_pattern) |
                         reinterpret_cast<uintptr_t>(d_ntext) | reinterpret_cast<uintptr_t>(d_npattern);
    if (m == 0 || e >= m || width < 3 || width > 8 || !sb::dibit_pack_fits(static_cast<int>(m)) ||
        al % 16) {
        set_err(err, PF_ERR_INVALID_PARAMETERS,
                "dibit path needs e < m, 3 <= width <= 8, a record that fits a pack tile and "
                "16-byte aligned record arrays");
        return PF_ERR_INVALID_PARAMETERS;
    }
    std::lock_guard<std::mutex> lock(ctx->mu);
    DeviceState& d = ctx->devs[0];
    PF_CUDA(cudaSetDevice(d.device));
    PF_CUDA(grow(d.d_scratch, d.scratch_words,
                 sb::planes_scratch_words(static_cast<long long>(n), static_cast<int>(m))));
    sb::FilterArgs a{};
    a.text = d_text;
    a.pattern = d_pattern;
    a.dibits = true;
    a.ntext = d_ntext;
    a.npattern = d_npattern;
    a.pitch = sb::dibit_pitch(static_cast<int>(m));
    a.n = static_cast<long long>(n);
    a.m = static_cast<int>(m);
    a.e = e;
    a.width = width;
    a.accept = d_accept_bitmap;
    a.estimates = d_estimates;
    a.planes = d.d_scratch;
    a.planes_words = d.scratch_words;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    PF_CUDA(scratch_acquire(d, s));
    PF_CUDA(sb::launch_filter(a, s));
    PF_CUDA(scratch_release(d, s));
    return PF_OK;
}

int pf_ctx_create(const int* devices, int count, pf_ctx** out) {
    if (!out) return PF_ERR_NULL_ARGUMENT;
    *out = nullptr;
    const int ndev = pf_device_count();
    if (ndev <= 0) return PF_ERR_NO_DEVICE;
    std::vector<int> ids;
    if (!devices || count <= 0)
        ids.push_back(0);
    else
        ids.assign(devices, devices + count);
    auto* ctx = new pf_ctx;
    for (int id : ids) {
        if (id < 0 || id >= ndev) {
            pf_ctx_destroy(ctx);
            return PF_ERR_NO_DEVICE;
        }
        DeviceState d;
        d.device = id;
        if (cudaSetDevice(id) != cudaSuccess ||
            cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking) != cudaSuccess) {
            cudaGetLastError();
            pf_ctx_destroy(ctx);
            return PF_ERR_NO_DEVICE;
        }
        cudaDeviceProp prop{};
        cudaGetDeviceProperties(&prop, id);
        if (prop.major < 10) {  // kernels are built for sm_100a only
            cudaStreamDestroy(d.stream);
            pf_ctx_destroy(ctx);
            return PF_ERR_NO_DEVICE;
        }
        ctx->devs.push_back(d);
    }
    *out = ctx;
    return PF_OK;
}

void pf_ctx_destroy(pf_ctx* ctx) {
    if (!ctx) return;
    for (auto& d : ctx->devs) {
        cudaSetDevice(d.device);
        if (d.stream) cudaStreamSynchronize(d.stream);
        cudaFree(d.d_text);
        cudaFree(d.d_pattern);
        cudaFree(d.d_accept);
        cudaFree(d.d_est);
        cudaFree(d.d_bits);
        cudaFree(d.d_outplanes);
        cudaFree(d.d_scratch);
        if (d.scratch_ev) cudaEventDestroy(d.scratch_ev);
        sb::split_destroy(d.split);
        d.split = nullptr;
        if (d.raw_stream) {
            cudaStreamSynchronize(d.raw_stream);
            cudaStreamDestroy(d.raw_stream);
        }
        for (int b = 0; b < 2; ++b) {
            cudaFree(d.d_raw[b]);
            if (d.raw_ev[b]) cudaEventDestroy(d.raw_ev[b]);
        }
        if (d.raw_done) cudaEventDestroy(d.raw_done);
        cudaFree(d.d_raw_scratch);
        cudaFree(d.d_raw_flag);
        if (d.h_small_in) cudaFreeHost(d.h_small_in);
        if (d.h_small_out) cudaFreeHost(d.h_small_out);
        cudaFree(d.d_small_counter);
        cudaFree(d.d_flag);
        cudaFree(d.d_key);
        cudaFree(d.d_stage);
        for (int b = 0; b < 2; ++b) {
            if (d.h_nib[b]) cudaFreeHost(d.h_nib[b]);
            cudaFree(d.d_nib[b]);
            if (d.h_nrow[b]) cudaFreeHost(d.h_nrow[b]);
            cudaFree(d.d_nrow[b]);
            if (d.nib_ev[b]) cudaEventDestroy(d.nib_ev[b]);
            if (d.h_pk[b]) cudaFreeHost(d.h_pk[b]);
            cudaFree(d.d_pk[b]);
            if (d.pk_ev[b]) cudaEventDestroy(d.pk_ev[b]);
            if (d.kern_ev[b]) cudaEventDestroy(d.kern_ev[b]);
        }
        if (d.up_ev) cudaEventDestroy(d.up_ev);
        if (d.copy_stream) {
            cudaStreamSynchronize(d.copy_stream);
            cudaStreamDestroy(d.copy_stream);
        }
        for (int b = 0; b < 2; ++b) {
            if (d.h_stage[b]) cudaFreeHost(d.h_stage[b]);
            if (d.stage_ev[b]) cudaEventDestroy(d.stage_ev[b]);
        }
        if (d.stream) cudaStreamDestroy(d.stream);
    }
    delete ctx;
}

int pf_ctx_device_count(const pf_ctx* ctx) { return ctx ? static_cast<int>(ctx->devs.size()) : 0; }

int pf_ctx_set_shard_chunk(pf_ctx* ctx, size_t chunk_pairs) {
    if (!ctx) return PF_ERR_NULL_ARGUMENT;
    std::lock_guard<std::mutex> lock(ctx->mu);
    ctx->shard_chunk = chunk_pairs == 0 ? 0 : (chunk_pairs + 31) / 32 * 32;
    return PF_OK;
}

}  // extern "C"

namespace {

// Pre-packed pairs [p0, p1) (packed_sequence plane words, pf_packed_words(m)
// u64 per sequence per pair) on one device: chunked H2D (pinned caller
// buffers are DMA'd in place, pageable ones are copied into double-buffered
// pinned staging by the host pool while the previous chunk is in flight),
// re-slice + search per chunk, outputs gathered at the end.
void run_packed_shard(DeviceState& d, const uint64_t* text, const uint64_t* pattern, size_t p0,
                      size_t p1, uint32_t m, uint32_t e, uint32_t width, uint32_t* accept_bitmap,
                      uint32_t* estimates, uint64_t* bits, ShardResult* res) {
    pf_error* err = &res->err;
    auto fail = [&](int st) { res->status = st; };
    auto cu = [&](cudaError_t ce, const char* what) {
        if (ce == cudaSuccess) return true;
        set_err(err, ce == cudaErrorMemoryAllocation ? PF_ERR_OUT_OF_MEMORY : PF_ERR_CUDA, what, ce);
        fail(ce == cudaErrorMemoryAllocation ? PF_ERR_OUT_OF_MEMORY : PF_ERR_CUDA);
        return false;
    };
    const size_t n = p1 - p0;
    if (n == 0) return;
    if (cudaSetDevice(d.device) != cudaSuccess) return fail(PF_ERR_NO_DEVICE);
    const size_t pw = pf_packed_words(m);  // u64 words per sequence per pair
    const size_t ngroups = (n + 31) / 32;
    const size_t wpp = (m + 63) / 64;
    if (!cu(grow(d.d_accept, d.accept_words, ngroups), "alloc accept")) return;
    if (estimates && !cu(grow(d.d_est, d.est_n, n), "alloc estimates")) return;
    if (bits && !cu(grow(d.d_bits, d.bits_words, n * wpp), "alloc bits")) return;
    if (e >= m) {  // shouji.cpp:48-49
        if (!cu(sb::launch_accept_all(static_cast<long long>(n), static_cast<int>(m), d.d_accept,
                                      estimates ? d.d_est : nullptr, bits ? d.d_bits : nullptr,
                                      d.stream),
                "accept_all"))
            return;
    } else {
        const bool pinned = is_pinned(text) && is_pinned(pattern);
        const long long chunk = std::min<long long>((static_cast<long long>(n) + 255) / 256 * 256,
                                                    1ll << 20);
        const size_t cwords = static_cast<size_t>(chunk) * pw;
        for (int b = 0; b < 2; ++b) {
            if (!cu(grow(d.d_pk[b], d.d_pk_words[b], 2 * cwords), "alloc packed chunk")) return;
            if (!d.pk_ev[b] &&
                !cu(cudaEventCreateWithFlags(&d.pk_ev[b], cudaEventDisableTiming), "event"))
                return;
        }
        if (!pinned && d.h_pk_words < 2 * cwords) {
            for (int b = 0; b < 2; ++b) {
                if (d.h_pk[b]) cudaFreeHost(d.h_pk[b]);
                d.h_pk[b] = nullptr;
            }
            d.h_pk_words = 0;
            for (int b = 0; b < 2; ++b)
                if (!cu(cudaHostAlloc(&d.h_pk[b], 2 * cwords * 8, cudaHostAllocPortable),
                        "alloc packed staging"))
                    return;
            d.h_pk_words = 2 * cwords;
        }
        if (!cu(grow(d.d_scratch, d.scratch_words, sb::planes_scratch_words(chunk, m)),
                "alloc planes"))
            return;
        if (bits && !cu(grow(d.d_outplanes, d.outplanes_words,
                             size_t(m) * static_cast<size_t>((chunk + 31) / 32)),
                        "alloc tally planes"))
            return;
        if (!cu(scratch_acquire(d, d.stream), "scratch order")) return;
        const long long nchunks = (static_cast<long long>(n) + chunk - 1) / chunk;
        for (long long i = 0; i < nchunks; ++i) {
            const int b = static_cast<int>(i & 1);
            const long long lo = i * chunk;
            const long long cn = std::min<long long>(chunk, static_cast<long long>(n) - lo);
            const uint64_t* st = text + (p0 + lo) * pw;
            const uint64_t* sp = pattern + (p0 + lo) * pw;
            const size_t cb = static_cast<size_t>(cn) * pw * 8;
            if (!pinned) {
                // the DMA that last read this staging buffer (chunk i-2) must be done
                if (i >= 2 && !cu(cudaEventSynchronize(d.pk_ev[b]), "staging wait")) return;
                sb::host_copy_parallel(d.h_pk[b], st, cb);
                sb::host_copy_parallel(d.h_pk[b] + cwords, sp, cb);
                st = d.h_pk[b];
                sp = d.h_pk[b] + cwords;
            }
            if (!cu(xfer(d.d_pk[b], st, cb, cudaMemcpyHostToDevice, d.stream), "H2D planes")) return;
            if (!cu(xfer(d.d_pk[b] + cwords, sp, cb, cudaMemcpyHostToDevice, d.stream),
                    "H2D planes"))
                return;
            if (!cu(cudaEventRecord(d.pk_ev[b], d.stream), "staging record")) return;
            sb::FilterArgs a{};
            a.packed_text = d.d_pk[b];
            a.packed_pattern = d.d_pk[b] + cwords;
            a.n = cn;
            a.m = static_cast<int>(m);
            a.e = e;
            a.width = width;
            a.accept = d.d_accept + lo / 32;
            a.estimates = estimates ? d.d_est + lo : nullptr;
            a.outplanes = bits ? d.d_outplanes : nullptr;
            a.planes = d.d_scratch;
            a.planes_words = d.scratch_words;
            if (!cu(sb::launch_filter(a, d.stream), "filter kernel")) return;
            if (bits && !cu(sb::launch_bits_transpose(d.d_outplanes, cn, static_cast<int>(m),
                                                      d.d_bits + static_cast<size_t>(lo) * wpp,
                                                      d.stream),
                            "bits"))
                return;
        }
        if (!cu(scratch_release(d, d.stream), "scratch order")) return;
    }
    if (!cu(xfer(accept_bitmap + p0 / 32, d.d_accept, ngroups * sizeof(uint32_t),
                 cudaMemcpyDeviceToHost, d.stream), "D2H accept"))
        return;
    if (estimates && !cu(xfer(estimates + p0, d.d_est, n * sizeof(uint32_t),
                              cudaMemcpyDeviceToHost, d.stream), "D2H estimates"))
        return;
    if (bits && !cu(xfer(bits + p0 * wpp, d.d_bits, n * wpp * sizeof(uint64_t),
                         cudaMemcpyDeviceToHost, d.stream), "D2H bits"))
        return;
    cu(cudaStreamSynchronize(d.stream), "sync");
}

// Shard boundaries of an n-pair host batch over nd devices: nd contiguous
// 32-aligned shards (parallel_for_pairs' n*t/T split, evaluate.cpp:36-37), or,
// with a shard chunk, consecutive chunks that the devices take round-robin
// (shard k on device k mod nd). Every boundary is a multiple of 32, so bitmap
// words never straddle devices.
std::vector<size_t> shard_bounds(size_t n, size_t nd, size_t chunk) {
    std::vector<size_t> b;
    if (chunk == 0 || nd == 1) {
        const size_t groups = (n + 31) / 32;
        for (size_t t = 0; t <= nd; ++t) b.push_back(std::min(n, groups * t / nd * 32));
        return b;
    }
    for (size_t p = 0; p < n; p += chunk) b.push_back(p);
    b.push_back(n);
    return b;
}

// ---- latency path: small batches ------------------------------------------------
// A per-pair caller (shouji_filter's signature, or the drop-in's coalesced
// handful of pairs) pays one launch of the latency kernel (small.cu) and one
// synchronisation: inputs are copied into mapped pinned staging that the kernel
// reads in place, and the kernel writes the bitmap, estimates and tally words
// straight back into mapped memory. PF_SMALL=0 turns it off (A/B runs).
bool small_applies(size_t n, uint32_t m) {
    const char* env = std::getenv("PF_SMALL");  // read per call: tests A/B both paths
    const bool on = !(env && env[0] == '0');
    return on && n <= static_cast<size_t>(sb::kSmallMaxN) && m <= static_cast<uint32_t>(sb::kSmallMaxM);
}

cudaError_t grow_mapped(uint8_t*& h, uint8_t*& dptr, size_t& have, size_t need) {
    if (need <= have && h) return cudaSuccess;
    if (h) cudaFreeHost(h);
    h = dptr = nullptr;
    have = 0;
    cudaError_t st = cudaHostAlloc(reinterpret_cast<void**>(&h), need,
                                   cudaHostAllocMapped | cudaHostAllocPortable);
    if (st != cudaSuccess) return st;
    st = cudaHostGetDevicePointer(reinterpret_cast<void**>(&dptr), h, 0);
    if (st != cudaSuccess) return st;
    have = need;
    return cudaSuccess;
}

int run_small(DeviceState& d, const uint8_t* text, const uint8_t* pattern, size_t stride,
              const uint64_t* tplanes, const uint64_t* pplanes, size_t n, uint32_t m, uint32_t e,
              uint32_t width, uint32_t* accept_bitmap, uint32_t* estimates, uint64_t* bits,
              pf_error* err) {
    PF_CUDA(cudaSetDevice(d.device));
    const size_t W = (m + 63) / 64;
    const size_t acc_words = (n + 31) / 32;
    const size_t in_bytes = text ? 2 * n * m : 2 * n * 3 * W * sizeof(uint64_t);
    // out: key (8 B), done flag (8 B), bits (n*W u64), estimates, accept bytes
    const size_t off_done = 8, off_bits = 16, off_est = off_bits + n * W * 8, off_acc = off_est + n * 4;
    const size_t out_bytes = off_acc + n;
    PF_CUDA(grow_mapped(d.h_small_in, d.d_small_in, d.small_in_bytes, std::max<size_t>(in_bytes, 4096)));
    PF_CUDA(grow_mapped(d.h_small_out, d.d_small_out, d.small_out_bytes, std::max<size_t>(out_bytes, 4096)));
    sb::SmallArgs a{};
    if (text) {
        for (size_t i = 0; i < n; ++i) {
            std::memcpy(d.h_small_in + i * m, text + i * stride, m);
            std::memcpy(d.h_small_in + (n + i) * m, pattern + i * stride, m);
        }
        a.text = d.d_small_in;
        a.pattern = d.d_small_in + n * m;
        a.stride = m;
    } else {
        const size_t pw = 3 * W;
        std::memcpy(d.h_small_in, tplanes, n * pw * 8);
        std::memcpy(d.h_small_in + n * pw * 8, pplanes, n * pw * 8);
        a.tplanes = reinterpret_cast<const uint64_t*>(d.d_small_in);
        a.pplanes = reinterpret_cast<const uint64_t*>(d.d_small_in + n * pw * 8);
    }
    auto* key = reinterpret_cast<volatile unsigned long long*>(d.h_small_out);
    *key = ~0ull;
    a.n = static_cast<int>(n);
    a.m = static_cast<int>(m);
    a.e = e;
    a.w = static_cast<int>(width);
    a.accept = d.d_small_out + off_acc;
    a.est = reinterpret_cast<uint32_t*>(d.d_small_out + off_est);
    a.bits = bits ? reinterpret_cast<uint64_t*>(d.d_small_out + off_bits) : nullptr;
    a.bad_key = text ? reinterpret_cast<unsigned long long*>(d.d_small_out) : nullptr;
    if (!d.d_small_counter) {
        PF_CUDA(cudaMalloc(&d.d_small_counter, sizeof(unsigned)));
        PF_CUDA(cudaMemset(d.d_small_counter, 0, sizeof(unsigned)));
    }
    a.counter = d.d_small_counter;
    a.done = reinterpret_cast<volatile unsigned*>(d.d_small_out + off_done);
    a.seq = ++d.small_seq;
    auto* done = reinterpret_cast<volatile unsigned*>(d.h_small_out + off_done);
    PF_CUDA(sb::launch_small(a, d.stream));
    // completion: the kernel's last CTA publishes seq into mapped memory after a
    // system fence; polling it costs less than a stream synchronisation. The
    // stream is queried now and then so that a failed launch cannot spin forever.
    for (unsigned spin = 1; *done != a.seq; ++spin) {
        if ((spin & 255) == 0) {
            const cudaError_t q = cudaStreamQuery(d.stream);
            if (q == cudaErrorNotReady) continue;
            PF_CUDA(q);
            if (*done != a.seq) {  // stream idle but no flag: should not happen
                set_err(err, PF_ERR_CUDA, "latency kernel finished without its completion flag");
                return PF_ERR_CUDA;
            }
        }
    }
    if (text && *key != ~0ull) {
        decode_illegal(*key, 0, text, pattern, stride, true, err);
        return PF_ERR_ILLEGAL_CHARACTER;
    }
    if (width < 3 || width > 8) {  // window_zero_table ctor (shouji.cpp:9-15)
        set_err(err, PF_ERR_INVALID_PARAMETERS, "window width must be in [3, 8]");
        return PF_ERR_INVALID_PARAMETERS;
    }
    std::memset(accept_bitmap, 0, acc_words * 4);
    const uint8_t* acc8 = d.h_small_out + off_acc;
    for (size_t i = 0; i < n; ++i)
        if (acc8[i]) accept_bitmap[i / 32] |= 1u << (i % 32);
    if (estimates) std::memcpy(estimates, d.h_small_out + off_est, n * 4);
    if (bits) std::memcpy(bits, d.h_small_out + off_bits, n * W * 8);
    return PF_OK;
}

int run_batch(pf_ctx* ctx, const uint8_t* text, const uint8_t* pattern, size_t stride, size_t n,
              uint32_t m, uint32_t e, uint32_t width, uint32_t* accept_bitmap, uint32_t* estimates,
              uint64_t* bits, int32_t* dist, pf_error* err, bool magnet = false) {
    if (err) std::memset(err, 0, sizeof(*err));
    if (!ctx) return PF_ERR_NULL_ARGUMENT;
    if (n == 0) return PF_OK;
    if (!text || !pattern || (!accept_bitmap && !dist)) return PF_ERR_NULL_ARGUMENT;
    if (m == 0) {  // packed_sequence::from_string("") (packed_sequence.cpp:8)
        set_err(err, PF_ERR_EMPTY_SEQUENCE, "empty sequence");
        return PF_ERR_EMPTY_SEQUENCE;
    }
    if (stride < m || m >= (1u << 24) || (dist && m > 1024) ||
        (magnet && e < m && !sb::magnet_supported(static_cast<int>(m)))) {
        set_err(err, PF_ERR_INVALID_PARAMETERS,
                dist     ? "stride < m or m > 1024 (edit distance)"
                : magnet ? "stride < m or m > 512 (MAGNET)"
                         : "stride < m or m >= 2^24");
        return PF_ERR_INVALID_PARAMETERS;
    }
    std::lock_guard<std::mutex> lock(ctx->mu);
    if (!dist && !magnet && small_applies(n, m))
        return run_small(ctx->devs[0], text, pattern, stride, nullptr, nullptr, n, m, e, width,
                         accept_bitmap, estimates, bits, err);
    const size_t nd = ctx->devs.size();
    const std::vector<size_t> bounds = shard_bounds(n, nd, ctx->shard_chunk);
    const size_t nshards = bounds.size() - 1;
    std::vector<ShardResult> res(nshards);
    auto work = [&](size_t t) {  // device t runs shards t, t+nd, ... in order
        for (size_t k = t; k < nshards; k += nd) {
            run_host_shard(ctx->devs[t], text, pattern, stride, bounds[k], bounds[k + 1], m, e,
                           width, accept_bitmap, estimates, bits, dist, magnet, &res[k]);
            if (res[k].status != PF_OK) break;
        }
    };
    if (nd == 1) {
        work(0);
    } else {
        std::vector<std::thread> pool;
        for (size_t t = 0; t < nd; ++t) pool.emplace_back(work, t);
        for (auto& th : pool) th.join();
    }
    // First failure in pair order wins (illegal characters are located per
    // shard; shards are in pair order).
    for (size_t k = 0; k < nshards; ++k) {
        if (res[k].status != PF_OK) {
            if (err) *err = res[k].err;
            if (err) err->status = res[k].status;
            return res[k].status;
        }
    }
    if (!dist && !magnet && (width < 3 || width > 8)) {  // window_zero_table ctor (shouji.cpp:9-15)
        set_err(err, PF_ERR_INVALID_PARAMETERS, "window width must be in [3, 8]");
        return PF_ERR_INVALID_PARAMETERS;
    }
    return PF_OK;
}

}  // namespace

extern "C" {

int pf_shouji_filter_batch(pf_ctx* ctx, const uint8_t* text, const uint8_t* pattern, size_t stride,
                           size_t n, uint32_t m, uint32_t e, uint32_t width,
                           uint32_t* accept_bitmap, uint32_t* estimates, uint64_t* bits,
                           pf_error* err) {
    return run_batch(ctx, text, pattern, stride, n, m, e, width, accept_bitmap, estimates, bits,
                     nullptr, err);
}

int pf_magnet_filter_batch(pf_ctx* ctx, const uint8_t* text, const uint8_t* pattern, size_t stride,
                           size_t n, uint32_t m, uint32_t e, uint32_t* accept_bitmap,
                           uint32_t* estimates, uint64_t* bits, pf_error* err) {
    return run_batch(ctx, text, pattern, stride, n, m, e, 4, accept_bitmap, estimates, bits,
                     nullptr, err, true);
}

int pf_magnet_filter_device(pf_ctx* ctx, const uint8_t* d_text, const uint8_t* d_pattern,
                            size_t pitch, size_t n, uint32_t m, uint32_t e,
                            uint32_t* d_accept_bitmap, uint32_t* d_estimates, uint64_t* d_bits,
                            void* stream, pf_error* err) {
    if (err) std::memset(err, 0, sizeof(*err));
    if (!ctx) return PF_ERR_NULL_ARGUMENT;
    if (n == 0) return PF_OK;
    if (!d_text || !d_pattern || !d_accept_bitmap) return PF_ERR_NULL_ARGUMENT;
    if (m == 0) {
        set_err(err, PF_ERR_EMPTY_SEQUENCE, "empty sequence");
        return PF_ERR_EMPTY_SEQUENCE;
    }
    if (pitch % 4 != 0 || pitch < m ||
        (reinterpret_cast<uintptr_t>(d_text) | reinterpret_cast<uintptr_t>(d_pattern)) % 16 != 0 ||
        m >= (1u << 24) || (e < m && !sb::magnet_supported(static_cast<int>(m)))) {
        set_err(err, PF_ERR_INVALID_PARAMETERS,
                "device records need 16-byte aligned bases, pitch % 4 == 0, pitch >= m, m <= 512");
        return PF_ERR_INVALID_PARAMETERS;
    }
    std::lock_guard<std::mutex> lock(ctx->mu);
    DeviceState& d = ctx->devs[0];
    PF_CUDA(cudaSetDevice(d.device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!d.d_flag) {
        PF_CUDA(cudaMalloc(&d.d_flag, sizeof(uint32_t)));
        PF_CUDA(cudaMalloc(&d.d_key, sizeof(unsigned long long)));
    }
    PF_CUDA(cudaMemsetAsync(d.d_flag, 0, sizeof(uint32_t), s));
    sb::FilterArgs a{};
    a.text = d_text;
    a.pattern = d_pattern;
    a.pitch = pitch;
    a.n = static_cast<long long>(n);
    a.m = static_cast<int>(m);
    a.e = e;
    a.err_flag = d.d_flag;
    PF_CUDA(sb::launch_validate(a, s));
    uint32_t flag = 0;
    PF_CUDA(cudaMemcpyAsync(&flag, d.d_flag, sizeof(flag), cudaMemcpyDeviceToHost, s));
    PF_CUDA(cudaStreamSynchronize(s));
    if (flag) {
        PF_CUDA(cudaMemsetAsync(d.d_key, 0xFF, sizeof(unsigned long long), s));  // key = ~0 on s
        PF_CUDA(sb::launch_locate(d_text, d_pattern, pitch, a.n, a.m, d.d_key, s));
        unsigned long long key = 0;
        PF_CUDA(cudaMemcpyAsync(&key, d.d_key, sizeof(key), cudaMemcpyDeviceToHost, s));
        PF_CUDA(cudaStreamSynchronize(s));
        decode_illegal(key, 0, d_text, d_pattern, pitch, false, err);
        return PF_ERR_ILLEGAL_CHARACTER;
    }
    if (e >= m)
        PF_CUDA(sb::launch_accept_all(a.n, a.m, d_accept_bitmap, d_estimates, d_bits, s));
    else
        PF_CUDA(sb::launch_magnet(d_text, d_pattern, pitch, a.n, a.m, static_cast<int>(e),
                                  d_accept_bitmap, d_estimates, d_bits, s));
    return PF_OK;
}

size_t pf_packed_words(uint32_t m) { return 3 * ((static_cast<size_t>(m) + 63) / 64); }

int pf_shouji_filter_packed_batch(pf_ctx* ctx, const uint64_t* text_planes,
                                  const uint64_t* pattern_planes, size_t n, uint32_t m, uint32_t e,
                                  uint32_t width, uint32_t* accept_bitmap, uint32_t* estimates,
                                  uint64_t* bits, pf_error* err) {
    if (err) std::memset(err, 0, sizeof(*err));
    if (!ctx) return PF_ERR_NULL_ARGUMENT;
    if (n == 0) return PF_OK;
    if (!text_planes || !pattern_planes || !accept_bitmap) return PF_ERR_NULL_ARGUMENT;
    if (m == 0) {
        set_err(err, PF_ERR_EMPTY_SEQUENCE, "empty sequence");
        return PF_ERR_EMPTY_SEQUENCE;
    }
    if (width < 3 || width > 8) {  // window_zero_table ctor (shouji.cpp:9-15), before e >= m
        set_err(err, PF_ERR_INVALID_PARAMETERS, "window width must be in [3, 8]");
        return PF_ERR_INVALID_PARAMETERS;
    }
    if (m >= (1u << 24)) {
        set_err(err, PF_ERR_INVALID_PARAMETERS, "m >= 2^24");
        return PF_ERR_INVALID_PARAMETERS;
    }
    std::lock_guard<std::mutex> lock(ctx->mu);
    if (small_applies(n, m))
        return run_small(ctx->devs[0], nullptr, nullptr, 0, text_planes, pattern_planes, n, m, e,
                         width, accept_bitmap, estimates, bits, err);
    const size_t nd = ctx->devs.size();
    const std::vector<size_t> bounds = shard_bounds(n, nd, ctx->shard_chunk);
    const size_t nshards = bounds.size() - 1;
    std::vector<ShardResult> res(nshards);
    auto work = [&](size_t t) {
        for (size_t k = t; k < nshards; k += nd) {
            run_packed_shard(ctx->devs[t], text_planes, pattern_planes, bounds[k], bounds[k + 1],
                             m, e, width, accept_bitmap, estimates, bits, &res[k]);
            if (res[k].status != PF_OK) break;
        }
    };
    if (nd == 1) {
        work(0);
    } else {
        std::vector<std::thread> pool;
        for (size_t t = 0; t < nd; ++t) pool.emplace_back(work, t);
        for (auto& th : pool) th.join();
    }
    for (size_t k = 0; k < nshards; ++k) {
        if (res[k].status != PF_OK) {
            if (err) *err = res[k].err;
            if (err) err->status = res[k].status;
            return res[k].status;
        }
    }
    return PF_OK;
}

int pf_shouji_filter_packed_device(pf_ctx* ctx, const uint64_t* d_text_planes,
                                   const uint64_t* d_pattern_planes, size_t n, uint32_t m,
                                   uint32_t e, uint32_t width, uint32_t* d_accept_bitmap,
                                   uint32_t* d_estimates, uint64_t* d_bits, void* stream,
                                   pf_error* err) {
    if (err) std::memset(err, 0, sizeof(*err));
    if (!ctx) return PF_ERR_NULL_ARGUMENT;
    if (n == 0) return PF_OK;
    if (!d_text_planes || !d_pattern_planes || !d_accept_bitmap) return PF_ERR_NULL_ARGUMENT;
    if (m == 0) {
        set_err(err, PF_ERR_EMPTY_SEQUENCE, "empty sequence");
        return PF_ERR_EMPTY_SEQUENCE;
    }
    if (width < 3 || width > 8 || m >= (1u << 24) ||
        (reinterpret_cast<uintptr_t>(d_text_planes) | reinterpret_cast<uintptr_t>(d_pattern_planes)) %
                8 != 0) {
        set_err(err, PF_ERR_INVALID_PARAMETERS,
                "window width must be in [3, 8]; plane arrays must be 8-byte aligned");
        return PF_ERR_INVALID_PARAMETERS;
    }
    std::lock_guard<std::mutex> lock(ctx->mu);
    DeviceState& d = ctx->devs[0];
    PF_CUDA(cudaSetDevice(d.device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (e >= m) {
        PF_CUDA(sb::launch_accept_all(static_cast<long long>(n), static_cast<int>(m),
                                      d_accept_bitmap, d_estimates, d_bits, s));
        return PF_OK;
    }
    const size_t ngroups = (n + 31) / 32;
    PF_CUDA(grow(d.d_scratch, d.scratch_words,
                 sb::planes_scratch_words(static_cast<long long>(n), static_cast<int>(m))));
    if (d_bits) PF_CUDA(grow(d.d_outplanes, d.outplanes_words, size_t(m) * ngroups));
    sb::FilterArgs a{};
    a.packed_text = d_text_planes;
    a.packed_pattern = d_pattern_planes;
    a.n = static_cast<long long>(n);
    a.m = static_cast<int>(m);
    a.e = e;
    a.width = width;
    a.accept = d_accept_bitmap;
    a.estimates = d_estimates;
    a.outplanes = d_bits ? d.d_outplanes : nullptr;
    a.planes = d.d_scratch;
    a.planes_words = d.scratch_words;
    PF_CUDA(scratch_acquire(d, s));
    PF_CUDA(sb::launch_filter(a, s));
    if (d_bits) PF_CUDA(sb::launch_bits_transpose(d.d_outplanes, a.n, a.m, d_bits, s));
    PF_CUDA(scratch_release(d, s));
    return PF_OK;
}

int pf_banded_edit_distance_batch(pf_ctx* ctx, const uint8_t* text, const uint8_t* pattern,
                                  size_t stride, size_t n, uint32_t m, uint32_t e, int32_t* out,
                                  pf_error* err) {
    if (!out) return PF_ERR_NULL_ARGUMENT;
    return run_batch(ctx, text, pattern, stride, n, m, e, 4, nullptr, nullptr, nullptr, out, err);
}

int pf_shouji_filter_device(pf_ctx* ctx, const uint8_t* d_text, const uint8_t* d_pattern,
                            size_t pitch, size_t n, uint32_t m, uint32_t e, uint32_t width,
                            uint32_t* d_accept_bitmap, uint32_t* d_estimates, uint64_t* d_bits,
                            void* stream, pf_error* err) {
    if (err) std::memset(err, 0, sizeof(*err));
    if (!ctx) return PF_ERR_NULL_ARGUMENT;
    if (n == 0) return PF_OK;
    if (!d_text || !d_pattern || !d_accept_bitmap) return PF_ERR_NULL_ARGUMENT;
    if (m == 0) {
        set_err(err, PF_ERR_EMPTY_SEQUENCE, "empty sequence");
        return PF_ERR_EMPTY_SEQUENCE;
    }
    if (pitch % 4 != 0 || pitch < m ||
        (reinterpret_cast<uintptr_t>(d_text) | reinterpret_cast<uintptr_t>(d_pattern)) % 16 != 0 ||
        m >= (1u << 24)) {
        set_err(err, PF_ERR_INVALID_PARAMETERS,
                "device records need 16-byte aligned bases and pitch % 4 == 0, pitch >= m");
        return PF_ERR_INVALID_PARAMETERS;
    }
    std::lock_guard<std::mutex> lock(ctx->mu);
    DeviceState& d = ctx->devs[0];
    PF_CUDA(cudaSetDevice(d.device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t ngroups = (n + 31) / 32;
    if (!d.d_flag) {
        PF_CUDA(cudaMalloc(&d.d_flag, sizeof(uint32_t)));
        PF_CUDA(cudaMalloc(&d.d_key, sizeof(unsigned long long)));
    }
    if (d_bits) PF_CUDA(grow(d.d_outplanes, d.outplanes_words, size_t(m) * ngroups));
    PF_CUDA(cudaMemsetAsync(d.d_flag, 0, sizeof(uint32_t), s));
    sb::FilterArgs a{};
    a.text = d_text;
    a.pattern = d_pattern;
    a.pitch = pitch;
    a.n = static_cast<long long>(n);
    a.m = static_cast<int>(m);
    a.e = e;
    a.width = width;
    a.accept = d_accept_bitmap;
    a.estimates = d_estimates;
    a.outplanes = d_bits ? d.d_outplanes : nullptr;
    a.err_flag = d.d_flag;
    a.planes = d.d_scratch;
    a.planes_words = d.scratch_words;
    const bool short_circuit = e >= m;
    const bool bad_width = width < 3 || width > 8;
    // The scratch (planes, and d_outplanes that bits_transpose reads) is held from
    // the filter launch until after the transpose.
    PF_CUDA(scratch_acquire(d, s));
    if (short_circuit || bad_width)
        PF_CUDA(sb::launch_validate(a, s));
    else
        PF_CUDA(launch_any_unordered(d, a, s));
    uint32_t flag = 0;
    PF_CUDA(cudaMemcpyAsync(&flag, d.d_flag, sizeof(flag), cudaMemcpyDeviceToHost, s));
    PF_CUDA(cudaStreamSynchronize(s));
    if (flag) {
        PF_CUDA(scratch_release(d, s));
        PF_CUDA(cudaMemsetAsync(d.d_key, 0xFF, sizeof(unsigned long long), s));  // key = ~0 on s
        PF_CUDA(sb::launch_locate(d_text, d_pattern, pitch, a.n, a.m, d.d_key, s));
        unsigned long long key = 0;
        PF_CUDA(cudaMemcpyAsync(&key, d.d_key, sizeof(key), cudaMemcpyDeviceToHost, s));
        PF_CUDA(cudaStreamSynchronize(s));
        decode_illegal(key, 0, d_text, d_pattern, pitch, false, err);
        return PF_ERR_ILLEGAL_CHARACTER;
    }
    if (bad_width) {
        PF_CUDA(scratch_release(d, s));
        set_err(err, PF_ERR_INVALID_PARAMETERS, "window width must be in [3, 8]");
        return PF_ERR_INVALID_PARAMETERS;
    }
    if (short_circuit)
        PF_CUDA(sb::launch_accept_all(a.n, a.m, d_accept_bitmap, d_estimates, d_bits, s));
    else if (d_bits)
        PF_CUDA(sb::launch_bits_transpose(d.d_outplanes, a.n, a.m, d_bits, s));
    PF_CUDA(scratch_release(d, s));
    return PF_OK;
}

int pf_shouji_filter_device_async(pf_ctx* ctx, const uint8_t* d_text, const uint8_t* d_pattern,
                                  size_t pitch, size_t n, uint32_t m, uint32_t e, uint32_t width,
                                  uint32_t* d_accept_bitmap, uint32_t* d_estimates,
                                  uint32_t* d_err_flag, void* stream) {
    pf_error* err = nullptr;
    if (!ctx || !d_err_flag) return PF_ERR_NULL_ARGUMENT;
    if (n == 0) return PF_OK;
    if (!d_text || !d_pattern || !d_accept_bitmap) return PF_ERR_NULL_ARGUMENT;
    if (m == 0) return PF_ERR_EMPTY_SEQUENCE;
    if (e >= m || width < 3 || width > 8 || pitch % 4 != 0 || pitch < m ||
        (reinterpret_cast<uintptr_t>(d_text) | reinterpret_cast<uintptr_t>(d_pattern)) % 16 != 0)
        return PF_ERR_INVALID_PARAMETERS;
    std::lock_guard<std::mutex> lock(ctx->mu);
    DeviceState& d = ctx->devs[0];
    PF_CUDA(cudaSetDevice(d.device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    sb::FilterArgs a{};
    a.text = d_text;
    a.pattern = d_pattern;
    a.pitch = pitch;
    a.n = static_cast<long long>(n);
    a.m = static_cast<int>(m);
    a.e = e;
    a.width = width;
    a.accept = d_accept_bitmap;
    a.estimates = d_estimates;
    a.outplanes = nullptr;
    a.err_flag = d_err_flag;
    a.planes = d.d_scratch;
    a.planes_words = d.scratch_words;
    PF_CUDA(launch_any(d, a, s));
    return PF_OK;
}

int pf_shouji_profile_stages(pf_ctx* ctx, const uint8_t* d_text, const uint8_t* d_pattern,
                             size_t pitch, size_t n, uint32_t m, uint32_t e, uint32_t width,
                             uint32_t* d_accept_bitmap, uint32_t* d_err_flag, int reps,
                             float* pack_ms, float* search_ms) {
    pf_error* err = nullptr;
    if (!ctx || !d_err_flag || !pack_ms || !search_ms || reps < 1) return PF_ERR_NULL_ARGUMENT;
    if (n == 0 || !d_text || !d_pattern || !d_accept_bitmap) return PF_ERR_NULL_ARGUMENT;
    if (m == 0 || e >= m || width < 3 || width > 8 || pitch % 4 != 0 || pitch < m)
        return PF_ERR_INVALID_PARAMETERS;
    std::lock_guard<std::mutex> lock(ctx->mu);
    DeviceState& d = ctx->devs[0];
    PF_CUDA(cudaSetDevice(d.device));
    // events owned by a guard so that every early return (PF_CUDA) destroys them
    struct Events {
        cudaEvent_t e[3] = {nullptr, nullptr, nullptr};
        ~Events() {
            for (auto& x : e)
                if (x) cudaEventDestroy(x);
        }
    } evs;
    cudaEvent_t* ev = evs.e;
    for (int i = 0; i < 3; ++i) PF_CUDA(cudaEventCreate(&ev[i]));
    sb::FilterArgs a{};
    a.text = d_text;
    a.pattern = d_pattern;
    a.pitch = pitch;
    a.n = static_cast<long long>(n);
    a.m = static_cast<int>(m);
    a.e = e;
    a.width = width;
    a.accept = d_accept_bitmap;
    a.err_flag = d_err_flag;
    a.stage_event = ev[1];
    double pk = 0.0, se = 0.0;
    for (int r = 0; r < reps; ++r) {
        PF_CUDA(cudaEventRecord(ev[0], d.stream));
        PF_CUDA(launch_any(d, a, d.stream));
        PF_CUDA(cudaEventRecord(ev[2], d.stream));
        PF_CUDA(cudaEventSynchronize(ev[2]));
        float t0 = 0.f, t1 = 0.f;
        PF_CUDA(cudaEventElapsedTime(&t0, ev[0], ev[1]));
        PF_CUDA(cudaEventElapsedTime(&t1, ev[1], ev[2]));
        pk += t0;
        se += t1;
    }
    *pack_ms = static_cast<float>(pk / reps);
    *search_ms = static_cast<float>(se / reps);
    return PF_OK;
}

int pf_int_peak(pf_ctx* ctx, int op, double* ops_per_second) {
    pf_error* err = nullptr;
    if (!ctx || !ops_per_second) return PF_ERR_NULL_ARGUMENT;
    std::lock_guard<std::mutex> lock(ctx->mu);
    DeviceState& d = ctx->devs[0];
    PF_CUDA(cudaSetDevice(d.device));
    PF_CUDA(sb::measure_int_peak(op, d.stream, ops_per_second));
    return PF_OK;
}

}  // extern "C"

namespace {

// Per-pair entry points (shouji_filter / magnet_filter signatures): the
// caller's packed_sequence objects would have been built (and validated)
// before the filter runs — pattern first, then text — then the filter checks
// lengths (shouji.cpp:44-45, magnet.cpp:79-80) and, for Shouji, the width
// (shouji.cpp:47, before the e >= m short-circuit). The pair then runs as a
// batch of one on the device.
int filter_one(pf_ctx* ctx, bool magnet, const char* pattern, size_t pattern_len,
               const char* text, size_t text_len, uint32_t e, uint32_t width, int* accept,
               uint32_t* estimate, uint64_t* bits, pf_error* err) {
    if (err) std::memset(err, 0, sizeof(*err));
    if (!ctx || !accept || !estimate) return PF_ERR_NULL_ARGUMENT;
    if (pattern_len == 0 || text_len == 0) {
        set_err(err, PF_ERR_EMPTY_SEQUENCE, "empty sequence");
        return PF_ERR_EMPTY_SEQUENCE;
    }
    if (!pattern || !text) return PF_ERR_NULL_ARGUMENT;
    for (int field = 0; field < 2; ++field) {
        const char* s = field == 0 ? pattern : text;
        const size_t len = field == 0 ? pattern_len : text_len;
        for (size_t i = 0; i < len; ++i) {
            const char c = s[i];
            if (c != 'A' && c != 'C' && c != 'G' && c != 'T' && c != 'N') {
                if (err) {
                    err->status = PF_ERR_ILLEGAL_CHARACTER;
                    err->pair = 0;
                    err->field = field == 0 ? 1u : 0u;  // 1 = pattern, 0 = text
                    err->position = i;
                    err->byte = static_cast<unsigned char>(c);
                    std::snprintf(err->message, sizeof(err->message),
                                  "illegal character at position %zu", i);
                }
                return PF_ERR_ILLEGAL_CHARACTER;
            }
        }
    }
    if (pattern_len != text_len) {
        set_err(err, PF_ERR_LENGTH_MISMATCH, "length mismatch");
        return PF_ERR_LENGTH_MISMATCH;
    }
    if (!magnet && (width < 3 || width > 8)) {
        set_err(err, PF_ERR_INVALID_PARAMETERS, "window width must be in [3, 8]");
        return PF_ERR_INVALID_PARAMETERS;
    }
    uint32_t acc = 0;
    const auto* t = reinterpret_cast<const uint8_t*>(text);
    const auto* p = reinterpret_cast<const uint8_t*>(pattern);
    const auto m = static_cast<uint32_t>(text_len);
    const int st = magnet ? pf_magnet_filter_batch(ctx, t, p, text_len, 1, m, e, &acc, estimate,
                                                   bits, err)
                          : pf_shouji_filter_batch(ctx, t, p, text_len, 1, m, e, width, &acc,
                                                   estimate, bits, err);
    if (st != PF_OK) return st;
    *accept = static_cast<int>(acc & 1u);
    return PF_OK;
}

}  // namespace

extern "C" {

int pf_shouji_filter_one(pf_ctx* ctx, const char* pattern, size_t pattern_len, const char* text,
                         size_t text_len, uint32_t e, uint32_t width, int* accept,
                         uint32_t* estimate, uint64_t* bits, pf_error* err) {
    return filter_one(ctx, false, pattern, pattern_len, text, text_len, e, width, accept, estimate,
                      bits, err);
}

int pf_magnet_filter_one(pf_ctx* ctx, const char* pattern, size_t pattern_len, const char* text,
                         size_t text_len, uint32_t e, int* accept, uint32_t* estimate,
                         uint64_t* bits, pf_error* err) {
    return filter_one(ctx, true, pattern, pattern_len, text, text_len, e, 4, accept, estimate,
                      bits, err);
}

void* pf_host_alloc(size_t bytes) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, std::max<size_t>(bytes, 1), cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}

void pf_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

int pf_generate_device(pf_ctx* ctx, int kind, uint64_t seed, uint32_t param, uint8_t* d_text,
                       uint8_t* d_pattern, size_t pitch, size_t n, uint32_t m, void* stream) {
    if (!ctx) return PF_ERR_NULL_ARGUMENT;
    pf_error* err = nullptr;
    std::lock_guard<std::mutex> lock(ctx->mu);
    DeviceState& d = ctx->devs[0];
    PF_CUDA(cudaSetDevice(d.device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const cudaError_t st = sb::launch_generate(kind, seed, param, d_text, d_pattern, pitch,
                                               static_cast<long long>(n), static_cast<int>(m), s);
    if (st == cudaErrorInvalidValue) return PF_ERR_INVALID_PARAMETERS;
    if (st != cudaSuccess) return PF_ERR_CUDA;
    return PF_OK;
}

}  // extern "C"
