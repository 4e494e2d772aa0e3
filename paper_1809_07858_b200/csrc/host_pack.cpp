// Host-side packing stage for host-resident batches (north star (1): "batched
// packing/upload stage with pinned, double-buffered host->HBM streaming").
//
// ASCII records (8 bits per base) become nibble records (pack.cuh: 4 bits per
// base, the low nibble of the ASCII byte) on the host's cores, so PCIe carries
// about half the bytes; the device pack kernel reads nibbles instead of bytes.
// Validation has the contract of packed_sequence::from_string
// (proj/src/packed_sequence.cpp:19-29): the first illegal byte in pair order,
// text before pattern, lowest position, is reported exactly.
//
// AVX-512 path, per 128 columns of a record: two (masked) 64-byte loads; a
// byte is legal iff a 64-entry VBMI byte permute maps it to itself (the
// mismatches are OR-accumulated and only tested once per task); per 8-column
// block the upper 4 columns' nibbles are shifted onto the lower 4 columns'
// (one 64-bit shift + one bit-select ternlog), and one two-source dword permute
// keeps the packed half of every qword. The stage streams: ~3 SIMD ops per 64
// input bytes, so it runs at the cores' memory bandwidth.
#include <immintrin.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "host_pack.h"
#include "pack.cuh"

namespace sb {

namespace {

bool valid_base(uint8_t c) { return c == 'A' || c == 'C' || c == 'G' || c == 'T' || c == 'N'; }

// First illegal byte of pairs [lo, hi) (pair order, text first, lowest position).
void scan_bad(const uint8_t* text, const uint8_t* pattern, size_t stride, int m, long long lo,
              long long hi, HostBad* bad) {
    for (long long r = lo; r < hi; ++r)
        for (int f = 0; f < 2; ++f) {
            const uint8_t* row = (f == 0 ? text : pattern) + r * stride;
            for (int c = 0; c < m; ++c)
                if (!valid_base(row[c])) {
                    bad->offer(static_cast<uint64_t>(r), f, c, row[c]);
                    return;
                }
        }
}

// ---- portable path ------------------------------------------------------------
bool pack_row_scalar(const uint8_t* src, int m, uint8_t* dst) {
    const int words = (m + 7) / 8;
    bool ok = true;
    for (int w = 0; w < words; ++w)
        for (int q = 0; q < 4; ++q) {
            const int c0 = 8 * w + q, c1 = c0 + 4;
            const uint8_t a = c0 < m ? src[c0] : 0, b = c1 < m ? src[c1] : 0;
            if (c0 < m) ok &= valid_base(a);
            if (c1 < m) ok &= valid_base(b);
            dst[4 * w + q] = static_cast<uint8_t>((a & 0x0F) | ((b & 0x0F) << 4));
        }
    return ok;
}

// Software prefetch of the records kPrefetchRows rows ahead, both sequences:
// the hardware prefetchers stop at 4 KiB page boundaries, and each core
// streams two record arrays. Measured on the B200 boxes' 16-core hosts
// (tools/exp_host_threads.py, bench.py e2e): the host batch path (pack + DMA)
// 510 -> 635-653 M pairs/s at 64 rows (32-96 all gain, 64 the most consistent),
// the pack alone +30-50% at 8 threads.
constexpr long long kPrefetchRows = 64;

inline void prefetch_rows(const uint8_t* text, const uint8_t* pattern, size_t stride, int m,
                          long long r) {
    const size_t off = static_cast<size_t>(r) * stride;
    for (size_t b = 0; b < static_cast<size_t>(m); b += 64) {
        _mm_prefetch(reinterpret_cast<const char*>(text + off + b), _MM_HINT_T0);
        _mm_prefetch(reinterpret_cast<const char*>(pattern + off + b), _MM_HINT_T0);
    }
}

// ---- AVX-512 path ---------------------------------------------------------------
#define SB_AVX512 __attribute__((target("avx512f,avx512bw,avx512vl,avx512vbmi,bmi,bmi2")))

// Low dword of every qword <- the 8 columns of that qword in nibble form.
SB_AVX512 inline __m512i nib8(__m512i v) {
    const __m512i t = _mm512_srli_epi64(v, 28);  // columns 4-7 over 0-3, shifted up 4 bits
    return _mm512_ternarylogic_epi32(_mm512_set1_epi8(0x0F), v, t, 0xCA);  // 0x0F ? v : t
}

SB_AVX512 void pack_rows_avx512(const uint8_t* text, const uint8_t* pattern, size_t stride, int m,
                                long long lo, long long hi, uint8_t* out_text,
                                uint8_t* out_pattern, HostBad* bad) {
    const size_t np = nibble_pitch(m);
    // byte x is legal iff lut[x & 63] == x; every other entry differs from all
    // bytes that index it (entry i holds i ^ 1 in its low 6 bits)
    alignas(64) uint8_t lb[64];
    for (int i = 0; i < 64; ++i) lb[i] = static_cast<uint8_t>(i ^ 1);
    for (uint8_t c : {'A', 'C', 'G', 'N', 'T'}) lb[c & 63] = c;
    const __m512i lut = _mm512_load_si512(lb);
    const __m512i even = _mm512_setr_epi32(0, 2, 4, 6, 8, 10, 12, 14, 16, 18, 20, 22, 24, 26, 28, 30);
    __m512i acc = _mm512_setzero_si512();
    auto mask_of = [](int w) -> __mmask64 {
        return w >= 64 ? ~0ull : (w <= 0 ? 0ull : ((1ull << w) - 1));
    };
    for (long long r = lo; r < hi; ++r) {
        if (r + kPrefetchRows < hi) prefetch_rows(text, pattern, stride, m, r + kPrefetchRows);
        for (int f = 0; f < 2; ++f) {
            const uint8_t* s = (f == 0 ? text : pattern) + r * stride;
            uint8_t* d = (f == 0 ? out_text : out_pattern) + r * np;
            for (int c0 = 0; c0 < m; c0 += 128) {
                const int w = m - c0;
                const __mmask64 k0 = mask_of(w), k1 = mask_of(w - 64);
                const __m512i a = _mm512_maskz_loadu_epi8(k0, s + c0);
                const __m512i b = _mm512_maskz_loadu_epi8(k1, s + c0 + 64);
                // masked-off lanes: permute -> 0 and the loaded byte is 0
                const __m512i la = _mm512_maskz_permutexvar_epi8(k0, a, lut);
                const __m512i lbv = _mm512_maskz_permutexvar_epi8(k1, b, lut);
                acc = _mm512_ternarylogic_epi32(acc, la, a, 0xF6);   // acc | (la ^ a)
                acc = _mm512_ternarylogic_epi32(acc, lbv, b, 0xF6);  // acc | (lb ^ b)
                const __m512i o = _mm512_permutex2var_epi32(nib8(a), even, nib8(b));
                const int ob = static_cast<int>(np) - c0 / 2;
                _mm512_mask_storeu_epi8(d + c0 / 2, mask_of(ob), o);
            }
        }
    }
    if (_mm512_test_epi8_mask(acc, acc)) scan_bad(text, pattern, stride, m, lo, hi, bad);
}

// ---- dibit records (pack.cuh) ------------------------------------------------------
// Per 64 columns: codes = (byte >> 1) & 3; within each 16-byte lane the four
// dwords (columns q, q+4, q+8, q+12 at the same byte) are merged with
// lane-local byte shifts and 2/4/6-bit dword shifts; the low dword of every
// lane is the packed word (vpcompressd keeps those 4). N columns are recorded
// in the returned 64-bit mask (bit 3 of the byte).
SB_AVX512 inline __m128i dib64(__m512i v) {
    const __m512i c = _mm512_and_si512(_mm512_srli_epi16(v, 1), _mm512_set1_epi8(0x03));
    const __m512i c1 = _mm512_slli_epi32(_mm512_bsrli_epi128(c, 4), 2);
    const __m512i c2 = _mm512_slli_epi32(_mm512_bsrli_epi128(c, 8), 4);
    const __m512i c3 = _mm512_slli_epi32(_mm512_bsrli_epi128(c, 12), 6);
    const __m512i r = _mm512_ternarylogic_epi32(_mm512_or_si512(c, c1), c2, c3, 0xFE);  // a|b|c
    return _mm512_castsi512_si128(_mm512_maskz_compress_epi32(0x1111, r));
}

// Rows [lo, hi) -> dibit rows (and N-plane rows when nplanes != nullptr).
// Returns true when any of these rows holds an N.
SB_AVX512 bool pack_dibit_rows_avx512(const uint8_t* text, const uint8_t* pattern, size_t stride,
                                      int m, long long lo, long long hi, uint8_t* out_text,
                                      uint8_t* out_pattern, uint8_t* n_text, uint8_t* n_pattern,
                                      HostBad* bad) {
    const size_t dp = dibit_pitch(m), np = nplane_pitch(m);
    alignas(64) uint8_t lb[64];
    for (int i = 0; i < 64; ++i) lb[i] = static_cast<uint8_t>(i ^ 1);
    for (uint8_t c : {'A', 'C', 'G', 'N', 'T'}) lb[c & 63] = c;
    const __m512i lut = _mm512_load_si512(lb);
    const __m512i bitn = _mm512_set1_epi8(0x08);
    __m512i acc = _mm512_setzero_si512();
    uint64_t anyn = 0;
    auto mask_of = [](int w) -> __mmask64 {
        return w >= 64 ? ~0ull : (w <= 0 ? 0ull : ((1ull << w) - 1));
    };
    for (long long r = lo; r < hi; ++r) {
        if (r + kPrefetchRows < hi) prefetch_rows(text, pattern, stride, m, r + kPrefetchRows);
        for (int f = 0; f < 2; ++f) {
            const uint8_t* s = (f == 0 ? text : pattern) + r * stride;
            uint8_t* d = (f == 0 ? out_text : out_pattern) + r * dp;
            uint8_t* nd = n_text ? (f == 0 ? n_text : n_pattern) + r * np : nullptr;
            for (int c0 = 0; c0 < m; c0 += 64) {
                const __mmask64 k = mask_of(m - c0);
                const __m512i v = _mm512_maskz_loadu_epi8(k, s + c0);
                acc = _mm512_ternarylogic_epi32(acc, _mm512_maskz_permutexvar_epi8(k, v, lut), v,
                                                0xF6);  // acc | (lut(v) ^ v)
                const uint64_t nm = _mm512_test_epi8_mask(v, bitn);
                anyn |= nm;
                const int ob = static_cast<int>(dp) - c0 / 4;  // bytes left in the row
                _mm_mask_storeu_epi8(d + c0 / 4, static_cast<__mmask16>(ob >= 16 ? 0xFFFF : ((1u << ob) - 1)),
                                     dib64(v));
                if (nd) {
                    const int nb = static_cast<int>(np) - c0 / 8;
                    const __m128i nv = _mm_cvtsi64_si128(static_cast<long long>(nm));
                    _mm_mask_storeu_epi8(nd + c0 / 8, static_cast<__mmask16>(nb >= 8 ? 0xFF : ((1u << nb) - 1)), nv);
                }
            }
        }
    }
    if (_mm512_test_epi8_mask(acc, acc)) scan_bad(text, pattern, stride, m, lo, hi, bad);
    return anyn != 0;
}

// Rows [lo, hi): the byte check of pack_dibit_rows_avx512 without the packing.
SB_AVX512 bool validate_rows_avx512(const uint8_t* text, const uint8_t* pattern, size_t stride,
                                    int m, long long lo, long long hi) {
    alignas(64) uint8_t lb[64];
    for (int i = 0; i < 64; ++i) lb[i] = static_cast<uint8_t>(i ^ 1);
    for (uint8_t c : {'A', 'C', 'G', 'N', 'T'}) lb[c & 63] = c;
    const __m512i lut = _mm512_load_si512(lb);
    __m512i acc = _mm512_setzero_si512();
    for (long long r = lo; r < hi; ++r) {
        if (r + kPrefetchRows < hi) prefetch_rows(text, pattern, stride, m, r + kPrefetchRows);
        for (int f = 0; f < 2; ++f) {
            const uint8_t* s = (f == 0 ? text : pattern) + r * stride;
            for (int c0 = 0; c0 < m; c0 += 64) {
                const int w = m - c0;
                const __mmask64 k = w >= 64 ? ~0ull : ((1ull << w) - 1);
                const __m512i v = _mm512_maskz_loadu_epi8(k, s + c0);
                acc = _mm512_ternarylogic_epi32(acc, _mm512_maskz_permutexvar_epi8(k, v, lut), v,
                                                0xF6);  // acc | (lut(v) ^ v)
            }
        }
    }
    return !_mm512_test_epi8_mask(acc, acc);
}

bool pack_dibit_rows_scalar(const uint8_t* text, const uint8_t* pattern, size_t stride, int m,
                            long long lo, long long hi, uint8_t* out_text, uint8_t* out_pattern,
                            uint8_t* n_text, uint8_t* n_pattern, HostBad* bad) {
    const size_t dp = dibit_pitch(m), np = nplane_pitch(m);
    bool ok = true, anyn = false;
    for (long long r = lo; r < hi; ++r)
        for (int f = 0; f < 2; ++f) {
            const uint8_t* s = (f == 0 ? text : pattern) + r * stride;
            uint8_t* d = (f == 0 ? out_text : out_pattern) + r * dp;
            std::memset(d, 0, dp);
            uint8_t* nd = n_text ? (f == 0 ? n_text : n_pattern) + r * np : nullptr;
            if (nd) std::memset(nd, 0, np);
            for (int c = 0; c < m; ++c) {
                const uint8_t x = s[c];
                ok &= valid_base(x);
                const int w = c / 16, rem = c % 16, q = rem % 4, t = rem / 4;
                d[4 * w + q] |= static_cast<uint8_t>(((x >> 1) & 3u) << (2 * t));
                if ((x >> 3) & 1u) {
                    anyn = true;
                    if (nd) nd[c / 8] |= static_cast<uint8_t>(1u << (c % 8));
                }
            }
        }
    if (!ok) scan_bad(text, pattern, stride, m, lo, hi, bad);
    return anyn;
}

bool has_avx512() {
    static const bool v = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw") &&
                          __builtin_cpu_supports("avx512vl") &&
                          __builtin_cpu_supports("avx512vbmi") && __builtin_cpu_supports("bmi") &&
                          __builtin_cpu_supports("bmi2");
    return v;
}

}  // namespace

bool host_pack_uses_simd() { return has_avx512(); }

void host_pack_nibbles(const uint8_t* text, const uint8_t* pattern, size_t stride, int m,
                       long long lo, long long hi, uint8_t* out_text, uint8_t* out_pattern,
                       HostBad* bad, bool allow_simd) {
    if (allow_simd && has_avx512()) {
        pack_rows_avx512(text, pattern, stride, m, lo, hi, out_text, out_pattern, bad);
        return;
    }
    const size_t np = nibble_pitch(m);
    bool ok = true;
    for (long long r = lo; r < hi; ++r) {
        ok &= pack_row_scalar(text + r * stride, m, out_text + r * np);
        ok &= pack_row_scalar(pattern + r * stride, m, out_pattern + r * np);
    }
    if (!ok) scan_bad(text, pattern, stride, m, lo, hi, bad);
}

// ---- a small persistent worker pool -------------------------------------------
namespace {

class Pool {
public:
    explicit Pool(unsigned n) {
        for (unsigned i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> l(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }
    unsigned size() const { return static_cast<unsigned>(workers_.size()); }
    // Run fn(0..tasks-1) on the workers and the caller; returns when all are done.
    void run(size_t tasks, const std::function<void(size_t)>& fn) {
        std::lock_guard<std::mutex> serial(submit_mu_);
        {
            std::lock_guard<std::mutex> l(mu_);
            fn_ = &fn;
            tasks_ = tasks;
            next_ = 0;
            done_ = 0;
            ++gen_;
        }
        cv_.notify_all();
        work();
        std::unique_lock<std::mutex> l(mu_);
        done_cv_.wait(l, [&] { return done_ == tasks_; });
        fn_ = nullptr;
    }

private:
    void work() {
        for (;;) {
            size_t i;
            const std::function<void(size_t)>* fn;
            {
                std::lock_guard<std::mutex> l(mu_);
                if (!fn_ || next_ >= tasks_) return;
                i = next_++;
                fn = fn_;
            }
            (*fn)(i);
            std::lock_guard<std::mutex> l(mu_);
            if (++done_ == tasks_) done_cv_.notify_all();
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> l(mu_);
                cv_.wait(l, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
            }
            work();
        }
    }
    std::vector<std::thread> workers_;
    std::mutex mu_, submit_mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(size_t)>* fn_ = nullptr;
    size_t tasks_ = 0, next_ = 0, done_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

// Threads = hardware threads, or PF_HOST_THREADS (e.g. cores / ranks when
// several processes share the host).
Pool& pool() {
    static Pool p([] {
        const char* e = std::getenv("PF_HOST_THREADS");
        const long v = e ? std::atol(e) : 0;
        const unsigned n = v > 0 ? static_cast<unsigned>(v) : std::thread::hardware_concurrency();
        return std::max(1u, n) - 1;
    }());
    return p;
}

}  // namespace

unsigned host_pack_threads() { return pool().size() + 1; }

void host_pack_nibbles_parallel(const uint8_t* text, const uint8_t* pattern, size_t stride,
                                long long n, int m, uint8_t* out_text, uint8_t* out_pattern,
                                HostBad* bad, unsigned threads, bool allow_simd) {
    if (n <= 0) return;
    const unsigned nt = std::min(threads ? threads : host_pack_threads(), host_pack_threads());
    // ~4 tasks per thread (load balance), at least 1024 pairs each
    const size_t tasks = static_cast<size_t>(std::max<long long>(
        1, std::min<long long>((n + 1023) / 1024, 4ll * nt)));
    std::vector<HostBad> bads(tasks);
    auto body = [&](size_t t) {
        const long long lo = n * static_cast<long long>(t) / static_cast<long long>(tasks);
        const long long hi = n * static_cast<long long>(t + 1) / static_cast<long long>(tasks);
        host_pack_nibbles(text, pattern, stride, m, lo, hi, out_text, out_pattern, &bads[t],
                          allow_simd);
    };
    if (tasks == 1 || nt == 1) {
        for (size_t t = 0; t < tasks; ++t) body(t);
    } else {
        pool().run(tasks, body);
    }
    for (const auto& b : bads)
        if (b.any) bad->offer(b.pair, b.field, b.pos, b.byte);
}

void host_validate_parallel(const uint8_t* text, const uint8_t* pattern, size_t stride,
                            long long n, int m, HostBad* bad) {
    if (n <= 0) return;
    const bool simd = has_avx512();
    const unsigned nt = host_pack_threads();
    const size_t tasks = static_cast<size_t>(std::max<long long>(
        1, std::min<long long>((n + 1023) / 1024, 4ll * nt)));
    std::vector<HostBad> bads(tasks);
    auto body = [&](size_t t) {
        const long long lo = n * static_cast<long long>(t) / static_cast<long long>(tasks);
        const long long hi = n * static_cast<long long>(t + 1) / static_cast<long long>(tasks);
        if (!simd || !validate_rows_avx512(text, pattern, stride, m, lo, hi))
            scan_bad(text, pattern, stride, m, lo, hi, &bads[t]);
    };
    if (tasks == 1)
        body(0);
    else
        pool().run(tasks, body);
    for (const auto& b : bads)
        if (b.any) bad->offer(b.pair, b.field, b.pos, b.byte);
}

void host_copy_parallel(void* dst, const void* src, size_t bytes) {
    const size_t tasks = std::max<size_t>(
        1, std::min<size_t>((bytes + (1u << 20) - 1) >> 20, 4ull * host_pack_threads()));
    auto body = [&](size_t t) {
        const size_t lo = bytes * t / tasks / 64 * 64;
        const size_t hi = t + 1 == tasks ? bytes : bytes * (t + 1) / tasks / 64 * 64;
        if (hi > lo)
            std::memcpy(static_cast<uint8_t*>(dst) + lo, static_cast<const uint8_t*>(src) + lo,
                        hi - lo);
    };
    if (tasks == 1)
        body(0);
    else
        pool().run(tasks, body);
}

namespace {
SB_AVX512 uint64_t stream_read_avx512(const uint8_t* p, size_t bytes) {
    __m512i acc = _mm512_setzero_si512();
    size_t i = 0;
    for (; i + 256 <= bytes; i += 256) {
        _mm_prefetch(reinterpret_cast<const char*>(p + i + 64 * 64), _MM_HINT_T0);
        _mm_prefetch(reinterpret_cast<const char*>(p + i + 64 * 64 + 128), _MM_HINT_T0);
        acc = _mm512_xor_si512(acc, _mm512_loadu_si512(p + i));
        acc = _mm512_xor_si512(acc, _mm512_loadu_si512(p + i + 64));
        acc = _mm512_xor_si512(acc, _mm512_loadu_si512(p + i + 128));
        acc = _mm512_xor_si512(acc, _mm512_loadu_si512(p + i + 192));
    }
    uint64_t x = static_cast<uint64_t>(_mm512_reduce_add_epi64(acc));
    for (; i < bytes; ++i) x += p[i];
    return x;
}
}  // namespace

double host_read_gbs(const uint8_t* buf, size_t bytes, int passes) {
    // The host pack's own access pattern (AVX-512 loads, software prefetch 64 lines
    // ahead) over a caller buffer, on the same worker pool: what the host cores can
    // stream out of this memory, i.e. the ceiling of any path that reads it once.
    if (!buf || bytes < (1u << 20) || passes < 1) return 0.0;
    const bool simd = has_avx512();
    const size_t tasks = 4ull * host_pack_threads();
    std::vector<uint64_t> sink(tasks, 0);
    auto body = [&](size_t t) {
        const size_t lo = bytes * t / tasks / 64 * 64;
        const size_t hi = t + 1 == tasks ? bytes : bytes * (t + 1) / tasks / 64 * 64;
        if (simd) {
            sink[t] += stream_read_avx512(buf + lo, hi - lo);
        } else {
            uint64_t x = 0;
            for (size_t i = lo; i + 8 <= hi; i += 8) {
                uint64_t v;
                std::memcpy(&v, buf + i, 8);
                x ^= v;
            }
            sink[t] += x;
        }
    };
    pool().run(tasks, body);  // warm (page tables, worker wake-up)
    const auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < passes; ++r) pool().run(tasks, body);
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    volatile uint64_t keep = 0;
    for (auto v : sink) keep = keep + v;
    (void)keep;
    return s > 0 ? double(bytes) * passes / s / 1e9 : 0.0;
}

void host_pack_dibits_parallel(const uint8_t* text, const uint8_t* pattern, size_t stride,
                               long long n, int m, uint8_t* out_text, uint8_t* out_pattern,
                               uint8_t* n_text, uint8_t* n_pattern, HostBad* bad, bool* has_n,
                               bool allow_simd) {
    *has_n = false;
    if (n <= 0) return;
    const bool simd = allow_simd && has_avx512();
    const unsigned nt = host_pack_threads();
    const size_t tasks = static_cast<size_t>(std::max<long long>(
        1, std::min<long long>((n + 1023) / 1024, 4ll * nt)));
    std::vector<HostBad> bads(tasks);
    std::vector<char> nflags(tasks, 0);
    auto run = [&](uint8_t* nt_out, uint8_t* np_out) {
        auto body = [&](size_t t) {
            const long long lo = n * static_cast<long long>(t) / static_cast<long long>(tasks);
            const long long hi = n * static_cast<long long>(t + 1) / static_cast<long long>(tasks);
            const bool any = simd ? pack_dibit_rows_avx512(text, pattern, stride, m, lo, hi, out_text,
                                                           out_pattern, nt_out, np_out, &bads[t])
                                  : pack_dibit_rows_scalar(text, pattern, stride, m, lo, hi, out_text,
                                                           out_pattern, nt_out, np_out, &bads[t]);
            nflags[t] = any ? 1 : 0;
        };
        if (tasks == 1)
            body(0);
        else
            pool().run(tasks, body);
    };
    // first pass: dibits, validation, N detection; the N planes are written
    // (second pass) only when some row of the batch holds an N
    run(nullptr, nullptr);
    for (const auto& b : bads)
        if (b.any) bad->offer(b.pair, b.field, b.pos, b.byte);
    if (bad->any) return;
    for (char f : nflags) *has_n = *has_n || f;
    if (*has_n && n_text && n_pattern) run(n_text, n_pattern);
}

}  // namespace sb
