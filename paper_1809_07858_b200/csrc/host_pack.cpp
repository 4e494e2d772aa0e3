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

}  // namespace sb
