// Seeded synthetic pair generator for BASELINE.json configs 1-4 (the paper's
// mrFAST candidate sets, are not available; these stand in
// with the configs' lengths, thresholds and edit distributions). One thread
// builds one pair. Draws come from a counter-based splitmix64 stream keyed by
// (kind, seed, param, pair), so the bytes are deterministic and independent
// of launch geometry. Edits are planted the way the reference generator does
// (generate_pairs, proj/src/dataset.cpp:71-126: substitution always changes
// the base, insertion at [0, size], deletion skipped at size 1, truncate or
// pad at the tail); the per-config rules are documented in DESIGN.md.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace sb {

namespace {

constexpr int kGenMaxM = 1024;
constexpr int kGenSlack = 64;

struct Rng {
    uint64_t s;
    __device__ uint64_t next() {
        uint64_t z = (s += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    __device__ double uniform() { return double(next() >> 11) * (1.0 / 9007199254740992.0); }
};

__device__ __forceinline__ char base_of(uint64_t r) { return "ACGT"[r & 3u]; }

__device__ __forceinline__ char other_base(char old, uint64_t r) {
    int idx = old == 'A' ? 0 : old == 'C' ? 1 : old == 'G' ? 2 : 3;
    return "ACGT"[(idx + 1 + int(r % 3)) % 4];
}

// Apply one edit of `type` (0 sub, 1 ins, 2 del) at a position drawn in
// [lo, hi) of the current string (clipped to its size).
__device__ void apply_edit(char* s, int& size, int type, int lo, int hi, Rng& rng) {
    switch (type) {
        case 0: {
            if (size == 0) return;
            const int h = hi < size ? hi : size;
            const int l = lo < h ? lo : 0;
            const int pos = l + int(rng.next() % uint64_t(h - l));
            if (s[pos] == 'N') return;
            s[pos] = other_base(s[pos], rng.next());
            break;
        }
        case 1: {
            if (size >= kGenMaxM + kGenSlack - 1) return;
            const int h = (hi < size ? hi : size) + 1;
            const int l = lo < h ? lo : 0;
            const int pos = l + int(rng.next() % uint64_t(h - l));
            const char b = base_of(rng.next());
            for (int i = size; i > pos; --i) s[i] = s[i - 1];
            s[pos] = b;
            ++size;
            break;
        }
        default: {
            if (size <= 1) return;
            const int h = hi < size ? hi : size;
            const int l = lo < h ? lo : 0;
            const int pos = l + int(rng.next() % uint64_t(h - l));
            for (int i = pos; i < size - 1; ++i) s[i] = s[i + 1];
            --size;
            break;
        }
    }
}

// Poisson(6) by inversion. exp(-6) is its correctly rounded double and every
// step is rounded on its own (no FMA contraction), so the CPU mirror
// (oracle/config_oracle.c, gen_poisson6) draws the same k bit for bit.
__device__ int poisson_inv6(Rng& rng) {
    const double u = rng.uniform();
    double p = 0x1.44e51f113d4d6p-9;  // exp(-6)
    double cdf = p;
    int k = 0;
    while (u > cdf && k < 200) {
        ++k;
        p = __dmul_rn(p, __ddiv_rn(6.0, double(k)));
        cdf = __dadd_rn(cdf, p);
    }
    return k;
}

__global__ void generate_pairs_kernel(int kind, uint64_t seed, uint32_t param, uint8_t* text,
                                      uint8_t* pattern, size_t pitch, long long n, int m) {
    const long long p = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= n) return;
    Rng rng{seed * 0x2545F4914F6CDD1Dull ^ (uint64_t(kind) << 56) ^ (uint64_t(param) << 40) ^
            (uint64_t(p) * 0xD1B54A32D192ED03ull)};
    rng.next();
    char t[kGenMaxM];
    char s[kGenMaxM + kGenSlack];

    // --- reference segment -------------------------------------------------
    if (kind == 4) {
        const uint64_t r = rng.next() % 10;
        if (r < 3) {  // tandem repeat of period 1..6
            const int period = 1 + int(rng.next() % 6);
            char unit[6];
            for (int i = 0; i < period; ++i) unit[i] = base_of(rng.next());
            for (int i = 0; i < m; ++i) t[i] = unit[i % period];
        } else {
            for (int i = 0; i < m; ++i) t[i] = base_of(rng.next());
            if (r == 3) {  // homopolymer runs of length 5..20
                const int runs = 1 + int(rng.next() % 4);
                for (int k = 0; k < runs; ++k) {
                    const int len = 5 + int(rng.next() % 16);
                    const int start = int(rng.next() % uint64_t(m));
                    const char b = base_of(rng.next());
                    for (int i = start; i < start + len && i < m; ++i) t[i] = b;
                }
            }
        }
    } else {
        for (int i = 0; i < m; ++i) t[i] = base_of(rng.next());
    }

    // --- read ----------------------------------------------------------------
    bool unrelated = false;
    int k = 0;
    int burst_lo = 0;
    const int e = int(param);
    switch (kind) {
        case 1:  // 50% planted k ~ U{0..2E}, 50% independent
            unrelated = (rng.next() & 1u) != 0;
            k = int(rng.next() % uint64_t(2 * e + 1));
            break;
        case 2:  // 30% unrelated, else k ~ Poisson(6)
            unrelated = rng.next() % 10 < 3;
            k = poisson_inv6(rng);
            break;
        case 3:  // k ~ U{0..2E}, half of the edits inside one 20-base burst
            k = int(rng.next() % uint64_t(2 * e + 1));
            burst_lo = m > 20 ? int(rng.next() % uint64_t(m - 20 + 1)) : 0;
            break;
        default:  // 4: k ~ U{0..40}
            k = int(rng.next() % 41);
            break;
    }
    int size = m;
    if (unrelated) {
        for (int i = 0; i < m; ++i) s[i] = base_of(rng.next());
    } else {
        for (int i = 0; i < m; ++i) s[i] = t[i];
        for (int q = 0; q < k; ++q) {
            int type;
            if (kind == 2) {
                const uint64_t r = rng.next() % 10;  // 60/20/20 sub/ins/del
                type = r < 6 ? 0 : (r < 8 ? 1 : 2);
            } else {
                type = int(rng.next() % 3);
            }
            int lo = 0, hi = 1 << 30;
            if (kind == 3 && (rng.next() & 1u)) {
                lo = burst_lo;
                hi = burst_lo + 20;
            }
            apply_edit(s, size, type, lo, hi, rng);
        }
        if (size > m) size = m;
        while (size < m) s[size++] = base_of(rng.next());
    }
    if (kind == 4) {  // 'N' at 0.1% of positions in both sequences
        for (int i = 0; i < m; ++i) {
            if (rng.next() % 1000 == 0) t[i] = 'N';
            if (rng.next() % 1000 == 0) s[i] = 'N';
        }
    }
    uint8_t* trow = text + p * pitch;
    uint8_t* prow = pattern + p * pitch;
    for (int i = 0; i < m; ++i) {
        trow[i] = static_cast<uint8_t>(t[i]);
        prow[i] = static_cast<uint8_t>(s[i]);
    }
}

}  // namespace

cudaError_t launch_generate(int kind, uint64_t seed, uint32_t param, uint8_t* text,
                            uint8_t* pattern, size_t pitch, long long n, int m, cudaStream_t s) {
    if (kind < 1 || kind > 4 || m < 1 || m > kGenMaxM) return cudaErrorInvalidValue;
    if (n <= 0) return cudaSuccess;
    const unsigned grid = static_cast<unsigned>((n + 127) / 128);
    generate_pairs_kernel<<<grid, 128, 0, s>>>(kind, seed, param, text, pattern, pitch, n, m);
    count_launch();
    return cudaGetLastError();
}

}  // namespace sb
