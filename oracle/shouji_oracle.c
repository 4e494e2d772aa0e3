/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the Shouji hot path.
 *
 * A plain-C restatement of the reference algorithm, written for clarity, not
 * speed: one byte per map cell, one loop per rule. It is the checker for the
 * CUDA path and is never linked into the product (libshouji_b200.so has no
 * CPU path). Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load it.
 *
 * Parity of this restatement is pinned two ways (tests/test_oracle.py):
 *   - against the reference's own golden vectors (proj/tests/test_shouji.cpp,
 *     test_neighborhood.cpp, test_packed_sequence.cpp), and
 *   - against the unmodified reference library compiled from its sources
 *     (oracle/_ref/libprefilter_ref.so, see oracle/Makefile), on seeded
 *     random inputs and on the committed fixtures in tests/golden/.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference).
 */
#include <pthread.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Status codes: identical to pf_status in include/shouji_b200.h. */
enum {
    SO_OK = 0,
    SO_EMPTY_SEQUENCE = 1,
    SO_ILLEGAL_CHARACTER = 2,
    SO_LENGTH_MISMATCH = 3,
    SO_THRESHOLD_TOO_LARGE = 4,
    SO_INVALID_PARAMETERS = 7,
};

typedef struct {
    int code;
    uint64_t pair;
    int field; /* 0 = text, 1 = pattern */
    uint64_t position;
    int byte;
} so_error;

/* packed_sequence::from_string — proj/src/packed_sequence.cpp:7-34.
 * Empty input -> empty_sequence_error (:8); the first byte outside
 * {A,C,G,T,N} -> illegal_character_error(pos, byte) (:27-28). Lower case is
 * rejected (proj/tests/test_packed_sequence.cpp:46-48). */
int so_validate(const char* s, size_t m, uint64_t* pos, int* byte) {
    if (m == 0) return SO_EMPTY_SEQUENCE;
    for (size_t i = 0; i < m; ++i) {
        switch (s[i]) {
            case 'A': case 'C': case 'G': case 'T': case 'N': break;
            default:
                *pos = i;
                *byte = (unsigned char)s[i];
                return SO_ILLEGAL_CHARACTER;
        }
    }
    return SO_OK;
}

/* bases_match — proj/include/prefilter/packed_sequence.hpp:58-61: an 'N' on
 * either side never matches, itself included. */
static int mismatch(char p, char t) { return p == 'N' || t == 'N' || p != t; }

/* neighborhood_map ctor — proj/src/neighborhood.cpp:41-79. Diagonal d holds
 * bit j = 1 iff pattern index j+d leaves [0,m) (:71-76) or the bases at
 * (j+d, j) mismatch (:67-69). out is (2e+1) x m bytes, row d+e. */
void so_neighborhood(const char* pattern, const char* text, size_t m, uint32_t e, uint8_t* out) {
    for (long d = -(long)e; d <= (long)e; ++d) {
        uint8_t* row = out + (size_t)(d + (long)e) * m;
        for (size_t j = 0; j < m; ++j) {
            const long i = (long)j + d;
            row[j] = (i < 0 || i >= (long)m) ? 1 : (uint8_t)mismatch(pattern[i], text[j]);
        }
    }
}

/* bitvector::extract(pos, w, pad=1) — proj/include/prefilter/bitvector.hpp:77-93:
 * w bits from pos, LSB = pos; positions >= size read as 1. */
static uint32_t extract_pad1(const uint8_t* bits, size_t m, size_t pos, unsigned w) {
    uint32_t v = 0;
    for (unsigned k = 0; k < w; ++k) {
        const size_t i = pos + k;
        const uint32_t b = i < m ? bits[i] : 1u;
        v |= b << k;
    }
    return v;
}

static unsigned zeros_of(uint32_t slice, unsigned w) {
    return w - (unsigned)__builtin_popcount(slice);
}

/* shouji_filter — proj/src/shouji.cpp:41-58, with select_window (:17-31) and
 * commit_window (:33-39) inlined. map is scratch of (2e+1) x m bytes; bits_out
 * receives the m-bit tally vector (one byte per bit). Preconditions handled by
 * the caller in reference order: lengths equal, 3 <= w <= 8 (:47, ctor :9-15),
 * e >= m short-circuit (:48-49). */
/* Deliberately wrong variants for mutation tests:
 * 1 reverse scan, 2 no leading-zero tie-break, 3 non-strict commit,
 * 4 pattern/text swapped. 0 = the reference rules. */
static int g_variant = 0;

static void shouji_core(const char* pattern, const char* text, size_t m, uint32_t e, unsigned w,
                        uint8_t* map, uint8_t* bits_out, uint32_t* estimate, int* accept) {
    if (g_variant == 4) {
        const char* tmp = pattern;
        pattern = text;
        text = tmp;
    }
    so_neighborhood(pattern, text, m, e, map);
    uint8_t* bv = bits_out;
    memset(bv, 1, m); /* bitvector bv(m, true) — :52 */
    for (size_t j = 0; j < m; ++j) {
        /* select_window: scan d = -e..+e, keep the first max-zeros slice; on a
         * zero-count tie replace only when the incumbent's leading bit is 1 and
         * the candidate's is 0 (:21-29). */
        const int rev = g_variant == 1;
        long best_d = rev ? (long)e : -(long)e;
        uint32_t best_s = extract_pad1(map + (size_t)(best_d + (long)e) * m, m, j, w);
        unsigned best_z = zeros_of(best_s, w);
        for (long k = -(long)e + 1; k <= (long)e; ++k) {
            const long d = rev ? -k : k;
            const uint32_t s = extract_pad1(map + (size_t)(d + (long)e) * m, m, j, w);
            const unsigned z = zeros_of(s, w);
            const int tie = g_variant != 2 && z == best_z && (best_s & 1u) && !(s & 1u);
            if (z > best_z || tie) {
                best_d = d;
                best_s = s;
                best_z = z;
            }
        }
        (void)best_d;
        /* commit_window: strictly more zeros than the incumbent span (pad 1)
         * -> deposit, dropping bits past the end (:35-37, bitvector.hpp:97-100). */
        const uint32_t inc = extract_pad1(bv, m, j, w);
        if (best_z > zeros_of(inc, w) || (g_variant == 3 && best_z == zeros_of(inc, w))) {
            for (unsigned k = 0; k < w && j + k < m; ++k) bv[j + k] = (uint8_t)((best_s >> k) & 1u);
        }
    }
    uint32_t ones = 0;
    for (size_t j = 0; j < m; ++j) ones += bv[j];
    *estimate = ones;
    *accept = ones <= e; /* :56-57 */
}

/* shouji_filter(pattern, text, e, width) for one pair of validated strings.
 * Returns SO_LENGTH_MISMATCH / SO_INVALID_PARAMETERS in the reference's
 * order (:44-47); e >= m accepts with estimate 0 and all-zero bits (:48-49). */
int so_shouji_one(const char* pattern, size_t pattern_len, const char* text, size_t text_len,
                  uint32_t e, unsigned w, uint8_t* bits_out, uint32_t* estimate, int* accept) {
    if (pattern_len != text_len) return SO_LENGTH_MISMATCH;
    if (w < 3 || w > 8) return SO_INVALID_PARAMETERS;
    const size_t m = text_len;
    if ((size_t)e >= m) {
        if (bits_out) memset(bits_out, 0, m);
        *estimate = 0;
        *accept = 1;
        return SO_OK;
    }
    uint8_t* map = (uint8_t*)malloc((2 * (size_t)e + 1) * m);
    uint8_t* bv = bits_out ? bits_out : (uint8_t*)malloc(m);
    shouji_core(pattern, text, m, e, w, map, bv, estimate, accept);
    if (!bits_out) free(bv);
    free(map);
    return SO_OK;
}

typedef struct {
    const char* text;
    const char* pattern;
    size_t stride, m, begin, end;
    uint32_t e;
    unsigned w;
    uint8_t* acc;
    uint32_t* estimates;
    uint64_t* bits;
    size_t words_per_pair;
} so_job;

static void* so_worker(void* arg) {
    so_job* job = (so_job*)arg;
    const size_t m = job->m;
    uint8_t* map = (uint8_t*)malloc((2 * (size_t)job->e + 1) * m);
    uint8_t* bv = (uint8_t*)malloc(m);
    for (size_t i = job->begin; i < job->end; ++i) {
        uint32_t est;
        int accept;
        shouji_core(job->pattern + i * job->stride, job->text + i * job->stride, m, job->e, job->w,
                    map, bv, &est, &accept);
        job->acc[i] = (uint8_t)accept;
        if (job->estimates) job->estimates[i] = est;
        if (job->bits) {
            uint64_t* dst = job->bits + i * job->words_per_pair;
            memset(dst, 0, job->words_per_pair * sizeof(uint64_t));
            for (size_t j = 0; j < m; ++j)
                if (bv[j]) dst[j >> 6] |= (uint64_t)1 << (j & 63);
        }
    }
    free(bv);
    free(map);
    return NULL;
}

/* Batch form over ASCII records, the way the reference's callers drive it:
 * every pair is packed first (text then pattern per pair, dataset.cpp:28-30),
 * so the first illegal byte in pair order wins; then shouji_filter runs per
 * pair through a static contiguous split like parallel_for_pairs
 * (evaluate.cpp:23-48). accept_bitmap is LSB-first, ceil(n/32) words. */
int so_shouji_batch(const char* text, const char* pattern, size_t stride, size_t n, size_t m,
                    uint32_t e, unsigned w, unsigned threads, uint32_t* accept_bitmap,
                    uint32_t* estimates, uint64_t* bits, so_error* err) {
    if (err) memset(err, 0, sizeof(*err));
    if (n == 0) return SO_OK;
    for (size_t i = 0; i < n; ++i) {
        for (int field = 0; field < 2; ++field) {
            uint64_t pos = 0;
            int byte = 0;
            const int st = so_validate((field == 0 ? text : pattern) + i * stride, m, &pos, &byte);
            if (st != SO_OK) {
                if (err) {
                    err->code = st;
                    err->pair = i;
                    err->field = field;
                    err->position = pos;
                    err->byte = byte;
                }
                return st;
            }
        }
    }
    if (w < 3 || w > 8) {
        if (err) err->code = SO_INVALID_PARAMETERS;
        return SO_INVALID_PARAMETERS;
    }
    const size_t words_per_pair = (m + 63) / 64;
    if (accept_bitmap) memset(accept_bitmap, 0, ((n + 31) / 32) * sizeof(uint32_t));
    if ((size_t)e >= m) {
        for (size_t i = 0; i < n; ++i) {
            if (accept_bitmap) accept_bitmap[i / 32] |= 1u << (i % 32);
            if (estimates) estimates[i] = 0;
        }
        if (bits) memset(bits, 0, n * words_per_pair * sizeof(uint64_t));
        return SO_OK;
    }
    uint8_t* acc = (uint8_t*)calloc(n, 1);
    if (threads < 1) threads = 1;
    if (threads > n) threads = (unsigned)n;
    pthread_t* tids = (pthread_t*)malloc(threads * sizeof(pthread_t));
    so_job* jobs = (so_job*)malloc(threads * sizeof(so_job));
    for (unsigned t = 0; t < threads; ++t) {
        so_job j = {text, pattern, stride, m, n * t / threads, n * (t + 1) / threads, e, w,
                    acc, estimates, bits, words_per_pair};
        jobs[t] = j;
        if (threads == 1)
            so_worker(&jobs[t]);
        else
            pthread_create(&tids[t], NULL, so_worker, &jobs[t]);
    }
    if (threads > 1)
        for (unsigned t = 0; t < threads; ++t) pthread_join(tids[t], NULL);
    if (accept_bitmap)
        for (size_t i = 0; i < n; ++i)
            if (acc[i]) accept_bitmap[i / 32] |= 1u << (i % 32);
    free(jobs);
    free(tids);
    free(acc);
    return SO_OK;
}

/* Test-only: select a mutated rule set for subsequent calls (not thread-safe
 * against concurrent batches; the tests call it serially). */
void so_set_variant(int v) { g_variant = v; }

/* ---- seeded generator: restatement of generate_pairs (proj/src/dataset.cpp:71-126) ----
 * std::mt19937_64 is the published MT19937-64 (Matsumoto & Nishimura 2000;
 * the parameters std::mersenne_twister_engine fixes for mt19937_64), default
 * seeding per [rand.eng.mers]. Draws are reduced by modulo exactly as the
 * reference does, so the bytes match the reference generator's. */
typedef struct {
    uint64_t mt[312];
    int mti;
} so_mt64;

static void mt64_seed(so_mt64* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->mti = 312;
}

static uint64_t mt64_next(so_mt64* r) {
    static const uint64_t mag01[2] = {0ULL, 0xB5026F5AA96619E9ULL};
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    if (r->mti >= 312) {
        int i;
        uint64_t x;
        for (i = 0; i < 312 - 156; ++i) {
            x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
            r->mt[i] = r->mt[i + 156] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        }
        for (; i < 311; ++i) {
            x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
            r->mt[i] = r->mt[i + (156 - 312)] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        }
        x = (r->mt[311] & UM) | (r->mt[0] & LM);
        r->mt[311] = r->mt[155] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        r->mti = 0;
    }
    uint64_t x = r->mt[r->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

/* text uniform ACGT (:92-93); k = lo + rng()%span (:96); type rng()%3 (:98);
 * substitution always changes the base (random_other_base :63-67); insertion
 * at rng()%(size+1) (:105); deletion skipped at size 1 (:111); then truncate
 * or pad with random bases at the tail (:119-120). Invalid parameters are
 * rejected in the reference's order (:72-78). */
int so_generate_pairs(uint64_t seed, size_t count, size_t len, uint32_t lo, uint32_t hi,
                      char* text, char* pattern, size_t stride) {
    if (count == 0 || len == 0 || lo > hi || hi > len) return SO_INVALID_PARAMETERS;
    static const char bases[4] = {'A', 'C', 'G', 'T'};
    so_mt64* rng = (so_mt64*)malloc(sizeof(so_mt64));
    mt64_seed(rng, seed);
    const uint64_t span = (uint64_t)hi - lo + 1;
    char* pat = (char*)malloc(len + (size_t)hi + 1);
    for (size_t p = 0; p < count; ++p) {
        char* t = text + p * stride;
        for (size_t i = 0; i < len; ++i) t[i] = bases[mt64_next(rng) % 4];
        size_t sz = len;
        memcpy(pat, t, len);
        const uint64_t edits = lo + mt64_next(rng) % span;
        for (uint64_t k = 0; k < edits; ++k) {
            switch (mt64_next(rng) % 3) {
                case 0: { /* substitution */
                    const size_t pos = (size_t)(mt64_next(rng) % sz);
                    int idx = 0;
                    while (bases[idx] != pat[pos]) ++idx;
                    pat[pos] = bases[(idx + 1 + mt64_next(rng) % 3) % 4];
                    break;
                }
                case 1: { /* insertion */
                    const size_t pos = (size_t)(mt64_next(rng) % (sz + 1));
                    const char b = bases[mt64_next(rng) % 4];
                    memmove(pat + pos + 1, pat + pos, sz - pos);
                    pat[pos] = b;
                    ++sz;
                    break;
                }
                case 2: { /* deletion */
                    if (sz == 1) break;
                    const size_t pos = (size_t)(mt64_next(rng) % sz);
                    memmove(pat + pos, pat + pos + 1, sz - pos - 1);
                    --sz;
                    break;
                }
            }
        }
        if (sz > len) sz = len;
        while (sz < len) pat[sz++] = bases[mt64_next(rng) % 4];
        memcpy(pattern + p * stride, pat, len);
    }
    free(pat);
    free(rng);
    return SO_OK;
}

/* substitution_pairs — proj/tests/acceptance_tests.cpp:252-276 (criterion 7's
 * substitution-only sets): per pair, text = m uniform bases (rng()%4); k =
 * rng() % (max_subs+1); k times: pos = rng()%m, then draw bases (rng()%4)
 * until one differs from pattern[pos] and write it. Same mt19937_64 stream
 * as generate_pairs. */
void so_substitution_pairs(uint64_t seed, size_t count, size_t m, uint32_t max_subs, char* text,
                           char* pattern, size_t stride) {
    static const char bases[4] = {'A', 'C', 'G', 'T'};
    so_mt64* rng = (so_mt64*)malloc(sizeof(so_mt64));
    mt64_seed(rng, seed);
    for (size_t p = 0; p < count; ++p) {
        char* t = text + p * stride;
        char* q = pattern + p * stride;
        for (size_t i = 0; i < m; ++i) t[i] = bases[mt64_next(rng) % 4];
        memcpy(q, t, m);
        const uint32_t k = (uint32_t)(mt64_next(rng) % ((uint64_t)max_subs + 1));
        for (uint32_t j = 0; j < k; ++j) {
            const size_t pos = (size_t)(mt64_next(rng) % m);
            char ch = bases[mt64_next(rng) % 4];
            while (ch == q[pos]) ch = bases[mt64_next(rng) % 4];
            q[pos] = ch;
        }
    }
    free(rng);
}

/* banded_edit_distance — proj/src/edit_distance.cpp:26-70, restated as the
 * plain full DP clipped at e+1 (equal lengths; N never matches). Returns the
 * distance, or -1 when it exceeds e. Used only for eval-style tests. */
int32_t so_banded_edit_distance(const char* a, const char* b, size_t m, uint32_t e) {
    uint32_t* prev = (uint32_t*)malloc((m + 1) * sizeof(uint32_t));
    uint32_t* cur = (uint32_t*)malloc((m + 1) * sizeof(uint32_t));
    for (size_t j = 0; j <= m; ++j) prev[j] = (uint32_t)j;
    for (size_t i = 1; i <= m; ++i) {
        cur[0] = (uint32_t)i;
        for (size_t j = 1; j <= m; ++j) {
            uint32_t v = prev[j - 1] + (mismatch(a[i - 1], b[j - 1]) ? 1u : 0u);
            if (prev[j] + 1 < v) v = prev[j] + 1;
            if (cur[j - 1] + 1 < v) v = cur[j - 1] + 1;
            cur[j] = v;
        }
        uint32_t* tmp = prev;
        prev = cur;
        cur = tmp;
    }
    const uint32_t d = prev[m];
    free(prev);
    free(cur);
    return d <= e ? (int32_t)d : -1;
}

/* ---- MAGNET (proj/src/magnet.cpp) --------------------------------------- */

/* longest_zero_run — proj/src/magnet.cpp:9-22: the longest run of zeros in
 * bits[lo..hi] (inclusive, hi clipped to m-1); the earliest wins ties; an
 * inverted or empty range gives len 0 with start = lo. */
void so_longest_zero_run(const uint8_t* bits, size_t m, size_t lo, size_t hi, size_t* start,
                         size_t* len) {
    size_t best_start = lo, best_len = 0, run_start = 0, run_len = 0;
    const size_t end = hi < m ? hi : m - 1;
    for (size_t i = lo; i <= end && lo <= hi; ++i) {
        if (!bits[i]) {
            if (run_len == 0) run_start = i;
            if (++run_len > best_len) {
                best_start = run_start;
                best_len = run_len;
            }
        } else {
            run_len = 0;
        }
    }
    *start = best_start;
    *len = best_len;
}

typedef struct {
    int diagonal;
    size_t start, len, lo, hi;
} so_extraction;

typedef struct {
    uint8_t* map; /* (2e+1) x m, row d+e, mutated by column masking */
    size_t m;
    uint32_t e;
    uint32_t budget;
    uint8_t* bv;
    so_extraction* out;
    size_t nout;
} so_magnet_state;

/* exen — proj/src/magnet.cpp:29-66: nominate each diagonal's longest run in
 * the active range in the order 0, -1, +1, -2, +2, ... (only a strictly longer
 * run displaces the incumbent), extract the winner (clear its bits in bv),
 * mask the run plus one flanking column on every diagonal
 * (neighborhood_map::mask_columns, neighborhood.cpp:88-91), then recurse into
 * the left range, then the right range, on the shared budget. */
static void so_exen(so_magnet_state* s, int64_t lo, int64_t hi) {
    if (s->budget == 0 || lo > hi) return;
    const size_t clo = (size_t)(lo < 0 ? 0 : lo);
    const size_t chi = (size_t)(hi >= (int64_t)s->m ? (int64_t)s->m - 1 : hi);
    if (clo > chi) return;
    const int e = (int)s->e;
    size_t best_start = 0, best_len = 0;
    int best_d = 0;
    for (int step = 0; step <= e; ++step) {
        for (int k = 0; k < 2; ++k) {
            const int d = k == 0 ? -step : step;
            size_t st, ln;
            so_longest_zero_run(s->map + (size_t)(d + e) * s->m, s->m, clo, chi, &st, &ln);
            if (ln > best_len) {
                best_start = st;
                best_len = ln;
                best_d = d;
            }
            if (step == 0) break;
        }
    }
    if (best_len == 0) return;
    --s->budget;
    for (size_t i = best_start; i < best_start + best_len; ++i) s->bv[i] = 0;
    if (s->out) {
        so_extraction x = {best_d, best_start, best_len, clo, chi};
        s->out[s->nout] = x;
    }
    ++s->nout;
    /* mask_columns(lo', hi') sets columns lo'..hi' (inclusive) to 1 on every diagonal */
    const size_t mlo = best_start > 0 ? best_start - 1 : 0;
    const size_t mhi = best_start + best_len;
    if (mlo <= mhi && mlo < s->m)
        for (int d = -e; d <= e; ++d)
            for (size_t i = mlo; i <= mhi && i < s->m; ++i) s->map[(size_t)(d + e) * s->m + i] = 1;
    so_exen(s, lo, (int64_t)best_start - 2);
    so_exen(s, (int64_t)(best_start + best_len) + 1, hi);
}

/* recover_subsequences — proj/src/magnet.cpp:70-75 (on a copy of the map). bv
 * (m bytes) starts all ones; out (nullable, >= budget entries) receives the
 * extractions in order. Returns the number of extractions. */
size_t so_recover_subsequences(const char* pattern, const char* text, size_t m, uint32_t e,
                               uint32_t budget, uint8_t* bv, so_extraction* out) {
    uint8_t* map = (uint8_t*)malloc((2 * (size_t)e + 1) * m);
    so_neighborhood(pattern, text, m, e, map);
    memset(bv, 1, m);
    so_magnet_state s = {map, m, e, budget, bv, out, 0};
    so_exen(&s, 0, (int64_t)m - 1);
    free(map);
    return s.nout;
}

/* magnet_filter — proj/src/magnet.cpp:77-87: length check, e >= m accepts
 * with estimate 0 and all-zero bits, else e+1 extractions; estimate =
 * popcount(bv), accept = estimate <= e. */
int so_magnet_one(const char* pattern, size_t pattern_len, const char* text, size_t text_len,
                  uint32_t e, uint8_t* bits_out, uint32_t* estimate, int* accept) {
    if (pattern_len != text_len) return SO_LENGTH_MISMATCH;
    const size_t m = text_len;
    if ((size_t)e >= m) {
        if (bits_out) memset(bits_out, 0, m);
        *estimate = 0;
        *accept = 1;
        return SO_OK;
    }
    uint8_t* bv = bits_out ? bits_out : (uint8_t*)malloc(m);
    so_recover_subsequences(pattern, text, m, e, e + 1, bv, NULL);
    uint32_t ones = 0;
    for (size_t j = 0; j < m; ++j) ones += bv[j];
    *estimate = ones;
    *accept = ones <= e;
    if (!bits_out) free(bv);
    return SO_OK;
}

typedef struct {
    const char* text;
    const char* pattern;
    size_t stride, m, begin, end;
    uint32_t e;
    uint8_t* acc;
    uint32_t* estimates;
    uint64_t* bits;
    size_t words_per_pair;
} so_mjob;

static void* so_magnet_worker(void* arg) {
    so_mjob* job = (so_mjob*)arg;
    const size_t m = job->m;
    uint8_t* bv = (uint8_t*)malloc(m);
    for (size_t i = job->begin; i < job->end; ++i) {
        uint32_t est;
        int accept;
        so_magnet_one(job->pattern + i * job->stride, m, job->text + i * job->stride, m, job->e,
                      bv, &est, &accept);
        job->acc[i] = (uint8_t)accept;
        if (job->estimates) job->estimates[i] = est;
        if (job->bits) {
            uint64_t* dst = job->bits + i * job->words_per_pair;
            memset(dst, 0, job->words_per_pair * sizeof(uint64_t));
            for (size_t j = 0; j < m; ++j)
                if (bv[j]) dst[j >> 6] |= (uint64_t)1 << (j & 63);
        }
    }
    free(bv);
    return NULL;
}

/* Batch MAGNET over ASCII records, as run_filter(magnet) is driven by the
 * reference's callers (evaluate.cpp:13-48): validation of every pair first
 * (text then pattern, first error wins), then magnet_filter per pair. */
int so_magnet_batch(const char* text, const char* pattern, size_t stride, size_t n, size_t m,
                    uint32_t e, unsigned threads, uint32_t* accept_bitmap, uint32_t* estimates,
                    uint64_t* bits, so_error* err) {
    if (err) memset(err, 0, sizeof(*err));
    if (n == 0) return SO_OK;
    for (size_t i = 0; i < n; ++i) {
        for (int field = 0; field < 2; ++field) {
            uint64_t pos = 0;
            int byte = 0;
            const int st = so_validate((field == 0 ? text : pattern) + i * stride, m, &pos, &byte);
            if (st != SO_OK) {
                if (err) {
                    err->code = st;
                    err->pair = i;
                    err->field = field;
                    err->position = pos;
                    err->byte = byte;
                }
                return st;
            }
        }
    }
    const size_t words_per_pair = (m + 63) / 64;
    if (accept_bitmap) memset(accept_bitmap, 0, ((n + 31) / 32) * sizeof(uint32_t));
    uint8_t* acc = (uint8_t*)calloc(n, 1);
    if (threads < 1) threads = 1;
    if (threads > n) threads = (unsigned)n;
    pthread_t* tids = (pthread_t*)malloc(threads * sizeof(pthread_t));
    so_mjob* jobs = (so_mjob*)malloc(threads * sizeof(so_mjob));
    for (unsigned t = 0; t < threads; ++t) {
        so_mjob j = {text, pattern, stride, m, n * t / threads, n * (t + 1) / threads, e,
                     acc, estimates, bits, words_per_pair};
        jobs[t] = j;
        if (threads == 1)
            so_magnet_worker(&jobs[t]);
        else
            pthread_create(&tids[t], NULL, so_magnet_worker, &jobs[t]);
    }
    if (threads > 1)
        for (unsigned t = 0; t < threads; ++t) pthread_join(tids[t], NULL);
    if (accept_bitmap)
        for (size_t i = 0; i < n; ++i)
            if (acc[i]) accept_bitmap[i / 32] |= 1u << (i % 32);
    free(jobs);
    free(tids);
    free(acc);
    return SO_OK;
}
