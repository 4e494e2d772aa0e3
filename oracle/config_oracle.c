/*
 * TEST INFRASTRUCTURE ONLY — full-size checker for the BASELINE configs.
 *
 * Two pieces, both compiled into oracle/_build/libshouji_oracle.so next to
 * shouji_oracle.c and never linked into the product:
 *
 *  1. so_gen_config*: a byte-identical CPU mirror of the device generator of
 *     BASELINE.json configs 1-4 (paper_1809_07858_b200/csrc/datagen.cu). The
 *     generator is counter based (one splitmix64 stream per pair, keyed by
 *     (kind, seed, param, pair)), so any pair index can be produced on its own:
 *     the GPU tests regenerate sampled rows here and compare bytes.
 *
 *  2. so_shouji_fast_*: the reference's shouji_filter (proj/src/shouji.cpp:41-58)
 *     restated with the same loops and rules as shouji_oracle.c, reordered only
 *     so the compiler can vectorise it:
 *       - neighborhood_map (proj/src/neighborhood.cpp:41-79): the mismatch cell
 *         of diagonal d at column j is computed per byte, with N coded
 *         differently in pattern and text so that "N never matches"
 *         (packed_sequence.hpp:58-61) is a plain inequality;
 *       - select_window (shouji.cpp:17-31): for every window j the candidates
 *         are visited in the reference's order d = -e..+e and the reference's
 *         two-clause rule (more zeros, or equal zeros with the incumbent's
 *         bit 0 set and the candidate's clear) decides; the loop nest is
 *         d-outer / j-inner, which visits each window's candidates in the
 *         same order;
 *       - commit_window (shouji.cpp:33-39) and the final popcount (:56-57) are
 *         the serial per-column loop of the reference.
 *     It is pinned to the plain restatement and to the reference library
 *     (oracle/_ref) on every config by tests/test_oracle_configs.py, and is what
 *     tests/golden/make_fullsize_digests.py runs over the full BASELINE sizes
 *     (the reference library cross-checks chunks of those runs).
 */
#include <pthread.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- 1. generator mirror (paper_1809_07858_b200/csrc/datagen.cu) ---------- */

#define GEN_MAX_M 1024
#define GEN_SLACK 64

typedef struct {
    uint64_t s;
} gen_rng;

static uint64_t gen_next(gen_rng* r) {
    uint64_t z = (r->s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static double gen_uniform(gen_rng* r) {
    return (double)(gen_next(r) >> 11) * (1.0 / 9007199254740992.0);
}

static char gen_base(uint64_t r) { return "ACGT"[r & 3u]; }

static char gen_other_base(char old, uint64_t r) {
    const int idx = old == 'A' ? 0 : old == 'C' ? 1 : old == 'G' ? 2 : 3;
    return "ACGT"[(idx + 1 + (int)(r % 3)) % 4];
}

static void gen_apply_edit(char* s, int* size, int type, int lo, int hi, gen_rng* rng) {
    switch (type) {
        case 0: {
            if (*size == 0) return;
            const int h = hi < *size ? hi : *size;
            const int l = lo < h ? lo : 0;
            const int pos = l + (int)(gen_next(rng) % (uint64_t)(h - l));
            if (s[pos] == 'N') return;
            s[pos] = gen_other_base(s[pos], gen_next(rng));
            break;
        }
        case 1: {
            if (*size >= GEN_MAX_M + GEN_SLACK - 1) return;
            const int h = (hi < *size ? hi : *size) + 1;
            const int l = lo < h ? lo : 0;
            const int pos = l + (int)(gen_next(rng) % (uint64_t)(h - l));
            const char b = gen_base(gen_next(rng));
            for (int i = *size; i > pos; --i) s[i] = s[i - 1];
            s[pos] = b;
            ++*size;
            break;
        }
        default: {
            if (*size <= 1) return;
            const int h = hi < *size ? hi : *size;
            const int l = lo < h ? lo : 0;
            const int pos = l + (int)(gen_next(rng) % (uint64_t)(h - l));
            for (int i = pos; i < *size - 1; ++i) s[i] = s[i + 1];
            --*size;
            break;
        }
    }
}

/* Poisson(6) by inversion; exp(-6) as its correctly rounded double and every
 * step rounded separately (the device uses __dmul_rn/__ddiv_rn/__dadd_rn, this
 * file is compiled with -ffp-contract=off). */
static int gen_poisson6(gen_rng* rng) {
    const double u = gen_uniform(rng);
    double p = 0x1.44e51f113d4d6p-9; /* exp(-6) */
    double cdf = p;
    int k = 0;
    while (u > cdf && k < 200) {
        ++k;
        p = p * (6.0 / (double)k);
        cdf = cdf + p;
    }
    return k;
}

/* One pair of config `kind` (1..4): the body of generate_pairs_kernel. */
int so_gen_config_pair(int kind, uint64_t seed, uint32_t param, uint64_t p, int m, char* trow,
                       char* prow) {
    if (kind < 1 || kind > 4 || m < 1 || m > GEN_MAX_M) return -1;
    gen_rng rng = {seed * 0x2545F4914F6CDD1Dull ^ ((uint64_t)kind << 56) ^ ((uint64_t)param << 40) ^
                   (p * 0xD1B54A32D192ED03ull)};
    gen_next(&rng);
    char t[GEN_MAX_M];
    char s[GEN_MAX_M + GEN_SLACK];

    if (kind == 4) {
        const uint64_t r = gen_next(&rng) % 10;
        if (r < 3) {
            const int period = 1 + (int)(gen_next(&rng) % 6);
            char unit[6];
            for (int i = 0; i < period; ++i) unit[i] = gen_base(gen_next(&rng));
            for (int i = 0; i < m; ++i) t[i] = unit[i % period];
        } else {
            for (int i = 0; i < m; ++i) t[i] = gen_base(gen_next(&rng));
            if (r == 3) {
                const int runs = 1 + (int)(gen_next(&rng) % 4);
                for (int k = 0; k < runs; ++k) {
                    const int len = 5 + (int)(gen_next(&rng) % 16);
                    const int start = (int)(gen_next(&rng) % (uint64_t)m);
                    const char b = gen_base(gen_next(&rng));
                    for (int i = start; i < start + len && i < m; ++i) t[i] = b;
                }
            }
        }
    } else {
        for (int i = 0; i < m; ++i) t[i] = gen_base(gen_next(&rng));
    }

    int unrelated = 0, k = 0, burst_lo = 0;
    const int e = (int)param;
    switch (kind) {
        case 1:
            unrelated = (gen_next(&rng) & 1u) != 0;
            k = (int)(gen_next(&rng) % (uint64_t)(2 * e + 1));
            break;
        case 2:
            unrelated = gen_next(&rng) % 10 < 3;
            k = gen_poisson6(&rng);
            break;
        case 3:
            k = (int)(gen_next(&rng) % (uint64_t)(2 * e + 1));
            burst_lo = m > 20 ? (int)(gen_next(&rng) % (uint64_t)(m - 20 + 1)) : 0;
            break;
        default:
            k = (int)(gen_next(&rng) % 41);
            break;
    }
    int size = m;
    if (unrelated) {
        for (int i = 0; i < m; ++i) s[i] = gen_base(gen_next(&rng));
    } else {
        for (int i = 0; i < m; ++i) s[i] = t[i];
        for (int q = 0; q < k; ++q) {
            int type;
            if (kind == 2) {
                const uint64_t r = gen_next(&rng) % 10;
                type = r < 6 ? 0 : (r < 8 ? 1 : 2);
            } else {
                type = (int)(gen_next(&rng) % 3);
            }
            int lo = 0, hi = 1 << 30;
            if (kind == 3 && (gen_next(&rng) & 1u)) {
                lo = burst_lo;
                hi = burst_lo + 20;
            }
            gen_apply_edit(s, &size, type, lo, hi, &rng);
        }
        if (size > m) size = m;
        while (size < m) s[size++] = gen_base(gen_next(&rng));
    }
    if (kind == 4) {
        for (int i = 0; i < m; ++i) {
            if (gen_next(&rng) % 1000 == 0) t[i] = 'N';
            if (gen_next(&rng) % 1000 == 0) s[i] = 'N';
        }
    }
    memcpy(trow, t, (size_t)m);
    memcpy(prow, s, (size_t)m);
    return 0;
}

/* Pairs [begin, begin+count) into records of `pitch` bytes (bytes past m are
 * left as they are). */
int so_gen_config(int kind, uint64_t seed, uint32_t param, int m, uint64_t begin, size_t count,
                  char* text, char* pattern, size_t pitch) {
    for (size_t i = 0; i < count; ++i) {
        const int st = so_gen_config_pair(kind, seed, param, begin + i, m, text + i * pitch,
                                          pattern + i * pitch);
        if (st) return st;
    }
    return 0;
}

/* Arbitrary pair indices (the GPU tests' sampled rows). */
int so_gen_config_rows(int kind, uint64_t seed, uint32_t param, int m, const uint64_t* idx,
                       size_t count, char* text, char* pattern, size_t pitch) {
    for (size_t i = 0; i < count; ++i) {
        const int st = so_gen_config_pair(kind, seed, param, idx[i], m, text + i * pitch,
                                          pattern + i * pitch);
        if (st) return st;
    }
    return 0;
}

/* ---- 2. shouji_filter, vectorisable restatement ---------------------------- */

typedef struct {
    int m;
    uint32_t e;
    unsigned w;
    uint8_t* pc;  /* pattern codes, padded: [e + m + e] */
    uint8_t* tc;  /* text codes [m] */
    uint8_t* dg;  /* one diagonal, padded with 1 to m + 8 */
    uint8_t* bs;  /* best slice per window */
    uint8_t* bz;  /* best zeros per window */
    uint8_t* bv;  /* tally bits, padded with 1 to m + 8 */
} fast_ws;

static int fast_ws_init(fast_ws* ws, int m, uint32_t e, unsigned w) {
    ws->m = m;
    ws->e = e;
    ws->w = w;
    const size_t pad = (size_t)m + 2 * (size_t)e + 16;
    ws->pc = (uint8_t*)malloc(pad);
    ws->tc = (uint8_t*)malloc((size_t)m + 16);
    ws->dg = (uint8_t*)malloc((size_t)m + 16);
    ws->bs = (uint8_t*)malloc((size_t)m + 16);
    ws->bz = (uint8_t*)malloc((size_t)m + 16);
    ws->bv = (uint8_t*)malloc((size_t)m + 16);
    return ws->pc && ws->tc && ws->dg && ws->bs && ws->bz && ws->bv ? 0 : -1;
}

static void fast_ws_free(fast_ws* ws) {
    free(ws->pc);
    free(ws->tc);
    free(ws->dg);
    free(ws->bs);
    free(ws->bz);
    free(ws->bv);
}

/* codes: A,C,G,T -> 0..3. 'N' -> 4 in the pattern and 5 in the text, and a
 * pattern index outside [0,m) -> 6: every such cell compares unequal to any
 * text code, which is exactly neighborhood.cpp:67-76 (out of range, N on either
 * side, or different bases). */
static uint8_t code_of(char c, uint8_t ncode) {
    switch (c) {
        case 'A': return 0;
        case 'C': return 1;
        case 'G': return 2;
        case 'T': return 3;
        default: return ncode;
    }
}

/* select_window over all windows for diagonals -e..+e (shouji.cpp:17-31), W a
 * compile-time width so the j loop vectorises. dg has 1 at [m, m+16)
 * (extract(pos, w, pad = 1)). */
static inline __attribute__((always_inline)) void select_all(
    const uint8_t* restrict pc, const uint8_t* restrict tc, uint8_t* restrict dg,
    uint8_t* restrict bs, uint8_t* restrict bz, int m, int e, const unsigned W) {
    for (int d = -e; d <= e; ++d) {
        /* neighborhood_map row d: bit j = cell (j+d, j) */
        const uint8_t* restrict prow = pc + e + d;
        for (int j = 0; j < m; ++j) dg[j] = prow[j] != tc[j];
        if (d == -e) {
            /* the scan starts from the first diagonal (shouji.cpp:19-20) */
            for (int j = 0; j < m; ++j) {
                /* slice = sum dg[j+k] << k, by Horner steps (byte adds vectorise) */
                uint8_t s = dg[j + W - 1], ones = dg[j + W - 1];
                for (int k = (int)W - 2; k >= 0; --k) {
                    s = (uint8_t)(s + s + dg[j + k]);
                    ones = (uint8_t)(ones + dg[j + k]);
                }
                bs[j] = s;
                bz[j] = (uint8_t)(W - ones);
            }
        } else {
            /* shouji.cpp:21-29: replace on more zeros, or on equal zeros when the
             * incumbent's leading bit is 1 and the candidate's is 0 */
            for (int j = 0; j < m; ++j) {
                /* slice = sum dg[j+k] << k, by Horner steps (byte adds vectorise) */
                uint8_t s = dg[j + W - 1], ones = dg[j + W - 1];
                for (int k = (int)W - 2; k >= 0; --k) {
                    s = (uint8_t)(s + s + dg[j + k]);
                    ones = (uint8_t)(ones + dg[j + k]);
                }
                const uint8_t z = (uint8_t)(W - ones);
                const uint8_t b = bz[j], sl = bs[j];
                const uint8_t lead = (uint8_t)((sl & (uint8_t)~s) & 1u); /* incumbent 1, candidate 0 */
                const uint8_t gt = (uint8_t)(z > b ? 0xFF : 0);
                const uint8_t eq = (uint8_t)(z == b ? 0xFF : 0);
                const uint8_t take = (uint8_t)(gt | (eq & (uint8_t)(0 - lead)));
                bs[j] = (uint8_t)((s & take) | (sl & (uint8_t)~take));
                bz[j] = (uint8_t)((z & take) | (b & (uint8_t)~take));
            }
        }
    }
}

/* Precondition (the reference's order, shouji.cpp:44-49): lengths equal,
 * 3 <= w <= 8, e < m, both strings validated. Returns the estimate; bits_out
 * (nullable) receives one byte per tally bit. */
static uint32_t fast_core(fast_ws* ws, const char* pattern, const char* text, uint8_t* bits_out) {
    const int m = ws->m;
    const int e = (int)ws->e;
    const unsigned w = ws->w;
    uint8_t* pc = ws->pc;
    for (int i = 0; i < e; ++i) pc[i] = 6;
    for (int i = 0; i < m; ++i) pc[e + i] = code_of(pattern[i], 4);
    for (int i = 0; i < e + 16; ++i) pc[e + m + i] = 6;
    for (int j = 0; j < m; ++j) ws->tc[j] = code_of(text[j], 5);
    uint8_t* dg = ws->dg;
    uint8_t* bs = ws->bs;
    uint8_t* bz = ws->bz;
    for (int j = m; j < m + 16; ++j) dg[j] = 1;
    switch (w) {
        case 3: select_all(pc, ws->tc, dg, bs, bz, m, e, 3); break;
        case 4: select_all(pc, ws->tc, dg, bs, bz, m, e, 4); break;
        case 5: select_all(pc, ws->tc, dg, bs, bz, m, e, 5); break;
        case 6: select_all(pc, ws->tc, dg, bs, bz, m, e, 6); break;
        case 7: select_all(pc, ws->tc, dg, bs, bz, m, e, 7); break;
        default: select_all(pc, ws->tc, dg, bs, bz, m, e, 8); break;
    }
    /* bitvector bv(m, true) (:52); commit_window per column (:53-55, :33-39) */
    uint8_t* bv = ws->bv;
    memset(bv, 1, (size_t)m + 16);
    for (int j = 0; j < m; ++j) {
        unsigned inc_ones = 0;
        for (unsigned k = 0; k < w; ++k) inc_ones += bv[j + k]; /* pad 1 past m */
        const unsigned inc_zeros = w - inc_ones;
        if (bz[j] > inc_zeros) {
            for (unsigned k = 0; k < w && j + (int)k < m; ++k) bv[j + k] = (bs[j] >> k) & 1u;
        }
    }
    uint32_t ones = 0;
    for (int j = 0; j < m; ++j) ones += bv[j];
    if (bits_out) memcpy(bits_out, bv, (size_t)m);
    return ones;
}

/* shouji_filter(pattern, text, e, w) on one validated pair of length m. */
int so_shouji_fast_one(const char* pattern, const char* text, int m, uint32_t e, unsigned w,
                       uint8_t* bits_out, uint32_t* estimate, int* accept) {
    if (w < 3 || w > 8) return 7;
    if ((int64_t)e >= m) {
        if (bits_out) memset(bits_out, 0, (size_t)m);
        *estimate = 0;
        *accept = 1;
        return 0;
    }
    fast_ws ws;
    if (fast_ws_init(&ws, m, e, w)) return -1;
    *estimate = fast_core(&ws, pattern, text, bits_out);
    *accept = *estimate <= e;
    fast_ws_free(&ws);
    return 0;
}

/* ---- batch drivers ---------------------------------------------------------- */

typedef struct {
    /* records mode */
    const char* text;
    const char* pattern;
    size_t stride;
    /* generator mode (text == NULL) */
    int kind;
    uint64_t seed;
    uint32_t param;
    uint64_t base;
    /* common */
    int m;
    uint32_t e;
    unsigned w;
    size_t begin, end;
    uint32_t* estimates;
    int status;
} fast_job;

static void* fast_worker(void* arg) {
    fast_job* job = (fast_job*)arg;
    fast_ws ws;
    if (fast_ws_init(&ws, job->m, job->e, job->w)) {
        job->status = -1;
        return NULL;
    }
    char tbuf[GEN_MAX_M], pbuf[GEN_MAX_M];
    for (size_t i = job->begin; i < job->end; ++i) {
        const char* t;
        const char* p;
        if (job->text) {
            t = job->text + i * job->stride;
            p = job->pattern + i * job->stride;
        } else {
            if (so_gen_config_pair(job->kind, job->seed, job->param, job->base + i, job->m, tbuf,
                                   pbuf)) {
                job->status = -1;
                break;
            }
            t = tbuf;
            p = pbuf;
        }
        job->estimates[i] = (int64_t)job->e >= job->m ? 0u : fast_core(&ws, p, t, NULL);
    }
    fast_ws_free(&ws);
    return NULL;
}

static int run_jobs(fast_job proto, size_t n, unsigned threads) {
    if (n == 0) return 0;
    if (threads < 1) threads = 1;
    if (threads > n) threads = (unsigned)n;
    pthread_t* tids = (pthread_t*)malloc(threads * sizeof(pthread_t));
    fast_job* jobs = (fast_job*)malloc(threads * sizeof(fast_job));
    for (unsigned t = 0; t < threads; ++t) {
        jobs[t] = proto;
        jobs[t].begin = n * t / threads;
        jobs[t].end = n * (t + 1) / threads;
        jobs[t].status = 0;
        pthread_create(&tids[t], NULL, fast_worker, &jobs[t]);
    }
    int st = 0;
    for (unsigned t = 0; t < threads; ++t) {
        pthread_join(tids[t], NULL);
        if (jobs[t].status) st = jobs[t].status;
    }
    free(jobs);
    free(tids);
    return st;
}

/* Estimates of n validated ASCII records (accept = estimate <= e, the
 * filter_decision invariant, filter_decision.hpp:12-16). */
int so_shouji_fast_batch(const char* text, const char* pattern, size_t stride, size_t n, int m,
                         uint32_t e, unsigned w, unsigned threads, uint32_t* estimates) {
    if (w < 3 || w > 8) return 7;
    fast_job proto;
    memset(&proto, 0, sizeof(proto));
    proto.text = text;
    proto.pattern = pattern;
    proto.stride = stride;
    proto.m = m;
    proto.e = e;
    proto.w = w;
    proto.estimates = estimates;
    return run_jobs(proto, n, threads);
}

/* Estimates of pairs [begin, begin+count) of config `kind`, generated on the
 * fly by the mirror above (no record buffers: the full BASELINE sizes stream
 * through in chunks). */
int so_config_estimates(int kind, uint64_t seed, uint32_t param, int m, uint32_t e, unsigned w,
                        uint64_t begin, size_t count, unsigned threads, uint32_t* estimates) {
    if (w < 3 || w > 8) return 7;
    if (kind < 1 || kind > 4 || m < 1 || m > GEN_MAX_M) return -1;
    fast_job proto;
    memset(&proto, 0, sizeof(proto));
    proto.kind = kind;
    proto.seed = seed;
    proto.param = param;
    proto.base = begin;
    proto.m = m;
    proto.e = e;
    proto.w = w;
    proto.estimates = estimates;
    return run_jobs(proto, count, threads);
}
