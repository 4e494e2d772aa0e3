// Pair datasets: TSV ingest, the seeded generator and TSV output — the caller
// side of the hot path.
//
// Reference: load_pairs / load_pairs_file / write_pairs / generate_pairs,
// proj/src/dataset.cpp:13-126 (declared proj/include/prefilter/dataset.hpp).
//
// Records are kept as fixed-stride ASCII (stride = m) in pageable host memory
// (huge pages), so a dataset can be handed to pf_shouji_filter_batch without
// another copy. The line scan (two parallel passes: count, then fill) and the
// structural checks (tabs, empty fields, lengths) run on the host cores; the
// well-formed prefix's bytes are checked with the host pack's exact AVX-512
// alphabet test on the same worker pool, and the first illegal byte (lowest
// pair, text before pattern, lowest position) is mapped back to its line. The
// error reported is the one the reference's line-by-line loader would throw
// first:
//   per line: field count -> text codec (empty, then bytes) -> pattern codec
//   -> text/pattern length -> dataset length; then "no pairs in input".
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include "../../include/shouji_b200.h"
#include "host_pack.h"

struct pf_dataset {
    uint8_t* text = nullptr;  // n x m, pinned when possible
    uint8_t* pattern = nullptr;
    bool pinned = false;
    size_t n = 0;
    uint32_t m = 0;
    std::string source;
};

namespace {

// PF_TRACE=1: phase timings of the loader on stderr (diagnostics)
struct Trace {
    bool on = [] {
        const char* e = std::getenv("PF_TRACE");
        return e && e[0] == '1';
    }();
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char* what) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[pf_dataset] %-22s %8.1f ms\n", what,
                     std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

void set_parse(pf_error* err, int status, uint64_t line, const std::string& msg) {
    if (!err) return;
    err->status = status;
    err->line = line;
    std::snprintf(err->message, sizeof(err->message), "%s", msg.c_str());
}

// Records live in pageable memory (2 MiB-aligned, transparent huge pages):
// pinning a multi-GB dataset costs ~0.45 s/GB, and the batch entry points
// read pageable records as fast (host-pack path) or stage them.
bool alloc_records(pf_dataset* ds, size_t n, uint32_t m) {
    const size_t al = size_t(1) << 21;
    const size_t bytes = (std::max<size_t>(n * m, 1) + al - 1) / al * al;
    void* t = std::aligned_alloc(al, bytes);
    void* p = std::aligned_alloc(al, bytes);
    if (!t || !p) {
        std::free(t);
        std::free(p);
        return false;
    }
    madvise(t, bytes, MADV_HUGEPAGE);
    madvise(p, bytes, MADV_HUGEPAGE);
    ds->pinned = false;
    ds->text = static_cast<uint8_t*>(t);
    ds->pattern = static_cast<uint8_t*>(p);
    ds->n = n;
    ds->m = m;
    return true;
}

bool valid_base(char c) { return c == 'A' || c == 'C' || c == 'G' || c == 'T' || c == 'N'; }

// packed_sequence::from_string's checks on one field (packed_sequence.cpp:8,27-28).
bool check_codec(const char* s, size_t len, uint64_t line, pf_error* err) {
    if (len == 0) {
        set_parse(err, PF_ERR_PARSE, line, "line " + std::to_string(line) + ": empty sequence");
        return false;
    }
    for (size_t i = 0; i < len; ++i) {
        if (!valid_base(s[i])) {
            set_parse(err, PF_ERR_PARSE, line,
                      "line " + std::to_string(line) + ": illegal character '" +
                          std::string(1, s[i]) + "' at position " + std::to_string(i));
            if (err) {
                err->position = i;
                err->byte = static_cast<unsigned char>(s[i]);
            }
            return false;
        }
    }
    return true;
}

struct line_info {
    size_t begin = 0, tab = 0, end = 0;  // [begin, tab) text, (tab, end) pattern
    int tabs = 0;                        // 1 = well-formed field count
};

// Lines of [begin, end) of buf (std::getline semantics: a final unterminated
// line counts, a trailing '\n' does not start a new line).
size_t count_lines(const char* buf, size_t begin, size_t end) {
    if (begin >= end) return 0;
    const size_t nl = static_cast<size_t>(std::count(buf + begin, buf + end, '\n'));
    return nl + (buf[end - 1] != '\n' ? 1 : 0);
}

// Split [begin, end) of buf into lines, written to out[0..count_lines).
void scan_lines(const char* buf, size_t begin, size_t end, line_info* out) {
    size_t pos = begin, k = 0;
    while (pos < end) {
        const char* nl = static_cast<const char*>(std::memchr(buf + pos, '\n', end - pos));
        const size_t le = nl ? static_cast<size_t>(nl - buf) : end;
        line_info li;
        li.begin = pos;
        li.end = le;
        const char* t1 = static_cast<const char*>(std::memchr(buf + pos, '\t', le - pos));
        if (t1) {
            li.tab = static_cast<size_t>(t1 - buf);
            const char* t2 = static_cast<const char*>(std::memchr(t1 + 1, '\t', le - li.tab - 1));
            li.tabs = t2 ? 2 : 1;
        }
        out[k++] = li;
        pos = le + 1;
    }
}

}  // namespace

extern "C" {

int pf_dataset_load_tsv(pf_ctx* ctx, const char* data, size_t len, const char* source_name,
                        pf_dataset** out, pf_error* err) {
    if (err) std::memset(err, 0, sizeof(*err));
    if (!out || (!data && len)) return PF_ERR_NULL_ARGUMENT;
    *out = nullptr;
    (void)ctx;  // the loader runs on the host cores; kept for the ABI (pf_dataset_* take a ctx)
    Trace tr;
    // ---- line scan, in parallel over newline-aligned chunks ----------------------
    const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<size_t> cut(nt + 1, 0);
    cut[nt] = len;
    for (unsigned t = 1; t < nt; ++t) {
        size_t c = len * t / nt;
        const char* nl = c < len ? static_cast<const char*>(std::memchr(data + c, '\n', len - c))
                                 : nullptr;
        cut[t] = nl ? static_cast<size_t>(nl - data) + 1 : len;
        if (cut[t] < cut[t - 1]) cut[t] = cut[t - 1];
    }
    // two passes: count each chunk's lines, then fill one array at the offsets
    std::vector<size_t> first(nt + 1, 0);
    {
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < nt; ++t)
            pool.emplace_back([&, t] { first[t + 1] = count_lines(data, cut[t], cut[t + 1]); });
        for (auto& th : pool) th.join();
    }
    for (unsigned t = 0; t < nt; ++t) first[t + 1] += first[t];
    std::vector<line_info> lines(first[nt]);
    {
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < nt; ++t)
            pool.emplace_back(
                [&, t] { scan_lines(data, cut[t], cut[t + 1], lines.data() + first[t]); });
        for (auto& th : pool) th.join();
    }
    tr.mark("line scan");

    // ---- first structural problem (field count, empty field, lengths) ------------
    size_t ls = lines.size();  // index of the first line with a structural problem
    uint32_t m = 0;
    for (size_t i = 0; i < lines.size(); ++i) {
        const line_info& li = lines[i];
        if (li.tabs != 1) { ls = i; break; }
        const size_t tl = li.tab - li.begin, pl = li.end - li.tab - 1;
        if (tl == 0 || pl == 0 || tl != pl) { ls = i; break; }
        if (i == 0) m = static_cast<uint32_t>(tl);
        if (tl != m || tl >= (1u << 24)) { ls = i; break; }
    }
    // ---- records of the well-formed prefix; bytes validated on the GPU ------------
    auto* ds = new pf_dataset;
    ds->source = source_name ? source_name : "<stream>";
    tr.mark("structure check");
    if (!alloc_records(ds, ls, m)) {
        delete ds;
        return PF_ERR_OUT_OF_MEMORY;
    }
    tr.mark("alloc records");
    {
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < nt; ++t)
            pool.emplace_back([&, t] {
                for (size_t i = ls * t / nt; i < ls * (t + 1) / nt; ++i) {
                    std::memcpy(ds->text + i * m, data + lines[i].begin, m);
                    std::memcpy(ds->pattern + i * m, data + lines[i].tab + 1, m);
                }
            });
        for (auto& th : pool) th.join();
    }
    tr.mark("copy records");
    if (ls > 0) {
        // the alphabet check of the well-formed prefix (the host pack's AVX-512
        // check, exact first offender in pair order)
        sb::HostBad bad;
        sb::host_validate_parallel(ds->text, ds->pattern, m, static_cast<long long>(ls),
                                   static_cast<int>(m), &bad);
        if (bad.any) {
            const uint64_t line = bad.pair + 1;
            const line_info& li = lines[bad.pair];
            const char* f = data + (bad.field == 0 ? li.begin : li.tab + 1);
            pf_dataset_free(ds);
            check_codec(f, m, line, err);  // same message the reference builds
            return PF_ERR_PARSE;
        }
        tr.mark("validation");
    }
    if (ls < lines.size()) {  // the structural line, checked in the reference's order
        const line_info& li = lines[ls];
        const uint64_t line = ls + 1;
        pf_dataset_free(ds);
        if (li.tabs == 0) {
            set_parse(err, PF_ERR_PARSE, line,
                      "line " + std::to_string(line) + ": expected two tab-separated fields");
            return PF_ERR_PARSE;
        }
        if (li.tabs == 2) {
            set_parse(err, PF_ERR_PARSE, line,
                      "line " + std::to_string(line) +
                          ": expected two tab-separated fields, found more");
            return PF_ERR_PARSE;
        }
        const size_t tl = li.tab - li.begin, pl = li.end - li.tab - 1;
        if (!check_codec(data + li.begin, tl, line, err)) return PF_ERR_PARSE;
        if (!check_codec(data + li.tab + 1, pl, line, err)) return PF_ERR_PARSE;
        if (tl == pl && tl >= (1u << 24) && (ls == 0 || tl == m)) {
            // a well-formed line the reference would load: the records' length is
            // beyond this implementation's limit (m < 2^24), not a length mismatch
            set_parse(err, PF_ERR_INVALID_PARAMETERS, line,
                      "line " + std::to_string(line) + ": sequence length " + std::to_string(tl) +
                          " exceeds the supported maximum of " + std::to_string((1u << 24) - 1));
            return PF_ERR_INVALID_PARAMETERS;
        }
        if (tl != pl) {
            set_parse(err, PF_ERR_LENGTH_MISMATCH, line,
                      "length mismatch at line " + std::to_string(line) + ": " +
                          std::to_string(tl) + " vs " + std::to_string(pl));
            return PF_ERR_LENGTH_MISMATCH;
        }
        set_parse(err, PF_ERR_LENGTH_MISMATCH, line,
                  "length mismatch at line " + std::to_string(line) + ": " + std::to_string(m) +
                      " vs " + std::to_string(tl));
        return PF_ERR_LENGTH_MISMATCH;
    }
    if (ls == 0) {
        pf_dataset_free(ds);
        set_parse(err, PF_ERR_PARSE, 1, "line 1: no pairs in input");
        return PF_ERR_PARSE;
    }
    *out = ds;
    return PF_OK;
}

int pf_dataset_load_tsv_file(pf_ctx* ctx, const char* path, pf_dataset** out, pf_error* err) {
    if (err) std::memset(err, 0, sizeof(*err));
    if (!path || !out) return PF_ERR_NULL_ARGUMENT;
    Trace tr;
    const int fd = open(path, O_RDONLY);
    if (fd < 0) {
        set_parse(err, PF_ERR_PARSE, 0, std::string("cannot open pair file: ") + path);
        if (err) err->status = PF_ERR_PARSE;
        return PF_ERR_PARSE;
    }
    struct stat st {};
    if (fstat(fd, &st) == 0 && S_ISREG(st.st_mode) && st.st_size > 0) {
        // a regular file is mapped, not copied: the loader's threads fault its
        // pages in parallel while they scan it (a sized fread moved ~2 GB/s)
        const size_t len = static_cast<size_t>(st.st_size);
        void* map = mmap(nullptr, len, PROT_READ, MAP_PRIVATE, fd, 0);
        close(fd);
        if (map != MAP_FAILED) {
            madvise(map, len, MADV_SEQUENTIAL);
            tr.mark("file map");
            const int rc = pf_dataset_load_tsv(ctx, static_cast<const char*>(map), len, path, out, err);
            munmap(map, len);
            return rc;
        }
        FILE* f = std::fopen(path, "rb");  // mapping refused: read it
        if (!f) {
            set_parse(err, PF_ERR_PARSE, 0, std::string("cannot open pair file: ") + path);
            if (err) err->status = PF_ERR_PARSE;
            return PF_ERR_PARSE;
        }
        std::string buf(len, '\0');
        buf.resize(std::fread(buf.data(), 1, len, f));
        std::fclose(f);
        return pf_dataset_load_tsv(ctx, buf.data(), buf.size(), path, out, err);
    }
    // empty, a pipe or a special file: read it to the end
    std::string buf;
    char tmp[1 << 16];
    for (ssize_t r; (r = read(fd, tmp, sizeof(tmp))) > 0;) buf.append(tmp, static_cast<size_t>(r));
    close(fd);
    tr.mark("file read");
    return pf_dataset_load_tsv(ctx, buf.data(), buf.size(), path, out, err);
}

// generate_pairs restated (dataset.cpp:71-126): one std::mt19937_64 stream,
// draws reduced by modulo, so the bytes equal the reference generator's.
int pf_dataset_generate(uint64_t seed, size_t count, uint32_t length, uint32_t lo, uint32_t hi,
                        pf_dataset** out, pf_error* err) {
    if (err) std::memset(err, 0, sizeof(*err));
    if (!out) return PF_ERR_NULL_ARGUMENT;
    *out = nullptr;
    auto bad = [&](const char* msg) {
        if (err) {
            err->status = PF_ERR_INVALID_PARAMETERS;
            std::snprintf(err->message, sizeof(err->message), "%s", msg);
        }
        return PF_ERR_INVALID_PARAMETERS;
    };
    if (count == 0) return bad("pair count must be positive");
    if (length == 0) return bad("sequence length must be positive");
    if (lo > hi) return bad("inverted edit range");
    if (hi > length) return bad("cannot plant more edits than bases");
    auto* ds = new pf_dataset;
    ds->source = "gen(seed=" + std::to_string(seed) + ",count=" + std::to_string(count) +
                 ",len=" + std::to_string(length) + ",edits=" + std::to_string(lo) + ".." +
                 std::to_string(hi) + ")";
    if (!alloc_records(ds, count, length)) {
        delete ds;
        return PF_ERR_OUT_OF_MEMORY;
    }
    static const char kBases[4] = {'A', 'C', 'G', 'T'};
    std::mt19937_64 rng(seed);
    const uint64_t span = uint64_t(hi) - lo + 1;
    std::string pat;
    pat.reserve(length + hi + 1);
    for (size_t p = 0; p < count; ++p) {
        uint8_t* t = ds->text + p * length;
        for (uint32_t i = 0; i < length; ++i) t[i] = static_cast<uint8_t>(kBases[rng() % 4]);
        pat.assign(reinterpret_cast<const char*>(t), length);
        const uint64_t k = lo + rng() % span;
        for (uint64_t q = 0; q < k; ++q) {
            switch (rng() % 3) {
                case 0: {  // substitution: always a different base
                    const size_t pos = rng() % pat.size();
                    const int idx = static_cast<int>(std::strchr(kBases, pat[pos]) - kBases);
                    pat[pos] = kBases[(idx + 1 + rng() % 3) % 4];
                    break;
                }
                case 1: {  // insertion at [0, size]
                    const size_t pos = rng() % (pat.size() + 1);
                    pat.insert(pat.begin() + static_cast<std::ptrdiff_t>(pos), kBases[rng() % 4]);
                    break;
                }
                default: {  // deletion, skipped at size 1
                    if (pat.size() == 1) break;
                    const size_t pos = rng() % pat.size();
                    pat.erase(pat.begin() + static_cast<std::ptrdiff_t>(pos));
                    break;
                }
            }
        }
        if (pat.size() > length) pat.resize(length);
        while (pat.size() < length) pat.push_back(kBases[rng() % 4]);
        std::memcpy(ds->pattern + p * length, pat.data(), length);
    }
    *out = ds;
    return PF_OK;
}

int pf_dataset_from_records(const uint8_t* text, const uint8_t* pattern, size_t stride, size_t n,
                            uint32_t m, const char* source_name, pf_dataset** out) {
    if (!out || (n && (!text || !pattern)) || stride < m) return PF_ERR_NULL_ARGUMENT;
    auto* ds = new pf_dataset;
    ds->source = source_name ? source_name : "<records>";
    if (!alloc_records(ds, n, m)) {
        delete ds;
        return PF_ERR_OUT_OF_MEMORY;
    }
    for (size_t i = 0; i < n; ++i) {
        std::memcpy(ds->text + i * m, text + i * stride, m);
        std::memcpy(ds->pattern + i * m, pattern + i * stride, m);
    }
    *out = ds;
    return PF_OK;
}

size_t pf_dataset_size(const pf_dataset* ds) { return ds ? ds->n : 0; }
uint32_t pf_dataset_length(const pf_dataset* ds) { return ds ? ds->m : 0; }
const uint8_t* pf_dataset_text(const pf_dataset* ds) { return ds ? ds->text : nullptr; }
const uint8_t* pf_dataset_pattern(const pf_dataset* ds) { return ds ? ds->pattern : nullptr; }
const char* pf_dataset_source(const pf_dataset* ds) { return ds ? ds->source.c_str() : ""; }

// write_pairs (dataset.cpp:53-56): TEXT '\t' PATTERN per line, LF endings.
int pf_dataset_write_tsv(const pf_dataset* ds, const char* path) {
    if (!ds || !path) return PF_ERR_NULL_ARGUMENT;
    FILE* f = std::strcmp(path, "-") == 0 ? stdout : std::fopen(path, "wb");
    if (!f) return PF_ERR_PARSE;
    std::string line(2 * size_t(ds->m) + 2, '\0');
    for (size_t i = 0; i < ds->n; ++i) {
        std::memcpy(&line[0], ds->text + i * ds->m, ds->m);
        line[ds->m] = '\t';
        std::memcpy(&line[ds->m + 1], ds->pattern + i * ds->m, ds->m);
        line[2 * size_t(ds->m) + 1] = '\n';
        std::fwrite(line.data(), 1, line.size(), f);
    }
    if (f != stdout) std::fclose(f);
    else std::fflush(f);
    return PF_OK;
}

void pf_dataset_free(pf_dataset* ds) {
    if (!ds) return;
    if (ds->pinned) {
        cudaFreeHost(ds->text);
        cudaFreeHost(ds->pattern);
    } else {
        std::free(ds->text);
        std::free(ds->pattern);
    }
    delete ds;
}

}  // extern "C"
