// shouji-b200 — command-line caller of the B200 Shouji path.
//
// Mirrors the reference CLI's subcommands for this path (proj/src/cli.cpp):
//   filter  one accept bit per pair (+ "\t<estimate>" with --verbose), JSON
//           summary on stderr or --report (run_filter_cmd, cli.cpp:127-165)
//   eval    filter vs the exact banded alignment oracle (both on the GPU),
//           confusion counts (run_eval_cmd, cli.cpp:167-203)
//   gen     write a generated pair file (run_gen_cmd, cli.cpp:205-219)
//   bench   time filter passes over generated data, CSV (run_bench_cmd, :221-266)
// Inputs: --pairs FILE|- (TEXT\tPATTERN lines) or --seed/--count/--len/--edits;
// threshold --e or --e-percent (floored). Exit codes: 0 ok, 1 usage, 2 data.
// --threads is accepted for compatibility; output bytes never depend on it.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <initializer_list>
#include <iostream>
#include <iterator>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "shouji_b200.h"

namespace {

struct usage_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct data_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct options {
    std::string cmd;
    std::string pairs_file;
    uint64_t seed = 0;
    size_t count = 0;
    std::string len;  // a number, or a list for bench
    std::string edits;
    std::string e;    // a number, or a list for bench
    std::optional<double> e_percent;
    std::string algo = "shouji";
    unsigned width = 4;
    unsigned threads = 1;
    unsigned repeats = 3;
    std::string report;
    bool verbose = false;
};

uint32_t parse_u32(const std::string& s, const std::string& flag) {
    if (s.empty() || s.find_first_not_of("0123456789") != std::string::npos)
        throw usage_error(flag + " expects an unsigned integer, got '" + s + "'");
    return static_cast<uint32_t>(std::stoul(s));
}

std::pair<uint32_t, uint32_t> parse_edits(const std::string& spec) {
    const auto dots = spec.find("..");
    if (dots == std::string::npos) {
        const auto n = parse_u32(spec, "--edits");
        return {n, n};
    }
    const uint32_t lo = parse_u32(spec.substr(0, dots), "--edits");
    const uint32_t hi = parse_u32(spec.substr(dots + 2), "--edits");
    if (lo > hi) throw usage_error("--edits range is inverted: '" + spec + "'");
    return {lo, hi};
}

std::vector<uint32_t> parse_list(const std::string& spec, const std::string& flag) {
    std::vector<uint32_t> out;
    std::stringstream ss(spec);
    std::string item;
    while (std::getline(ss, item, ',')) out.push_back(parse_u32(item, flag));
    if (out.empty()) throw usage_error(flag + " expects a comma-separated list");
    return out;
}

std::string json_escape(const std::string& s) {
    std::string o;
    for (char c : s) {
        switch (c) {
            case '"': o += "\\\""; break;
            case '\\': o += "\\\\"; break;
            case '\n': o += "\\n"; break;
            case '\t': o += "\\t"; break;
            default:
                if (static_cast<unsigned char>(c) < 0x20) {
                    char b[8];
                    std::snprintf(b, sizeof(b), "\\u%04x", c);
                    o += b;
                } else {
                    o += c;
                }
        }
    }
    return o;
}

// nlohmann::ordered_json::dump(2) layout for a flat object.
struct json_obj {
    std::vector<std::pair<std::string, std::string>> kv;
    void str(const std::string& k, const std::string& v) { kv.emplace_back(k, "\"" + json_escape(v) + "\""); }
    void num(const std::string& k, uint64_t v) { kv.emplace_back(k, std::to_string(v)); }
    void dbl(const std::string& k, double v) {
        char b[64];
        std::snprintf(b, sizeof(b), "%.17g", v);
        std::string s = b;
        if (s.find_first_of(".eE") == std::string::npos) s += ".0";
        kv.emplace_back(k, s);
    }
    std::string dump() const {
        std::string o = "{\n";
        for (size_t i = 0; i < kv.size(); ++i)
            o += "  \"" + kv[i].first + "\": " + kv[i].second + (i + 1 < kv.size() ? ",\n" : "\n");
        return o + "}";
    }
};

// The GPU context, created on first use (so usage errors are reported before
// a missing device, as the reference resolves its options first).
struct ctx_holder {
    pf_ctx* ctx_ = nullptr;
    pf_ctx* get() {
        if (!ctx_ && pf_ctx_create(nullptr, 0, &ctx_) != PF_OK)
            throw data_error("no usable CUDA device");
        return ctx_;
    }
    ~ctx_holder() { pf_ctx_destroy(ctx_); }
};

struct dataset_holder {
    pf_dataset* ds = nullptr;
    ~dataset_holder() { pf_dataset_free(ds); }
};

void check(int st, const pf_error& err) {
    if (st == PF_OK) return;
    if (st == PF_ERR_INVALID_PARAMETERS) throw usage_error(err.message);
    throw data_error(err.message[0] ? err.message : pf_status_string(st));
}

std::optional<uint32_t> opt_e(const options& o) {
    if (o.e.empty()) return std::nullopt;
    return parse_u32(o.e, "--e");
}

uint32_t resolve_threshold(const options& o, size_t m) {
    const auto e = opt_e(o);
    if (e && o.e_percent) throw usage_error("--e and --e-percent are mutually exclusive");
    if (e) return *e;
    if (o.e_percent) return static_cast<uint32_t>(std::floor(double(m) * *o.e_percent / 100.0));
    throw usage_error("one of --e or --e-percent is required");
}

// --pairs FILE / - or the generator; the threshold needs m, and the generator's
// default edit range 0..2e needs the threshold (cli.cpp:96-110).
// The CUDA context (driver init, ~1 s) is created on a helper thread while the
// host cores load or generate the pairs; the filter calls that follow use it.
struct ctx_init {
    ctx_holder& ch;
    std::thread t;
    explicit ctx_init(ctx_holder& c) : ch(c), t([this] {
        try {
            ch.get();
        } catch (...) {  // reported by the next ch.get() on the main thread
        }
    }) {}
    ~ctx_init() { t.join(); }
};

uint32_t resolve_input(const options& o, ctx_holder& ch, dataset_holder& dh) {
    pf_error err{};
    if (!o.pairs_file.empty()) {
        int st;
        {
            ctx_init init(ch);
            if (o.pairs_file == "-") {
                std::string buf((std::istreambuf_iterator<char>(std::cin)),
                                std::istreambuf_iterator<char>());
                st = pf_dataset_load_tsv(nullptr, buf.data(), buf.size(), "<stdin>", &dh.ds, &err);
            } else {
                st = pf_dataset_load_tsv_file(nullptr, o.pairs_file.c_str(), &dh.ds, &err);
            }
        }
        check(st, err);
        return resolve_threshold(o, pf_dataset_length(dh.ds));
    }
    const uint32_t len = o.len.empty() ? 0 : parse_u32(o.len, "--len");
    if (o.count == 0 || len == 0) throw usage_error("provide --pairs FILE or both --count and --len");
    const uint32_t e = resolve_threshold(o, len);
    const uint32_t dhi = static_cast<uint32_t>(std::min<uint64_t>(2 * uint64_t(e), len));
    const auto ed = o.edits.empty() ? std::make_pair(0u, dhi) : parse_edits(o.edits);
    int st;
    {
        ctx_init init(ch);
        st = pf_dataset_generate(o.seed, o.count, len, ed.first, ed.second, &dh.ds, &err);
    }
    check(st, err);
    return e;
}

void emit_report(const std::string& text, const std::string& file) {
    if (file.empty()) {
        std::cerr << text << '\n';
        return;
    }
    std::ofstream f(file, std::ios::binary);
    if (!f) throw data_error("cannot open report file: " + file);
    f << text << '\n';
}

bool bit(const std::vector<uint32_t>& bm, size_t i) { return (bm[i / 32] >> (i % 32)) & 1u; }

// run_filter(algo, ...) over the whole dataset (evaluate.cpp:13-21): Shouji or MAGNET.
int run_algo(pf_ctx* ctx, const std::string& algo, const uint8_t* text, const uint8_t* pattern,
             size_t n, uint32_t m, uint32_t e, uint32_t width, uint32_t* acc, uint32_t* est,
             pf_error* err) {
    if (algo == "magnet")
        return pf_magnet_filter_batch(ctx, text, pattern, m, n, m, e, acc, est, nullptr, err);
    return pf_shouji_filter_batch(ctx, text, pattern, m, n, m, e, width, acc, est, nullptr, err);
}

void require_algo(const std::string& algo, std::initializer_list<const char*> allowed) {
    std::string names;
    for (const char* a : allowed) {
        if (algo == a) return;
        names += (names.empty() ? "" : ", ") + std::string(a);
    }
    throw usage_error("--algo " + algo + " is not one of: " + names);
}

int cmd_filter(const options& o) {
    require_algo(o.algo, {"shouji", "magnet", "oracle"});
    ctx_holder ch;
    dataset_holder dh;
    const uint32_t e = resolve_input(o, ch, dh);
    const size_t n = pf_dataset_size(dh.ds);
    const uint32_t m = pf_dataset_length(dh.ds);
    std::vector<uint32_t> acc((n + 31) / 32), est(n);
    std::vector<int32_t> dist;
    pf_error err{};
    if (o.algo == "oracle") {
        dist.resize(n);
        check(pf_banded_edit_distance_batch(ch.get(), pf_dataset_text(dh.ds), pf_dataset_pattern(dh.ds),
                                            m, n, m, e, dist.data(), &err),
              err);
    } else {
        check(run_algo(ch.get(), o.algo, pf_dataset_text(dh.ds), pf_dataset_pattern(dh.ds), n, m, e,
                       o.width, acc.data(), est.data(), &err),
              err);
    }
    std::string out;
    out.reserve(n * (o.verbose ? 6 : 2));
    size_t accepted = 0;
    for (size_t i = 0; i < n; ++i) {
        bool a;
        if (o.algo == "oracle") {
            a = dist[i] >= 0;
            out += a ? '1' : '0';
            if (o.verbose) out += '\t' + (a ? std::to_string(dist[i]) : std::string("-"));
        } else {
            a = bit(acc, i);
            out += a ? '1' : '0';
            if (o.verbose) out += '\t' + std::to_string(est[i]);
        }
        out += '\n';
        accepted += a;
    }
    std::fwrite(out.data(), 1, out.size(), stdout);
    std::fflush(stdout);
    json_obj j;
    j.str("command", "filter");
    j.str("algo", o.algo);
    j.num("width", o.width);
    j.num("m", m);
    j.str("source", pf_dataset_source(dh.ds));
    j.num("e", e);
    j.num("total", n);
    j.num("accepted", accepted);
    j.num("rejected", n - accepted);
    emit_report(j.dump(), o.report);
    return 0;
}

int cmd_eval(const options& o) {
    require_algo(o.algo, {"shouji", "magnet"});
    ctx_holder ch;
    dataset_holder dh;
    const uint32_t e = resolve_input(o, ch, dh);
    const size_t n = pf_dataset_size(dh.ds);
    const uint32_t m = pf_dataset_length(dh.ds);
    std::vector<uint32_t> acc((n + 31) / 32), est(n);
    std::vector<int32_t> dist(n);
    pf_error err{};
    check(run_algo(ch.get(), o.algo, pf_dataset_text(dh.ds), pf_dataset_pattern(dh.ds), n, m, e,
                   o.width, acc.data(), est.data(), &err),
          err);
    check(pf_banded_edit_distance_batch(ch.get(), pf_dataset_text(dh.ds), pf_dataset_pattern(dh.ds), m,
                                        n, m, e, dist.data(), &err),
          err);
    size_t oa = 0, orj = 0, fa = 0, fr = 0, fals_a = 0, fals_r = 0;
    std::string out;
    for (size_t i = 0; i < n; ++i) {
        const bool a = bit(acc, i), within = dist[i] >= 0;
        (within ? oa : orj)++;
        (a ? fa : fr)++;
        if (a && !within) ++fals_a;
        if (!a && within) ++fals_r;
        out += a ? '1' : '0';
        if (o.verbose) {
            out += '\t' + std::to_string(est[i]) + '\t';
            out += within ? std::to_string(dist[i]) : std::string("-");
        }
        out += '\n';
    }
    std::fwrite(out.data(), 1, out.size(), stdout);
    std::fflush(stdout);
    // evaluate.cpp:63-78
    json_obj j;
    j.str("command", "eval");
    j.str("algo", o.algo);
    j.num("width", o.width);
    j.num("m", m);
    j.str("source", pf_dataset_source(dh.ds));
    j.num("e", e);
    j.num("total", n);
    j.num("oracle_accepted", oa);
    j.num("oracle_rejected", orj);
    j.num("filter_accepted", fa);
    j.num("filter_rejected", fr);
    j.num("falsely_accepted", fals_a);
    j.num("falsely_rejected", fals_r);
    j.dbl("fa_rate", orj == 0 ? 0.0 : double(fals_a) / double(orj));
    j.dbl("fr_rate", oa == 0 ? 0.0 : double(fals_r) / double(oa));
    emit_report(j.dump(), o.report);
    return 0;
}

int cmd_gen(const options& o) {
    const uint32_t len = o.len.empty() ? 0 : parse_u32(o.len, "--len");
    if (o.count == 0 || len == 0) throw usage_error("gen requires --count and --len");
    if (o.edits.empty()) throw usage_error("gen requires --edits");
    const auto ed = parse_edits(o.edits);
    dataset_holder dh;
    pf_error err{};
    check(pf_dataset_generate(o.seed, o.count, len, ed.first, ed.second, &dh.ds, &err), err);
    const std::string path = o.pairs_file.empty() ? "-" : o.pairs_file;
    if (pf_dataset_write_tsv(dh.ds, path.c_str()) != PF_OK)
        throw data_error("cannot open output file: " + path);
    return 0;
}

// run_bench (bench.cpp:11-42) on the GPU path: 1 warm-up + repeats passes of
// the batch call over pre-generated pairs, median reported.
int cmd_bench(const options& o) {
    require_algo(o.algo, {"shouji", "magnet"});
    const auto lens = parse_list(o.len, "--len");
    const auto es = parse_list(o.e, "--e");
    const size_t count = o.count ? o.count : 10000;
    ctx_holder ch;
    std::ostringstream csv;
    csv << "algo,m,e,count,repeats,median_seconds,pairs_per_second,bases_per_second\n";
    std::vector<std::vector<double>> med(es.size(), std::vector<double>(lens.size(), 0.0));
    for (size_t li = 0; li < lens.size(); ++li) {
        for (size_t ei = 0; ei < es.size(); ++ei) {
            const auto ed = o.edits.empty()
                                ? std::make_pair(0u, static_cast<uint32_t>(std::min<uint64_t>(
                                                         2 * uint64_t(es[ei]), lens[li])))
                                : parse_edits(o.edits);
            dataset_holder dh;
            pf_error err{};
            check(pf_dataset_generate(o.seed, count, lens[li], ed.first, ed.second, &dh.ds, &err), err);
            std::vector<uint32_t> acc((count + 31) / 32);
            std::vector<double> secs;
            for (unsigned r = 0; r <= o.repeats; ++r) {
                const auto t0 = std::chrono::steady_clock::now();
                check(run_algo(ch.get(), o.algo, pf_dataset_text(dh.ds), pf_dataset_pattern(dh.ds),
                               count, lens[li], es[ei], o.width, acc.data(), nullptr, &err),
                      err);
                const double s =
                    std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                if (r > 0) secs.push_back(s);
            }
            std::sort(secs.begin(), secs.end());
            const double m = secs[secs.size() / 2];
            med[ei][li] = m;
            csv << o.algo << ',' << lens[li] << ',' << es[ei] << ',' << count << ',' << o.repeats << ','
                << m << ',' << (m > 0 ? count / m : 0.0) << ',' << (m > 0 ? count * double(lens[li]) / m : 0.0)
                << '\n';
        }
    }
    if (lens.size() > 1) {
        csv << "\nalgo,e,m_from,m_to,time_ratio\n";
        for (size_t ei = 0; ei < es.size(); ++ei)
            for (size_t li = 0; li + 1 < lens.size(); ++li)
                csv << o.algo << ',' << es[ei] << ',' << lens[li] << ',' << lens[li + 1] << ','
                    << med[ei][li + 1] / med[ei][li] << '\n';
    }
    if (o.report.empty()) {
        std::cout << csv.str();
    } else {
        std::ofstream f(o.report, std::ios::binary);
        if (!f) throw data_error("cannot open report file: " + o.report);
        f << csv.str();
    }
    return 0;
}

options parse_args(int argc, char** argv) {
    if (argc < 2) throw usage_error("a subcommand is required: filter, eval, gen, bench");
    options o;
    o.cmd = argv[1];
    if (o.cmd != "filter" && o.cmd != "eval" && o.cmd != "gen" && o.cmd != "bench")
        throw usage_error("unknown subcommand '" + o.cmd + "'");
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= argc) throw usage_error(a + " requires an argument");
            return argv[++i];
        };
        if (a == "--pairs") o.pairs_file = val();
        else if (a == "--seed") o.seed = std::stoull(val());
        else if (a == "--count") o.count = parse_u32(val(), "--count");
        else if (a == "--len") o.len = val();
        else if (a == "--edits") o.edits = val();
        else if (a == "--e") o.e = val();
        else if (a == "--e-percent") o.e_percent = std::stod(val());
        else if (a == "--algo") o.algo = val();
        else if (a == "--width") {
            o.width = parse_u32(val(), "--width");
            if (o.width < 3 || o.width > 8) throw usage_error("--width: value not in range 3 to 8");
        } else if (a == "--threads") {
            o.threads = parse_u32(val(), "--threads");
            if (o.threads < 1 || o.threads > 4096) throw usage_error("--threads: value not in range 1 to 4096");
        } else if (a == "--repeats") o.repeats = std::max(1u, parse_u32(val(), "--repeats"));
        else if (a == "--report") o.report = val();
        else if (a == "--verbose") o.verbose = true;
        else throw usage_error("unknown option " + a);
    }
    if (o.cmd == "bench" && (o.len.empty() || o.e.empty()))
        throw usage_error("bench requires --len and --e");
    return o;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        const options o = parse_args(argc, argv);
        if (o.cmd == "filter") return cmd_filter(o);
        if (o.cmd == "eval") return cmd_eval(o);
        if (o.cmd == "gen") return cmd_gen(o);
        return cmd_bench(o);
    } catch (const usage_error& e) {
        std::cerr << "usage error: " << e.what() << '\n';
        return 1;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 2;
    }
}
