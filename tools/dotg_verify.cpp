// dotg_verify.cpp - run a reference JSONL corpus through the B200 kernels (§8(f) item 3).
//
// Reads the reference's corpus format (src/testgen.cpp:195-255: one JSON object per line,
// fields op, bits, category, a, b, expected as minimal lowercase hex, flag 0/1 for
// add/sub) and verifies every case on the device: cases are grouped by (op, bits) and
// each group is ONE batched call (dotg_add_batch_host / dotg_sub_batch_host /
// dotg_mul_batch_host), instead of the reference's per-case loop (bench.cpp:147-170).
// Output and exit codes follow `dotarith verify` (tools/dotarith_cli.cpp:57-82):
//   "kernel b200 (w=8, sm_100a): N cases, K mismatches", the AddSubStats line
//   "chunks C, phase4 triggers T (rate R)" when the corpus has add/sub cases, up to 10
//   "mismatch at case i" lines, exit 0 = all match, 1 = mismatch, 2 = usage / input error.
//
// `dotg-verify bench <corpus.jsonl> [--width w] [--reps R] [--csv path]` is the device
// counterpart of `dotarith bench` (dotarith_cli.cpp:103-139, bench.cpp:176-245) over a
// corpus file: per (op, bits) group the verification gate first (no row for a group that
// mismatches, exit 1), then R timed repetitions of the group's batched call with the
// operands resident in device memory (CUDA events; ns per case, mean and Student-t 95%
// half-width like bench.cpp:216-225), the same call through the host-buffer entry point
// (PCIe copies included), and the group's Phase-4 rate.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "dotg.h"

namespace {

using Limbs = std::vector<uint64_t>;

struct Case {
    std::string op;
    unsigned bits = 0;
    Limbs a, b, expected;
    unsigned flag = 0;
};

// Minimal parser for the flat JSON objects the reference writes (string and unsigned
// integer values only).
std::map<std::string, std::string> parse_object(const std::string& s) {
    std::map<std::string, std::string> kv;
    size_t i = 0;
    auto ws = [&] {
        while (i < s.size() && (s[i] == ' ' || s[i] == '\t' || s[i] == '\r')) ++i;
    };
    auto str = [&]() -> std::string {
        if (i >= s.size() || s[i] != '"') throw std::invalid_argument("expected a string");
        std::string out;
        for (++i; i < s.size() && s[i] != '"'; ++i) {
            if (s[i] == '\\') throw std::invalid_argument("escapes are not used by the corpus format");
            out.push_back(s[i]);
        }
        if (i >= s.size()) throw std::invalid_argument("unterminated string");
        ++i;
        return out;
    };
    ws();
    if (i >= s.size() || s[i++] != '{') throw std::invalid_argument("expected '{'");
    ws();
    if (i < s.size() && s[i] == '}') return kv;
    for (;;) {
        ws();
        const std::string key = str();
        ws();
        if (i >= s.size() || s[i++] != ':') throw std::invalid_argument("expected ':'");
        ws();
        std::string val;
        if (i < s.size() && s[i] == '"') {
            val = str();
        } else {
            const size_t j = i;
            while (i < s.size() && s[i] >= '0' && s[i] <= '9') ++i;
            if (i == j) throw std::invalid_argument("expected a string or an unsigned integer");
            val = s.substr(j, i - j);
        }
        kv[key] = val;
        ws();
        if (i < s.size() && s[i] == ',') {
            ++i;
            continue;
        }
        if (i < s.size() && s[i] == '}') break;
        throw std::invalid_argument("expected ',' or '}'");
    }
    return kv;
}

// from_hex (src/limbs.cpp:55-98): optional 0x, '_' separators, padded to min_limbs.
Limbs from_hex(const std::string& text, size_t min_limbs) {
    std::string s = text;
    if (s.size() >= 2 && s[0] == '0' && (s[1] == 'x' || s[1] == 'X')) s = s.substr(2);
    std::vector<uint8_t> nib;
    bool seen = false;
    for (char c : s) {
        if (c == '_') {
            if (!seen) throw std::invalid_argument("hex numeral: leading '_' separator");
            continue;
        }
        int d = c >= '0' && c <= '9' ? c - '0' : c >= 'a' && c <= 'f' ? c - 'a' + 10 : c >= 'A' && c <= 'F' ? c - 'A' + 10 : -1;
        if (d < 0) throw std::invalid_argument(std::string("hex numeral: invalid character '") + c + "'");
        seen = true;
        if (!nib.empty() || d != 0) nib.push_back(uint8_t(d));
    }
    if (!seen) throw std::invalid_argument("hex numeral: no digits");
    Limbs w;
    size_t pos = nib.size();
    while (pos > 0) {
        const size_t take = pos < 16 ? pos : 16;
        uint64_t v = 0;
        for (size_t k = pos - take; k < pos; ++k) v = (v << 4) | nib[k];
        w.push_back(v);
        pos -= take;
    }
    if (w.size() < min_limbs) w.resize(min_limbs, 0);
    return w;
}

std::vector<Case> read_corpus(const std::string& path) {  // read_vectors, testgen.cpp:211-255
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open for reading: " + path);
    std::vector<Case> out;
    std::string line;
    size_t lineno = 0;
    while (std::getline(in, line)) {
        ++lineno;
        if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
        try {
            auto kv = parse_object(line);
            Case c;
            c.op = kv.at("op");
            if (c.op != "add" && c.op != "sub" && c.op != "mul") throw std::invalid_argument("unknown op name: " + c.op);
            c.bits = unsigned(std::stoul(kv.at("bits")));
            if (c.bits == 0 || c.bits % 64) throw std::invalid_argument("bits must be a positive multiple of 64");
            (void)kv.at("category");
            const size_t m = c.bits / 64;
            c.a = from_hex(kv.at("a"), m);
            c.b = from_hex(kv.at("b"), m);
            if (c.a.size() > m || c.b.size() > m) throw std::invalid_argument("operand wider than the declared bits");
            c.expected = from_hex(kv.at("expected"), c.op == "mul" ? 0 : m);
            if (c.op != "mul") {
                c.flag = unsigned(std::stoul(kv.at("flag")));
                if (c.flag > 1) throw std::invalid_argument("flag must be 0 or 1");
                if (c.expected.size() != m) throw std::invalid_argument("expected value wider than the operands");
            }
            out.push_back(std::move(c));
        } catch (const std::exception& e) {
            throw std::runtime_error(path + ": parse error at line " + std::to_string(lineno) + ": " + e.what());
        }
    }
    return out;
}

using Groups = std::map<std::pair<std::string, unsigned>, std::vector<size_t>>;

Groups group_cases(const std::vector<Case>& corpus) {  // one batched device call per (op, bits)
    Groups groups;
    for (size_t i = 0; i < corpus.size(); ++i) groups[{corpus[i].op, corpus[i].bits}].push_back(i);
    return groups;
}

// Row-major operands of one group.
void gather(const std::vector<Case>& corpus, const std::vector<size_t>& ids, size_t m, Limbs& A, Limbs& B) {
    const size_t n = ids.size();
    A.assign(n * m, 0);
    B.assign(n * m, 0);
    for (size_t k = 0; k < n; ++k)
        for (size_t j = 0; j < m; ++j) {
            A[k * m + j] = corpus[ids[k]].a[j];
            B[k * m + j] = corpus[ids[k]].b[j];
        }
}

int host_call(const std::string& op, Limbs& out, const Limbs& A, const Limbs& B, std::vector<uint32_t>& fl,
              size_t m, size_t n) {
    return op == "mul"   ? dotg_mul_batch_host(out.data(), A.data(), B.data(), m, n)
           : op == "add" ? dotg_add_batch_host(out.data(), A.data(), B.data(), fl.data(), m, n)
                         : dotg_sub_batch_host(out.data(), A.data(), B.data(), fl.data(), m, n);
}

// Verification gate of one group: ids of the mismatching cases.
std::vector<size_t> check_group(const std::vector<Case>& corpus, const std::string& op, size_t m,
                                const std::vector<size_t>& ids) {
    const size_t n = ids.size();
    const bool mul = op == "mul";
    Limbs A, B;
    gather(corpus, ids, m, A, B);
    Limbs out(n * m * (mul ? 2 : 1));
    std::vector<uint32_t> fl(n);
    if (host_call(op, out, A, B, fl, m, n) != DOTG_OK)
        throw std::runtime_error(std::string("device call failed: ") + dotg_last_error());
    std::vector<size_t> bad;
    for (size_t k = 0; k < n; ++k) {
        const Case& c = corpus[ids[k]];
        bool ok;
        if (mul) {
            size_t len = 2 * m;
            while (len > 0 && out[k * 2 * m + len - 1] == 0) --len;  // products compare trimmed
            ok = c.expected == Limbs(out.begin() + k * 2 * m, out.begin() + k * 2 * m + len);
        } else {
            ok = c.expected == Limbs(out.begin() + k * m, out.begin() + (k + 1) * m) && c.flag == fl[k];
        }
        if (!ok) bad.push_back(ids[k]);
    }
    return bad;
}

// AddSubStats of the add/sub cases of `ids` (bench.cpp:160-161 collects them for the vector
// add/sub kernels): chunks of lane_count(width) limbs and how many would have taken the
// rare Phase 4, derived on the device per case (dotg_words_host_stats).
void group_stats(const std::vector<Case>& corpus, const std::vector<size_t>& ids, int width, uint64_t& chunks,
                 uint64_t& fires) {
    for (const size_t i : ids) {
        const Case& c = corpus[i];
        if (c.op == "mul") continue;
        Limbs o(c.a.size());
        uint32_t carry = 0;
        if (dotg_words_host_stats(c.op == "sub", o.data(), c.a.data(), c.b.data(), c.a.size(), width, &carry,
                                  &chunks, &fires) != DOTG_OK)
            throw std::runtime_error(std::string("stats call failed: ") + dotg_last_error());
    }
}

double t95(size_t dof) {  // two-sided Student t, 95% (bench.cpp:216-225 uses the same table idea)
    static const double tab[] = {0, 12.706, 4.303, 3.182, 2.776, 2.571, 2.447, 2.365, 2.306, 2.262, 2.228,
                                 2.201, 2.179, 2.160, 2.145, 2.131, 2.120, 2.110, 2.101, 2.093, 2.086,
                                 2.080, 2.074, 2.069, 2.064, 2.060, 2.056, 2.052, 2.048, 2.045, 2.042};
    return dof < sizeof(tab) / sizeof(tab[0]) ? tab[dof] : 1.960;
}

void mean_ci(const std::vector<double>& v, double& mean, double& ci) {
    mean = 0;
    for (double x : v) mean += x;
    mean /= double(v.size());
    ci = 0;
    if (v.size() > 1) {
        double var = 0;
        for (double x : v) var += (x - mean) * (x - mean);
        var /= double(v.size() - 1);
        ci = t95(v.size() - 1) * std::sqrt(var / double(v.size()));
    }
}

#define CUDA_OR_THROW(x)                                                                            \
    do {                                                                                            \
        const cudaError_t e_ = (x);                                                                 \
        if (e_ != cudaSuccess) throw std::runtime_error(std::string(#x ": ") + cudaGetErrorString(e_)); \
    } while (0)

int cmd_bench(const std::vector<Case>& corpus, int width, unsigned reps, const std::string& csv_path) {
    const Groups groups = group_cases(corpus);
    bool mismatched = false;
    std::string csv = "op,bits,w,kernel,cases,ns_per_op_device,ci95_device,ns_per_op_host,ci95_host,phase4,timer\n";
    const std::string wname = width == 0 ? "scalar" : "w" + std::to_string(width);
    std::printf("%-4s %6s %7s %-12s %7s %14s %10s %14s %10s %8s %s\n", "op", "bits", "w", "kernel", "cases",
                "ns/op(dev)", "ci95", "ns/op(host)", "ci95", "phase4", "timer");
    for (const auto& [key, ids] : groups) {
        const std::string& op = key.first;
        const size_t m = key.second / 64, n = ids.size();
        const std::vector<size_t> bad = check_group(corpus, op, m, ids);
        if (!bad.empty()) {  // no row for a group that fails verification (bench.cpp:201-204)
            std::fprintf(stderr, "bench: b200 failed verification at %u bits (%s): %zu mismatches\n", key.second,
                         op.c_str(), bad.size());
            mismatched = true;
            continue;
        }
        const bool mul = op == "mul";
        Limbs A, B;
        gather(corpus, ids, m, A, B);
        const size_t in_bytes = n * m * 8, out_bytes = in_bytes * (mul ? 2 : 1);
        uint64_t *da = nullptr, *db = nullptr, *dout = nullptr;
        uint32_t* dfl = nullptr;
        cudaStream_t st = nullptr;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        CUDA_OR_THROW(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        CUDA_OR_THROW(cudaEventCreate(&e0));
        CUDA_OR_THROW(cudaEventCreate(&e1));
        CUDA_OR_THROW(cudaMalloc(&da, in_bytes));
        CUDA_OR_THROW(cudaMalloc(&db, in_bytes));
        CUDA_OR_THROW(cudaMalloc(&dout, out_bytes));
        CUDA_OR_THROW(cudaMalloc(&dfl, n * 4));
        CUDA_OR_THROW(cudaMemcpy(da, A.data(), in_bytes, cudaMemcpyHostToDevice));
        CUDA_OR_THROW(cudaMemcpy(db, B.data(), in_bytes, cudaMemcpyHostToDevice));
        auto dev_call = [&] {
            const int rc = mul ? dotg_mul_batch(dout, da, db, m, n, DOTG_ROW_MAJOR, st)
                           : op == "add" ? dotg_add_batch(dout, da, db, dfl, m, n, DOTG_ROW_MAJOR, st)
                                         : dotg_sub_batch(dout, da, db, dfl, m, n, DOTG_ROW_MAJOR, st);
            if (rc != DOTG_OK) throw std::runtime_error(std::string("device call failed: ") + dotg_last_error());
        };
        // device-resident: each sample is a CUDA-event-timed launch sequence of `inner` calls
        const unsigned inner = 10;
        std::vector<double> dev(reps), host(reps);
        for (int w = 0; w < 3; ++w) dev_call();
        for (unsigned r = 0; r < reps; ++r) {
            CUDA_OR_THROW(cudaEventRecord(e0, st));
            for (unsigned k = 0; k < inner; ++k) dev_call();
            CUDA_OR_THROW(cudaEventRecord(e1, st));
            CUDA_OR_THROW(cudaEventSynchronize(e1));
            float ms = 0;
            CUDA_OR_THROW(cudaEventElapsedTime(&ms, e0, e1));
            dev[r] = double(ms) * 1e6 / double(inner) / double(n);
        }
        // host buffers: the same call through the host entry point, copies included
        Limbs out(out_bytes / 8);
        std::vector<uint32_t> fl(n);
        for (unsigned r = 0; r < reps; ++r) {
            CUDA_OR_THROW(cudaEventRecord(e0, nullptr));
            if (host_call(op, out, A, B, fl, m, n) != DOTG_OK)
                throw std::runtime_error(std::string("device call failed: ") + dotg_last_error());
            CUDA_OR_THROW(cudaEventRecord(e1, nullptr));
            CUDA_OR_THROW(cudaEventSynchronize(e1));
            float ms = 0;
            CUDA_OR_THROW(cudaEventElapsedTime(&ms, e0, e1));
            host[r] = double(ms) * 1e6 / double(n);
        }
        cudaFree(da);
        cudaFree(db);
        cudaFree(dout);
        cudaFree(dfl);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaStreamDestroy(st);
        uint64_t chunks = 0, fires = 0;
        group_stats(corpus, ids, width, chunks, fires);
        const double p4 = chunks ? double(fires) / double(chunks) : 0.0;
        double dm, dc, hm, hc;
        mean_ci(dev, dm, dc);
        mean_ci(host, hm, hc);
        std::printf("%-4s %6u %7s %-12s %7zu %14.3f %10.3f %14.3f %10.3f %8.4f %s\n", op.c_str(), key.second,
                    wname.c_str(), "b200", n, dm, dc, hm, hc, p4, "cuda-events");
        char line[512];
        std::snprintf(line, sizeof line, "%s,%u,%s,b200,%zu,%.4f,%.4f,%.4f,%.4f,%.6f,cuda-events\n", op.c_str(),
                      key.second, wname.c_str(), n, dm, dc, hm, hc, p4);
        csv += line;
    }
    std::printf("timer: cuda-events (device clock; ns per case, batched per (op, bits) group)\n");
    if (!csv_path.empty()) {
        std::ofstream f(csv_path, std::ios::binary | std::ios::trunc);
        if (!f || !(f << csv)) throw std::runtime_error("cannot write " + csv_path);
    }
    return mismatched ? 1 : 0;
}

}  // namespace

// `dotg-verify stats [--k-max K] [--samples N] [--seed S]`: dotarith stats
// (dotarith_cli.cpp:141-156, bench.cpp:261-289) with the census and the Monte-Carlo pass
// counted on the device. Exit 0 when every row matches its closed form and the carry
// frequency is within 0.5 +/- 0.001, else 1.
int cmd_stats(int argc, char** argv) {
    unsigned k_max = 12;
    uint64_t samples = 10000000, seed = 1;
    for (int i = 2; i < argc; i += 2) {
        const std::string opt = argv[i];
        if (i + 1 >= argc) {
            std::fprintf(stderr, "option %s needs a value\n", opt.c_str());
            return 2;
        }
        const char* v = argv[i + 1];
        if (opt == "--k-max") k_max = unsigned(std::strtoul(v, nullptr, 10));
        else if (opt == "--samples") samples = std::strtoull(v, nullptr, 10);
        else if (opt == "--seed") seed = std::strtoull(v, nullptr, 10);
        else {
            std::fprintf(stderr, "unknown option: %s\n", opt.c_str());
            return 2;
        }
    }
    if (k_max < 1 || k_max > 16) {
        std::fprintf(stderr, "stats: k_max must be in 1..16\n");
        return 2;
    }
    bool ok = true;
    std::printf("%3s %22s %22s %s\n", "k", "max-sum (got/closed)", "carry (got/closed)", "match");
    for (unsigned k = 1; k <= k_max; ++k) {
        uint64_t c[2] = {0, 0};
        if (dotg_carry_census(k, c) != DOTG_OK) {
            std::fprintf(stderr, "error: %s\n", dotg_last_error());
            return 2;
        }
        const uint64_t cm = uint64_t(1) << k, cc = (uint64_t(1) << (k - 1)) * ((uint64_t(1) << k) - 1);
        const bool match = c[0] == cm && c[1] == cc;
        ok = ok && match;
        std::printf("%3u %10llu /%10llu %10llu /%10llu %s\n", k, static_cast<unsigned long long>(c[0]),
                    static_cast<unsigned long long>(cm), static_cast<unsigned long long>(c[1]),
                    static_cast<unsigned long long>(cc), match ? "yes" : "NO");
    }
    uint64_t carries = 0;
    if (dotg_mc_carry(samples, seed, &carries) != DOTG_OK) {
        std::fprintf(stderr, "error: %s\n", dotg_last_error());
        return 2;
    }
    const double f = samples ? double(carries) / double(samples) : 0.0;
    const bool within = samples && std::fabs(f - 0.5) <= 0.001;
    std::printf("monte-carlo: %llu samples, carry frequency %.6f (0.5 +/- 0.001: %s)\n",
                static_cast<unsigned long long>(samples), f, within ? "yes" : "NO");
    return ok && within ? 0 : 1;
}

int main(int argc, char** argv) {
    const std::string cmd = argc >= 2 ? argv[1] : "";
    if (cmd == "stats") return cmd_stats(argc, argv);
    if (argc < 3 || (cmd != "verify" && cmd != "bench")) {
        std::fprintf(stderr,
                     "usage: dotg-verify verify <corpus.jsonl> [--width scalar|2|4|8]\n"
                     "       dotg-verify bench <corpus.jsonl> [--width scalar|2|4|8] [--reps R] [--csv path]\n"
                     "       dotg-verify stats [--k-max K] [--samples N] [--seed S]\n");
        return 2;
    }
    int width = 8;
    unsigned reps = 10;
    std::string csv_path;
    for (int i = 3; i < argc; i += 2) {
        const std::string opt = argv[i];
        if (i + 1 >= argc) {
            std::fprintf(stderr, "option %s needs a value\n", opt.c_str());
            return 2;
        }
        const std::string val = argv[i + 1];
        if (opt == "--width") {
            width = val == "scalar" ? 0 : std::atoi(val.c_str());
        } else if (opt == "--reps" && cmd == "bench") {
            reps = unsigned(std::strtoul(val.c_str(), nullptr, 10));
            if (reps == 0) {
                std::fprintf(stderr, "bench needs at least one repetition\n");
                return 2;
            }
        } else if (opt == "--csv" && cmd == "bench") {
            csv_path = val;
        } else {
            std::fprintf(stderr, "unknown option: %s\n", opt.c_str());
            return 2;
        }
    }
    if (dotg_validate_width(width) != DOTG_OK) {
        std::fprintf(stderr, "unknown width: expected one of 2, 4, 8, scalar\n");
        return 2;
    }
    std::vector<Case> corpus;
    try {
        corpus = read_corpus(argv[2]);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    }
    if (cmd == "bench") {
        try {
            return cmd_bench(corpus, width, reps, csv_path);
        } catch (const std::exception& e) {
            std::fprintf(stderr, "error: %s\n", e.what());
            return 2;
        }
    }
    std::vector<size_t> bad;
    uint64_t chunks = 0, fires = 0;
    try {
        for (const auto& [key, ids] : group_cases(corpus)) {
            const std::vector<size_t> b = check_group(corpus, key.first, key.second / 64, ids);
            bad.insert(bad.end(), b.begin(), b.end());
        }
        std::vector<size_t> all(corpus.size());
        for (size_t i = 0; i < all.size(); ++i) all[i] = i;
        group_stats(corpus, all, width, chunks, fires);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    }
    std::sort(bad.begin(), bad.end());
    std::printf("kernel b200 (w=%s, sm_100a): %zu cases, %zu mismatches\n",
                width == 0 ? "scalar" : std::to_string(width).c_str(), corpus.size(), bad.size());
    if (chunks > 0)
        std::printf("chunks %llu, phase4 triggers %llu (rate %.6f)\n", static_cast<unsigned long long>(chunks),
                    static_cast<unsigned long long>(fires), double(fires) / double(chunks));
    for (size_t s = 0; s < bad.size(); ++s) {
        if (s == 10) {
            std::printf("  ... %zu more\n", bad.size() - 10);
            break;
        }
        std::printf("  mismatch at case %zu\n", bad[s]);
    }
    return bad.empty() ? 0 : 1;
}
