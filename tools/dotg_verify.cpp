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
#include <algorithm>
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

}  // namespace

int main(int argc, char** argv) {
    if (argc < 3 || std::string(argv[1]) != "verify") {
        std::fprintf(stderr, "usage: dotg-verify verify <corpus.jsonl> [--width scalar|2|4|8]\n");
        return 2;
    }
    int width = 8;
    for (int i = 3; i + 1 < argc; i += 2) {
        if (std::string(argv[i]) == "--width") {
            const std::string w = argv[i + 1];
            width = w == "scalar" ? 0 : std::atoi(w.c_str());
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
    // group case ids by (op, bits): one batched device call per group
    std::map<std::pair<std::string, unsigned>, std::vector<size_t>> groups;
    for (size_t i = 0; i < corpus.size(); ++i) groups[{corpus[i].op, corpus[i].bits}].push_back(i);
    std::vector<size_t> bad;
    for (const auto& [key, ids] : groups) {
        const size_t m = key.second / 64, n = ids.size();
        Limbs A(n * m), B(n * m);
        for (size_t k = 0; k < n; ++k)
            for (size_t j = 0; j < m; ++j) {
                A[k * m + j] = corpus[ids[k]].a[j];
                B[k * m + j] = corpus[ids[k]].b[j];
            }
        const bool mul = key.first == "mul";
        Limbs out(n * m * (mul ? 2 : 1));
        std::vector<uint32_t> fl(n);
        int rc = mul ? dotg_mul_batch_host(out.data(), A.data(), B.data(), m, n)
                     : key.first == "add" ? dotg_add_batch_host(out.data(), A.data(), B.data(), fl.data(), m, n)
                                          : dotg_sub_batch_host(out.data(), A.data(), B.data(), fl.data(), m, n);
        if (rc != DOTG_OK) {
            std::fprintf(stderr, "error: device call failed: %s\n", dotg_last_error());
            return 2;
        }
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
    }
    // AddSubStats of the add/sub cases (bench.cpp:160-161 collects them for the vector
    // add/sub kernels): chunks of lane_count(width) limbs and how many would have taken
    // the rare Phase 4, derived on the device per case (dotg_words_host_stats).
    uint64_t chunks = 0, fires = 0;
    for (const Case& c : corpus) {
        if (c.op == "mul") continue;
        Limbs o(c.a.size());
        uint32_t carry = 0;
        if (dotg_words_host_stats(c.op == "sub", o.data(), c.a.data(), c.b.data(), c.a.size(), width, &carry,
                                  &chunks, &fires) != DOTG_OK) {
            std::fprintf(stderr, "error: stats call failed: %s\n", dotg_last_error());
            return 2;
        }
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
