// test_shim.cpp - C++ drop-in parity test: the reference's own test cases
// (proj/tests/test_addsub.cpp, test_mul.cpp, test_oracle.cpp), restated against
// dot_b200:: (include/dot_b200.hpp -> libdotg.so on the B200) with the same seeded
// std::mt19937_64 draws, checked against the oracle restatement (oracle/dot_oracle.c).
// Dependency-free: a minimal CHECK runner instead of doctest (absent in this image).
#include <cstdio>
#include <functional>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "dot_b200.hpp"

extern "C" {
#include "../../oracle/dot_oracle.h"
}

using namespace dot_b200;

namespace {
int g_checks = 0, g_fail = 0;
const char* g_case = "";
#define CHECK(c)                                                                      \
    do {                                                                              \
        ++g_checks;                                                                   \
        if (!(c)) {                                                                   \
            ++g_fail;                                                                 \
            std::fprintf(stderr, "FAIL [%s] %s:%d: %s\n", g_case, __FILE__, __LINE__, #c); \
        }                                                                             \
    } while (0)
#define CHECK_THROWS_AS(expr, T)          \
    do {                                  \
        bool thrown_ = false;             \
        try {                             \
            (void)(expr);                 \
        } catch (const T&) {              \
            thrown_ = true;               \
        } catch (...) {                   \
        }                                 \
        CHECK(thrown_ && #expr);          \
    } while (0)
#define CHECK_NOTHROW(expr)               \
    do {                                  \
        bool ok_ = true;                  \
        try {                             \
            (void)(expr);                 \
        } catch (...) {                   \
            ok_ = false;                  \
        }                                 \
        CHECK(ok_ && #expr);              \
    } while (0)

constexpr limb_t kMax = ~limb_t(0);

Limbs uniform_limbs(std::mt19937_64& rng, std::size_t m) {
    Limbs a(m);
    for (auto& x : a) x = rng();
    return a;
}
Limbs spiky_limbs(std::mt19937_64& rng, std::size_t m) {  // test_addsub.cpp:28-40
    Limbs a(m);
    for (auto& x : a) {
        switch (rng() & 3u) {
            case 0: x = kMax; break;
            case 1: x = 0; break;
            default: x = rng(); break;
        }
    }
    return a;
}
WordsResult oracle_add(const Limbs& a, const Limbs& b) {
    WordsResult r;
    r.limbs.resize(a.size());
    r.flag = dotor_add(r.limbs.data(), a.data(), b.data(), a.size());
    return r;
}
WordsResult oracle_sub(const Limbs& a, const Limbs& b) {
    WordsResult r;
    r.limbs.resize(a.size());
    r.flag = dotor_sub(r.limbs.data(), a.data(), b.data(), a.size());
    return r;
}
Limbs oracle_mul_padded(const Limbs& a, const Limbs& b) {
    Limbs r(a.size() + b.size(), 0);
    dotor_mul(r.data(), a.data(), a.size(), b.data(), b.size());
    return r;
}
bool oracle_eq(const Limbs& a, const Limbs& b) {
    return dotor_compare(a.data(), a.size(), b.data(), b.size()) == 0;
}

void run(const char* name, const std::function<void()>& f) {
    g_case = name;
    try {
        f();
    } catch (const std::exception& e) {
        ++g_fail;
        std::fprintf(stderr, "FAIL [%s] unexpected exception: %s\n", name, e.what());
    }
}
}  // namespace

int main() {
    run("add chunk: all-ones plus carry-in clears every lane", [] {  // test_addsub.cpp:50-57
        const ChunkResult r = add_w_limbs(Limbs(8, kMax), Limbs(8, 0), 1, 8);
        for (unsigned i = 0; i < 8; ++i) CHECK(r.sums[i] == 0);
        CHECK(r.carry_out == 1);
        CHECK(r.phase4_fired);
    });
    run("sub chunk: borrow-in cascades through zero lanes", [] {  // 59-66
        const ChunkResult r = sub_w_limbs(Limbs(8, 0), Limbs(8, 0), 1, 8);
        for (unsigned i = 0; i < 8; ++i) CHECK(r.sums[i] == kMax);
        CHECK(r.carry_out == 1);
        CHECK(r.phase4_fired);
    });
    run("add chunk: generated carry ripples into a later lane", [] {  // 68-79
        const ChunkResult r = add_w_limbs(Limbs{kMax, kMax, 0, 0, 0, 0, 0, 0}, Limbs{1, 0, 0, 0, 0, 0, 0, 0}, 0, 8);
        CHECK(r.sums[0] == 0 && r.sums[1] == 0 && r.sums[2] == 1);
        for (unsigned i = 3; i < 8; ++i) CHECK(r.sums[i] == 0);
        CHECK(r.carry_out == 0);
        CHECK(r.phase4_fired);
    });
    run("chunk argument validation", [] {  // 81-90
        const Limbs a(8, 1), b(8, 1), short_b(7, 1);
        CHECK_THROWS_AS(add_w_limbs(a, b, 0, 0), std::invalid_argument);
        CHECK_THROWS_AS(add_w_limbs(a, b, 0, 9), std::invalid_argument);
        CHECK_THROWS_AS(add_w_limbs(a, b, 2, 8), std::invalid_argument);
        CHECK_THROWS_AS(add_w_limbs(a, short_b, 0, 8), std::invalid_argument);
        CHECK_THROWS_AS(sub_w_limbs(a, b, 0, 9), std::invalid_argument);
    });
    run("random chunks match the oracle chunk for every w", [] {  // 92-118
        std::mt19937_64 rng(0x9d5c0ff1u);
        for (unsigned w = 1; w <= 8; ++w) {
            for (int iter = 0; iter < 300; ++iter) {
                const Limbs a = spiky_limbs(rng, w), b = spiky_limbs(rng, w);
                const unsigned cin = unsigned(rng() & 1u);
                for (int sub = 0; sub < 2; ++sub) {
                    Limbs want(8, 0);
                    int p4 = 0;
                    const unsigned wc = dotor_chunk(sub, want.data(), a.data(), b.data(), cin, w, &p4);
                    const ChunkResult r = sub ? sub_w_limbs(a, b, cin, w) : add_w_limbs(a, b, cin, w);
                    CHECK(Limbs(r.sums.begin(), r.sums.begin() + w) == Limbs(want.begin(), want.begin() + w));
                    CHECK(r.carry_out == wc);
                    CHECK(r.phase4_fired == (p4 != 0));
                }
            }
        }
    });
    run("compare ignores high zero limbs", [] {  // test_limbs.cpp compare cases
        CHECK(compare(Limbs{1, 0, 0}, Limbs{1}) == 0);
        CHECK(compare(Limbs{0, 1}, Limbs{kMax}) == 1);
        CHECK(compare(Limbs{}, Limbs{0}) == 0);
        CHECK(compare(Limbs{5}, Limbs{6, 0}) == -1);
    });
    run("column pipeline stages through the drop-in", [] {  // test_mul.cpp:54-252
        std::mt19937_64 rng(11);
        const Limbs a = uniform_limbs(rng, 5), b = uniform_limbs(rng, 5);
        ColumnBuffers buf = gather_columns(a, b);
        CHECK(buf.m == 5 && buf.m_a.size() == 25 && buf.col_lo.size() == 10);
        for (std::size_t i = 0; i < 5; ++i) CHECK(buf.m_a[10 + i] == a[i] && buf.m_b[10 + i] == b[4 - i]);
        CHECK_THROWS_AS(gather_columns(Limbs{1, 2}, Limbs{1}), std::invalid_argument);
        CHECK_THROWS_AS(gather_columns(Limbs{}, Limbs{}), std::invalid_argument);
        compute_partials(buf, kSaturated);
        for (std::size_t t = 0; t < 25; ++t) {
            const u128 p = u128(buf.m_a[t]) * buf.m_b[t];
            CHECK(buf.p_lo[t] == limb_t(p) && buf.p_hi[t] == limb_t(p >> 64));
        }
        const auto cols = align_and_reduce(buf);
        CHECK(carry_pass(cols, kSaturated) == oracle_mul_padded(a, b));
        Limbs x(4, 0), y(4, 0);  // a lone pair: column 6 holds 2^62
        x[2] = limb_t(1) << 63;
        y[3] = limb_t(1) << 63;
        ColumnBuffers lone = gather_columns(x, y);
        compute_partials(lone, kSaturated);
        const auto lc = align_and_reduce(lone);
        for (std::size_t c = 0; c < lc.size(); ++c) CHECK(lc[c] == (c == 6 ? u128(limb_t(1) << 62) : u128(0)));
        const std::vector<u128> full{~u128(0)};
        CHECK(carry_pass(full, kUnsaturated).size() == 3);  // residual appended
        CHECK_THROWS_AS(carry_pass(full, RadixConfig{48}), std::invalid_argument);
    });
    run("2^512 - 1 plus 1 rolls over into the flag", [] {  // test_addsub.cpp:124-130
        const WordsResult r = dot_add_words(Limbs(8, kMax), Limbs{1});
        CHECK(r.limbs == Limbs(8, 0));
        CHECK(r.flag == 1);
    });
    run("adding zero is the identity", [] {
        std::mt19937_64 rng(7);
        const Limbs a = uniform_limbs(rng, 12);
        const WordsResult r = dot_add_words(a, Limbs{});
        CHECK(r.limbs == a);
        CHECK(r.flag == 0);
    });
    run("carry crosses the chunk boundary into a masked tail", [] {
        Limbs a(9, kMax), b(9, 0);
        b[0] = 1;
        const WordsResult r = dot_add_words(a, b, Width::w8);
        CHECK(r.limbs == Limbs(9, 0));
        CHECK(r.flag == 1);
    });
    run("subtracting below zero wraps and reports the borrow", [] {
        const WordsResult r = dot_sub_words(Limbs{0}, Limbs{1});
        CHECK(r.limbs == Limbs{kMax});
        CHECK(r.flag == 1);
    });
    run("words match the oracle across sizes and widths", [] {  // test_addsub.cpp:161-180
        std::mt19937_64 rng(0x51edbeefu);
        const std::size_t sizes[] = {1, 2, 3, 5, 7, 8, 9, 13, 16, 17, 31, 32, 33, 64};
        for (const std::size_t m : sizes) {
            for (int iter = 0; iter < 25; ++iter) {
                const Limbs a = spiky_limbs(rng, m), b = spiky_limbs(rng, m);
                const WordsResult aw = oracle_add(a, b), sw = oracle_sub(a, b);
                for (const Width w : {Width::scalar, Width::w2, Width::w4, Width::w8}) {
                    const WordsResult ag = dot_add_words(a, b, w);
                    CHECK(ag.limbs == aw.limbs && ag.flag == aw.flag);
                    const WordsResult sg = dot_sub_words(a, b, w);
                    CHECK(sg.limbs == sw.limbs && sg.flag == sw.flag);
                }
            }
        }
    });
    run("add then sub round-trips, flag acting as the extra limb", [] {  // 182-199
        std::mt19937_64 rng(0xabad1deau);
        for (int iter = 0; iter < 60; ++iter) {
            const std::size_t m = 1 + rng() % 40;
            const Limbs a = spiky_limbs(rng, m), b = spiky_limbs(rng, m);
            WordsResult sum = dot_add_words(a, b);
            Limbs wide = sum.limbs;
            wide.push_back(sum.flag);
            Limbs wide_b = b;
            wide_b.resize(wide.size(), 0);
            const WordsResult back = dot_sub_words(wide, wide_b);
            CHECK(back.flag == 0);
            CHECK(oracle_eq(back.limbs, a));
        }
    });
    run("unequal lengths are padded like the oracle with an equal pad", [] {  // 201-217
        std::mt19937_64 rng(0x00c0ffeeu);
        for (int iter = 0; iter < 60; ++iter) {
            const std::size_t ma = 1 + rng() % 20, mb = 1 + rng() % 20;
            const Limbs a = spiky_limbs(rng, ma), b = spiky_limbs(rng, mb);
            Limbs pa = a, pb = b;
            const std::size_t m = ma > mb ? ma : mb;
            pa.resize(m, 0);
            pb.resize(m, 0);
            const WordsResult want = oracle_add(pa, pb);
            const WordsResult got = dot_add_words(a, b);
            CHECK(got.limbs == want.limbs && got.flag == want.flag);
        }
    });
    run("span form length mismatch throws", [] {  // 219-223
        Limbs a(4, 1), b(5, 1), out(5, 0);
        CHECK_THROWS_AS(dot_add_words(std::span<limb_t>(out), a, b), std::invalid_argument);
        CHECK_THROWS_AS(dot_sub_words(std::span<limb_t>(out), a, b), std::invalid_argument);
    });
    run("output may alias either input exactly", [] {  // 250-276
        std::mt19937_64 rng(0x0dd5eedu);
        for (int iter = 0; iter < 40; ++iter) {
            const std::size_t m = 1 + rng() % 24;
            const Limbs a = spiky_limbs(rng, m), b = spiky_limbs(rng, m);
            const WordsResult want = oracle_add(a, b);
            Limbs acc = a;
            const unsigned c1 = dot_add_words(std::span<limb_t>(acc), acc, b);
            CHECK(acc == want.limbs && c1 == want.flag);
            Limbs acc2 = b;
            const unsigned c2 = dot_add_words(std::span<limb_t>(acc2), a, acc2);
            CHECK(acc2 == want.limbs && c2 == want.flag);
            const WordsResult dwant = oracle_sub(a, b);
            Limbs acc3 = a;
            const unsigned c3 = dot_sub_words(std::span<limb_t>(acc3), acc3, b);
            CHECK(acc3 == dwant.limbs && c3 == dwant.flag);
        }
    });
    run("full propagation chains", [] {  // 299-317
        const std::size_t m = 64;
        Limbs a(m, kMax), b(m, 0);
        b[0] = 1;
        const WordsResult r = dot_add_words(a, b);
        CHECK(r.limbs == Limbs(m, 0) && r.flag == 1);
        const WordsResult d = dot_sub_words(Limbs(m, 0), Limbs{1});
        CHECK(d.limbs == Limbs(m, kMax) && d.flag == 1);
    });
    run("phase 4 never fires on uniform random operands", [] {  // test_addsub.cpp:282-297
        std::mt19937_64 rng(0x5eedf00du);
        for (const Width w : {Width::scalar, Width::w2, Width::w4, Width::w8}) {
            AddSubStats st;
            for (int iter = 0; iter < 20; ++iter) {
                const Limbs a = uniform_limbs(rng, 8), b = uniform_limbs(rng, 8);
                (void)dot_add_words(a, b, w, &st);
                (void)dot_sub_words(a, b, w, &st);
            }
            CHECK(st.phase4_triggers == 0);
            CHECK(st.chunks_processed == 20u * 2u * (8 / lane_count(w)));
        }
    });
    run("phase 4 fires on every chunk of a full propagation chain", [] {  // 299-317
        const std::size_t m = 64;
        Limbs a(m, kMax), b(m, 0);
        b[0] = 1;
        for (const Width w : {Width::scalar, Width::w2, Width::w4, Width::w8}) {
            AddSubStats st;
            const WordsResult r = dot_add_words(a, b, w, &st);
            CHECK(r.limbs == Limbs(m, 0) && r.flag == 1);
            CHECK(st.chunks_processed == m / lane_count(w));
            CHECK(st.phase4_rate() == 1.0);
            AddSubStats sb;
            const WordsResult d = dot_sub_words(Limbs(m, 0), Limbs{1}, w, &sb);
            CHECK(d.limbs == Limbs(m, kMax) && d.flag == 1);
            CHECK(sb.phase4_rate() == 1.0);
        }
    });
    run("tick collection: phase laps of the timed kernel, results and counters unchanged", [] {
        // (addsub.hpp:57-63; acceptance-style check of bench.cpp:227-247's phase split)
        std::mt19937_64 rng(41);
        for (const std::size_t m : {4u, 64u, 256u}) {
            Limbs a(m), b(m);
            for (auto& x : a) x = rng();
            for (auto& x : b) x = rng();
            AddSubStats st, plain;
            st.collect_ticks = true;
            const WordsResult r = dot_add_words(a, b, Width::w8, &st);
            const WordsResult q = dot_add_words(a, b, Width::w8, &plain);
            CHECK(r.limbs == q.limbs && r.flag == q.flag);
            CHECK(st.chunks_processed == plain.chunks_processed && st.phase4_triggers == plain.phase4_triggers);
            CHECK(st.load_ticks > 0 && st.add_ticks > 0 && st.carry_gen_ticks > 0 && st.carry_add_ticks > 0 &&
                  st.store_ticks > 0 && st.overflow_ticks == 0);
            CHECK(st.carry_to_add_ratio() > 0.0);
            Limbs o(m);  // span form, exact aliasing out == a
            Limbs a2 = a;
            AddSubStats sa;
            sa.collect_ticks = true;
            CHECK(dot_add_words(std::span<limb_t>(a2), std::span<const limb_t>(a2), std::span<const limb_t>(b),
                                Width::w8, &sa) == r.flag);
            CHECK(a2 == r.limbs && sa.chunks_processed == plain.chunks_processed);
        }
        AddSubStats st;  // lengths outside the timed kernel's cover are rejected
        st.collect_ticks = true;
        CHECK_THROWS_AS(dot_add_words(Limbs(5, 1), Limbs(5, 1), Width::w8, &st), std::logic_error);
    });
    run("one-limb product is exactly the two-limb scalar product", [] {  // test_mul.cpp:323-331
        std::mt19937_64 rng(21);
        for (int iter = 0; iter < 50; ++iter) {
            const limb_t x = rng(), y = rng();
            const unsigned __int128 p = (unsigned __int128)x * y;
            CHECK(dot_mul_words(Limbs{x}, Limbs{y}) == (Limbs{limb_t(p), limb_t(p >> 64)}));
        }
    });
    run("generic product matches the oracle across sizes", [] {  // test_mul.cpp:345-359
        std::mt19937_64 rng(23);
        const std::size_t sizes[] = {1, 2, 3, 4, 5, 6, 7, 8, 12, 16, 24, 33, 48, 64, 256, 1000, 4096};
        for (const std::size_t m : sizes) {
            for (int iter = 0; iter < 12; ++iter) {
                const Limbs a = uniform_limbs(rng, m), b = uniform_limbs(rng, m);
                const Limbs got = dot_mul_words(a, b);
                CHECK(got.size() == 2 * m);
                CHECK(got == oracle_mul_padded(a, b));
            }
        }
    });
    run("generic product commutes and respects identity and zero", [] {  // 377-389
        std::mt19937_64 rng(25);
        for (int iter = 0; iter < 30; ++iter) {
            const std::size_t m = 1 + rng() % 16;
            const Limbs a = uniform_limbs(rng, m), b = uniform_limbs(rng, m);
            CHECK(dot_mul_words(a, b) == dot_mul_words(b, a));
            Limbs one(m, 0);
            one[0] = 1;
            CHECK(oracle_eq(dot_mul_words(a, one), a));
            const Limbs z = dot_mul_words(a, Limbs(m, 0));
            CHECK(oracle_eq(z, Limbs{}));
        }
    });
    run("product distributes over addition", [] {  // 391-411
        std::mt19937_64 rng(26);
        for (int iter = 0; iter < 30; ++iter) {
            const std::size_t m = 1 + rng() % 12;
            const Limbs a = uniform_limbs(rng, m), b = uniform_limbs(rng, m), c = uniform_limbs(rng, m);
            WordsResult s = dot_add_words(b, c);
            Limbs sum = s.limbs;
            sum.push_back(s.flag);
            Limbs a_pad = a;
            a_pad.resize(sum.size(), 0);
            const Limbs lhs = dot_mul_words(a_pad, sum);
            WordsResult r = dot_add_words(dot_mul_words(a, b), dot_mul_words(a, c));
            Limbs rhs = r.limbs;
            rhs.push_back(r.flag);
            CHECK(oracle_eq(lhs, rhs));
        }
    });
    run("mul argument validation", [] {  // test_mul.cpp:97-101
        CHECK_THROWS_AS(dot_mul_words(Limbs{1, 2}, Limbs{1}), std::invalid_argument);
        CHECK_THROWS_AS(dot_mul_words(Limbs{}, Limbs{}), std::invalid_argument);
        CHECK_THROWS_AS(dot_mul_words(Limbs{1}, Limbs{1}, RadixConfig{40}), std::invalid_argument);
    });
    run("karatsuba matches the oracle across thresholds and sizes", [] {  // test_mul.cpp:429-442
        std::mt19937_64 rng(28);
        const std::size_t sizes[] = {1, 2, 3, 4, 5, 7, 9, 16, 23, 33, 64, 100};
        for (const std::size_t theta : {1u, 2u, 4u, 8u}) {
            for (const std::size_t m : sizes) {
                const Limbs a = uniform_limbs(rng, m), b = uniform_limbs(rng, m);
                Limbs want = oracle_mul_padded(a, b);
                while (!want.empty() && want.back() == 0) want.pop_back();
                CHECK(karatsuba_mul(a, b, {.theta = theta}) == want);
            }
        }
        CHECK(karatsuba_mul(Limbs{1, 2}, Limbs{}).empty());
        CHECK_THROWS_AS(karatsuba_mul(Limbs{1}, Limbs{1}, {.theta = 0}), std::invalid_argument);
    });
    run("5x5 / 4x4 / 52-bit radix routes", [] {  // test_mul.cpp:258-317
        std::mt19937_64 rng(18);
        const limb_t mask52 = (limb_t(1) << 52) - 1;
        for (int iter = 0; iter < 200; ++iter) {
            Limbs a(5), b(5);
            for (auto& x : a) x = rng() & mask52;
            for (auto& x : b) x = rng() & mask52;
            const Limbs got = dot_mul_5x5(a, b);
            CHECK(got.size() == 10);
            Limbs want = oracle_mul_padded(unpack_52_to_64(a), unpack_52_to_64(b));
            while (!want.empty() && want.back() == 0) want.pop_back();
            CHECK(unpack_52_to_64(got) == want);
        }
        const Limbs ones(4, kMax);
        const Limbs sq = dot_mul_4x4(ones, ones);
        CHECK(sq.size() == 8 && sq[0] == 1 && sq[4] == kMax - 1 && sq[7] == kMax);
        std::mt19937_64 r2(19);
        Limbs x(4);
        for (auto& v : x) v = r2();
        const Limbs one_prod = dot_mul_4x4(x, Limbs{1, 0, 0, 0});
        CHECK(Limbs(one_prod.begin(), one_prod.begin() + 4) == x);
        Limbs bad(5, 1);
        bad[2] = limb_t(1) << 52;
        CHECK_THROWS_AS(dot_mul_5x5(bad, Limbs(5, 1)), std::invalid_argument);
        CHECK_THROWS_AS(dot_mul_5x5(Limbs(4, 1), Limbs(5, 1)), std::invalid_argument);
        CHECK_THROWS_AS(dot_mul_words(Limbs{kMax}, Limbs{1}, kUnsaturated), std::invalid_argument);
        for (std::size_t m : {1u, 3u, 4u, 9u}) {
            Limbs y(m);
            for (auto& v : y) v = r2();
            y.back() |= 1;
            CHECK(unpack_52_to_64(pack_64_to_52(y)) == y);
        }
    });
    run("batched extension matches the span form", [] {
        std::mt19937_64 rng(99);
        const std::size_t m = 64, B = 3000;
        Limbs a(m * B), b(m * B), out(m * B);
        for (auto& x : a) x = rng();
        for (auto& x : b) x = rng();
        std::vector<std::uint32_t> fl(B);
        dot_sub_batch(out, a, b, fl, m);
        for (std::size_t p = 0; p < B; p += 97) {
            Limbs pa(a.begin() + p * m, a.begin() + (p + 1) * m), pb(b.begin() + p * m, b.begin() + (p + 1) * m);
            const WordsResult w = oracle_sub(pa, pb);
            CHECK(Limbs(out.begin() + p * m, out.begin() + (p + 1) * m) == w.limbs && fl[p] == w.flag);
        }
    });
    run("value helpers, radix checks and width names (limbs.hpp:51-89, addsub.hpp:39-44)", [] {
        // test_limbs.cpp:149-153, test_addsub.cpp:369-370, test_mul.cpp:387
        CHECK_NOTHROW(check_limbs(Limbs{~limb_t(0)}, kSaturated));
        CHECK_NOTHROW(check_limbs(Limbs{(limb_t(1) << 52) - 1}, kUnsaturated));
        CHECK_THROWS_AS(check_limbs(Limbs{limb_t(1) << 52}, kUnsaturated), std::invalid_argument);
        CHECK_THROWS_AS(check_radix(RadixConfig{32}), std::invalid_argument);
        for (const Width w : {Width::scalar, Width::w2, Width::w4, Width::w8}) {
            CHECK(width_from_string(to_string(w)) == w);
            CHECK(dispatch_note(w) == "sm_100a");
        }
        CHECK_THROWS_AS(width_from_string("w16"), std::invalid_argument);
        const Limbs x{5, 0, 7, 0, 0};
        CHECK(sig_limbs(x) == 3 && normalized(x) == (Limbs{5, 0, 7}));
        CHECK(is_zero(Limbs{0, 0}) && is_zero(Limbs{}) && !is_zero(x));
        CHECK(dot_b200::eq(x, Limbs{5, 0, 7}) && !dot_b200::eq(x, Limbs{5, 0, 8}));
        CHECK(compare(std::span<const limb_t>(x), std::span<const limb_t>(Limbs{6})) == 1);
        std::mt19937_64 rng(321);
        for (std::size_t m : {1u, 16u, 64u}) {
            Limbs a(m);
            for (auto& v : a) v = rng();
            CHECK(is_zero(dot_mul_words(a, Limbs(m, 0))));
        }
    });
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
