// dot_b200.hpp - header-only C++ drop-in for the reference's hot-path API, over the C ABI.
//
// Mirrors namespace dot of the reference (include/dot/limbs.hpp, addsub.hpp, mul.hpp):
// same type names, same signatures, same argument meaning, same std::invalid_argument
// cases. A caller switches by replacing `#include "dot/addsub.hpp"` / `"dot/mul.hpp"`
// with this header and `dot::` with `dot_b200::` (or a namespace alias), and linking
// libdotg.so. The arithmetic runs on the B200 (sm_100a); host spans are staged through
// device memory by the *_host entry points of dotg.h. There is no CPU fallback: without
// a usable device every call throws std::runtime_error.
//
// Differences, by design:
//   * AddSubStats (addsub.hpp:53-72): chunks_processed / phase4_triggers are produced
//     (derived on the device); collect_ticks fills the phase ticks with SM-clock laps of
//     the timed team kernel (dotg_addsub_phase_ticks_host; power-of-two m <= 256, other
//     lengths throw std::logic_error).
//   * dot_mul_4x4 computes the 64-bit product directly (the reference routes it through
//     52-bit repacking and dot_mul_5x5; the 8 result limbs are identical).
//   * Partial aliasing of out with a/b (undefined in the reference) throws.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "dotg.h"

namespace dot_b200 {

using limb_t = std::uint64_t;       // limbs.hpp:17
using Limbs = std::vector<limb_t>;  // limbs.hpp:18

struct WordsResult {  // limbs.hpp:28-31
    Limbs limbs;
    unsigned flag = 0;
};

struct RadixConfig {  // limbs.hpp:39-49
    unsigned limb_bits = 64;
};
inline constexpr RadixConfig kSaturated{64};
inline constexpr RadixConfig kUnsaturated{52};

enum class Width : std::uint8_t { scalar = 0, w2 = 2, w4 = 4, w8 = 8 };  // addsub.hpp:30
constexpr unsigned lane_count(Width w) { return w == Width::scalar ? 8u : static_cast<unsigned>(w); }

inline constexpr std::size_t kMaxMulLimbs = std::size_t(1) << 24;  // mul.hpp:30

// The reference's AddSubStats (addsub.hpp:53-72): the counters are derived on the device
// from a, b and the result (csrc/stats.cu); collect_ticks fills the phase ticks from the
// timed team kernel (SM clock laps) for power-of-two m <= 256 and throws
// std::logic_error otherwise.
struct AddSubStats {
    std::uint64_t chunks_processed = 0;
    std::uint64_t phase4_triggers = 0;
    bool collect_ticks = false;
    // addsub.hpp:57-63, in SM clock cycles summed over the kernel's warps (see dotg.h)
    std::uint64_t load_ticks = 0;
    std::uint64_t add_ticks = 0;
    std::uint64_t carry_gen_ticks = 0;
    std::uint64_t carry_add_ticks = 0;
    std::uint64_t store_ticks = 0;
    std::uint64_t overflow_ticks = 0;
    double phase4_rate() const {
        return chunks_processed ? double(phase4_triggers) / double(chunks_processed) : 0.0;
    }
    // addsub.cpp:258-263
    double carry_to_add_ratio() const {
        if (add_ticks == 0) return 0.0;
        return double(carry_gen_ticks + carry_add_ticks + store_ticks + overflow_ticks) / double(add_ticks);
    }
    void merge(const AddSubStats& o) {
        chunks_processed += o.chunks_processed;
        phase4_triggers += o.phase4_triggers;
        load_ticks += o.load_ticks;
        add_ticks += o.add_ticks;
        carry_gen_ticks += o.carry_gen_ticks;
        carry_add_ticks += o.carry_add_ticks;
        store_ticks += o.store_ticks;
        overflow_ticks += o.overflow_ticks;
    }
};

namespace detail {
inline void check(int rc) {
    if (rc == DOTG_OK) return;
    const std::string msg = dotg_last_error();
    if (rc == DOTG_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error("dotg: " + msg);
}
inline bool ticks_supported(std::size_t m) { return m != 0 && m <= 256 && (m & (m - 1)) == 0; }
inline void no_ticks(const AddSubStats* st, std::size_t m) {
    if (st != nullptr && st->collect_ticks && !ticks_supported(m))
        throw std::logic_error("AddSubStats::collect_ticks: the timed device kernel covers power-of-two m <= 256");
}
inline void validate(Width w) { check(dotg_validate_width(static_cast<int>(w))); }

inline unsigned run_words(bool sub, std::span<limb_t> out, std::span<const limb_t> a,
                          std::span<const limb_t> b, Width w, AddSubStats* st) {
    validate(w);
    if (a.size() != b.size() || out.size() != a.size())  // addsub.cpp:139-140
        throw std::invalid_argument("dot add/sub: operand lengths differ (caller pads)");
    no_ticks(st, a.size());
    std::uint32_t carry = 0;
    if (st != nullptr && st->collect_ticks) {
        // the counters first (into scratch: out may alias a or b), then the phase laps of
        // the timed team kernel, which writes out
        std::uint64_t ch = 0, fi = 0;
        std::uint32_t c2 = 0;
        std::vector<limb_t> scratch(a.size());
        check(dotg_words_host_stats(sub ? 1 : 0, scratch.data(), a.data(), b.data(), a.size(), static_cast<int>(w),
                                    &c2, &ch, &fi));
        st->chunks_processed += ch;
        st->phase4_triggers += fi;
        std::uint64_t t[6] = {};
        check(dotg_addsub_phase_ticks_host(sub ? 1 : 0, out.data(), a.data(), b.data(), &carry, a.size(), 1, t));
        st->load_ticks += t[0];
        st->add_ticks += t[1];
        st->carry_gen_ticks += t[2];
        st->carry_add_ticks += t[3];
        st->store_ticks += t[4];
        st->overflow_ticks += t[5];
        return carry;
    }
    if (st != nullptr) {
        std::uint64_t ch = 0, fi = 0;
        check(dotg_words_host_stats(sub ? 1 : 0, out.data(), a.data(), b.data(), a.size(), static_cast<int>(w),
                                    &carry, &ch, &fi));
        st->chunks_processed += ch;
        st->phase4_triggers += fi;
        return carry;
    }
    check(sub ? dotg_sub_words_host(out.data(), a.data(), b.data(), a.size(), &carry)
              : dotg_add_words_host(out.data(), a.data(), b.data(), a.size(), &carry));
    return carry;
}

inline WordsResult run_limbs(bool sub, const Limbs& a, const Limbs& b, Width w,
                             AddSubStats* st) {  // addsub.cpp:192-211
    const std::size_t m = a.size() > b.size() ? a.size() : b.size();
    Limbs pa = a, pb = b;
    pa.resize(m, 0);
    pb.resize(m, 0);
    WordsResult r;
    r.limbs.resize(m);
    r.flag = run_words(sub, r.limbs, pa, pb, w, st);
    return r;
}
}  // namespace detail

// Chunk-level operations (addsub.hpp:78-89): one chunk of w lanes, 1 <= w <= 8.
struct ChunkResult {
    std::array<limb_t, 8> sums{};  // first w entries valid
    unsigned carry_out = 0;        // borrow_out for subtraction
    bool phase4_fired = false;
};

namespace detail {
inline ChunkResult run_chunk(bool sub, std::span<const limb_t> a, std::span<const limb_t> b, unsigned carry_in,
                             unsigned w) {  // addsub.cpp:172-190
    if (w < 1 || w > 8) throw std::invalid_argument("chunk width must be in 1..8");
    if (a.size() != w || b.size() != w) throw std::invalid_argument("chunk operands must have exactly w limbs");
    if (carry_in > 1) throw std::invalid_argument("carry_in must be 0 or 1");
    ChunkResult r;
    std::uint32_t co = 0, fired = 0;
    check(dotg_chunk_host(sub ? 1 : 0, r.sums.data(), &co, &fired, a.data(), b.data(), carry_in, w));
    r.carry_out = co;
    r.phase4_fired = fired != 0;
    return r;
}
}  // namespace detail

inline ChunkResult add_w_limbs(std::span<const limb_t> a, std::span<const limb_t> b, unsigned carry_in,
                               unsigned w) {
    return detail::run_chunk(false, a, b, carry_in, w);
}
inline ChunkResult sub_w_limbs(std::span<const limb_t> a, std::span<const limb_t> b, unsigned borrow_in,
                               unsigned w) {
    return detail::run_chunk(true, a, b, borrow_in, w);
}

// out = a + b (mod 2^(64m)); returns the carry (addsub.hpp:98-100).
inline unsigned dot_add_words(std::span<limb_t> out, std::span<const limb_t> a, std::span<const limb_t> b,
                              Width w = Width::w8, AddSubStats* stats = nullptr) {
    return detail::run_words(false, out, a, b, w, stats);
}
// out = a - b (mod 2^(64m)); returns the borrow (addsub.hpp:101-103).
inline unsigned dot_sub_words(std::span<limb_t> out, std::span<const limb_t> a, std::span<const limb_t> b,
                              Width w = Width::w8, AddSubStats* stats = nullptr) {
    return detail::run_words(true, out, a, b, w, stats);
}
// Value forms: unequal lengths are zero-padded to the longer one (addsub.hpp:106-109).
inline WordsResult dot_add_words(const Limbs& a, const Limbs& b, Width w = Width::w8,
                                 AddSubStats* stats = nullptr) {
    return detail::run_limbs(false, a, b, w, stats);
}
inline WordsResult dot_sub_words(const Limbs& a, const Limbs& b, Width w = Width::w8,
                                 AddSubStats* stats = nullptr) {
    return detail::run_limbs(true, a, b, w, stats);
}

// Value ordering ignoring high zero limbs: -1 / 0 / +1 (limbs.hpp:84, limbs.cpp:46-53).
inline int compare(const Limbs& a, const Limbs& b) {
    const std::size_t m = a.size() > b.size() ? a.size() : b.size();
    Limbs pa = a, pb = b;
    pa.resize(m, 0);
    pb.resize(m, 0);
    std::int32_t r = 0;
    detail::check(dotg_compare_host(&r, pa.data(), pb.data(), m, 1));
    return r;
}
inline int compare(std::span<const limb_t> a, std::span<const limb_t> b) {  // limbs.hpp:83
    return compare(Limbs(a.begin(), a.end()), Limbs(b.begin(), b.end()));
}

// The host-side value helpers of limbs.hpp:51-89 (lengths, zeros and headroom bits only;
// nothing here is arithmetic on the path).
inline std::size_t sig_limbs(std::span<const limb_t> a) {  // limbs.hpp:80
    std::size_t n = a.size();
    for (; n != 0 && a[n - 1] == 0; --n) {
    }
    return n;
}
inline Limbs normalized(Limbs a) {  // limbs.hpp:81
    a.resize(sig_limbs(a));
    return a;
}
inline bool eq(const Limbs& a, const Limbs& b) { return compare(a, b) == 0; }  // limbs.hpp:88
inline bool is_zero(const Limbs& a) { return sig_limbs(a) == 0; }           // limbs.hpp:89
inline void check_radix(RadixConfig cfg) {                                   // limbs.hpp:51-52
    if (cfg.limb_bits != 64 && cfg.limb_bits != 52)
        throw std::invalid_argument("RadixConfig: limb_bits must be 64 or 52");
}
inline void check_limbs(const Limbs& a, RadixConfig cfg) {  // limbs.hpp:54-55
    check_radix(cfg);
    if (cfg.limb_bits == 64) return;
    for (std::size_t i = 0; i < a.size(); ++i)
        if (a[i] >> cfg.limb_bits)
            throw std::invalid_argument("limb " + std::to_string(i) + " exceeds the configured limb width");
}

// Width names (addsub.hpp:39-44). The widths select nothing on the device; dispatch_note
// names what actually runs.
inline std::string_view to_string(Width w) {
    switch (w) {
        case Width::scalar: return "scalar";
        case Width::w2: return "2";
        case Width::w4: return "4";
        case Width::w8: return "8";
    }
    return "?";
}
inline Width width_from_string(std::string_view s) {
    if (s == "scalar") return Width::scalar;
    if (s == "2") return Width::w2;
    if (s == "4") return Width::w4;
    if (s == "8") return Width::w8;
    throw std::invalid_argument("unknown width: expected one of 2, 4, 8, scalar");
}
inline std::string_view dispatch_note(Width w) {
    detail::validate(w);
    return "sm_100a";  // every width runs the same B200 kernels
}

// ---- The column pipeline as separate stages (mul.hpp:32-67, mul.cpp:12-90), each run on
// the device (dotg_*_host stages of dotg.h); dot_mul_words below does not go through them
// (its kernels fuse the four stages in registers).
using u128 = unsigned __int128;  // limbs.hpp:20-24

constexpr std::size_t num_pairs(std::size_t c, std::size_t m) {  // mul.hpp:36-38
    const std::size_t x = c + 1, y = 2 * m - 1 - c;
    return x < m ? (x < y ? x : y) : (m < y ? m : y);
}

struct ColumnBuffers {  // mul.hpp:42-49
    std::size_t m = 0;
    std::vector<limb_t> m_a;
    std::vector<limb_t> m_b;
    std::vector<limb_t> p_lo;
    std::vector<limb_t> p_hi;
    std::vector<u128> col_lo;
};

inline ColumnBuffers gather_columns(const Limbs& a, const Limbs& b) {  // mul.cpp:12-36
    if (a.size() != b.size()) throw std::invalid_argument("dot mul: operand lengths differ (caller pads)");
    ColumnBuffers buf;
    buf.m = a.size();
    buf.m_a.resize(buf.m * buf.m);
    buf.m_b.resize(buf.m * buf.m);
    detail::check(dotg_gather_columns_host(buf.m_a.data(), buf.m_b.data(), a.data(), b.data(), buf.m));
    buf.p_lo.assign(buf.m * buf.m, 0);
    buf.p_hi.assign(buf.m * buf.m, 0);
    buf.col_lo.assign(2 * buf.m, 0);
    return buf;
}

inline void compute_partials(ColumnBuffers& buf, RadixConfig cfg, Width w = Width::w8) {  // mul.cpp:38-52
    detail::validate(w);
    buf.p_lo.resize(buf.m_a.size());
    buf.p_hi.resize(buf.m_a.size());
    if (buf.m_b.size() != buf.m_a.size()) throw std::invalid_argument("column buffers: m_a / m_b sizes differ");
    detail::check(dotg_compute_partials_host(buf.p_lo.data(), buf.p_hi.data(), buf.m_a.data(), buf.m_b.data(),
                                             buf.m_a.size(), static_cast<int>(cfg.limb_bits)));
}

inline std::span<const u128> align_and_reduce(ColumnBuffers& buf) {  // mul.cpp:54-68
    std::vector<limb_t> cols(4 * buf.m);
    detail::check(dotg_align_and_reduce_host(cols.data(), buf.p_lo.data(), buf.p_hi.data(), buf.m));
    buf.col_lo.resize(2 * buf.m);
    for (std::size_t c = 0; c < 2 * buf.m; ++c) buf.col_lo[c] = u128(cols[2 * c]) | (u128(cols[2 * c + 1]) << 64);
    return {buf.col_lo.data(), buf.col_lo.size()};
}

inline Limbs carry_pass(std::span<const u128> columns, RadixConfig cfg) {  // mul.cpp:70-90
    std::vector<limb_t> cols(2 * columns.size());
    for (std::size_t c = 0; c < columns.size(); ++c) {
        cols[2 * c] = limb_t(columns[c]);
        cols[2 * c + 1] = limb_t(columns[c] >> 64);
    }
    Limbs out(columns.size() + 2);
    std::uint32_t n = 0;
    detail::check(dotg_carry_pass_host(out.data(), &n, out.size(), cols.data(), columns.size(),
                                       static_cast<int>(cfg.limb_bits)));
    out.resize(n);
    return out;
}

// Exact product, exactly 2m limbs; equal lengths 1 <= m <= 2^24 (mul.hpp:75-76).
inline Limbs dot_mul_words(const Limbs& a, const Limbs& b, RadixConfig cfg = kSaturated,
                           Width w = Width::w8) {
    if (cfg.limb_bits != 64 && cfg.limb_bits != 52)
        throw std::invalid_argument("RadixConfig: limb_bits must be 64 or 52");
    detail::validate(w);
    if (a.size() != b.size()) throw std::invalid_argument("dot mul: operand lengths differ (caller pads)");
    if (a.empty()) throw std::invalid_argument("dot mul: operands need at least one limb");
    if (a.size() > kMaxMulLimbs)
        throw std::invalid_argument("dot mul: limb count exceeds the column accumulator bound");
    Limbs out(2 * a.size());
    if (cfg.limb_bits == 52)  // unsaturated radix: limbs < 2^52 (checked), 2m limbs < 2^52
        detail::check(dotg_mul52_batch_host(out.data(), a.data(), b.data(), a.size(), 1));
    else
        detail::check(dotg_mul_batch_host(out.data(), a.data(), b.data(), a.size(), 1));
    return out;
}

// Fixed 5-limb product over 52-bit limbs, exactly 10 limbs (mul.hpp:78-80).
inline Limbs dot_mul_5x5(const Limbs& a, const Limbs& b) {
    if (a.size() != 5 || b.size() != 5) throw std::invalid_argument("dot mul 5x5: operands must be exactly 5 limbs");
    return dot_mul_words(a, b, kUnsaturated);
}

// Fixed 4-limb product, exactly 8 limbs (mul.hpp:82-85).
inline Limbs dot_mul_4x4(const Limbs& a, const Limbs& b) {
    if (a.size() != 4 || b.size() != 4) throw std::invalid_argument("dot mul 4x4: operands must be exactly 4 limbs");
    return dot_mul_words(a, b);
}

// 64 <-> 52-bit re-slicing (limbs.hpp:111-117); host representation helpers.
inline Limbs pack_64_to_52(const Limbs& a) {
    const std::size_t n = (a.size() * 64 + 51) / 52;
    Limbs out(n);
    for (std::size_t j = 0; j < n; ++j) {
        const std::size_t bit = j * 52, word = bit / 64;
        const unsigned off = unsigned(bit % 64);
        limb_t v = a[word] >> off;
        if (off > 12 && word + 1 < a.size()) v |= a[word + 1] << (64 - off);
        out[j] = v & ((limb_t(1) << 52) - 1);
    }
    return out;
}
inline Limbs unpack_52_to_64(const Limbs& a) {
    Limbs out((a.size() * 52 + 63) / 64, 0);
    for (std::size_t j = 0; j < a.size(); ++j) {
        if (a[j] >> 52) throw std::invalid_argument("limb " + std::to_string(j) + " exceeds the configured limb width");
        const std::size_t bit = j * 52, word = bit / 64;
        const unsigned off = unsigned(bit % 64);
        out[word] |= a[j] << off;
        if (off > 12) out[word + 1] |= a[j] >> (64 - off);
    }
    while (!out.empty() && out.back() == 0) out.pop_back();
    return out;
}

struct KaratsubaConfig {  // mul.hpp:91-93
    std::size_t theta = 4;
};

// mul.hpp:95-102: inputs trimmed, unequal lengths padded at entry, result trimmed.
// Breadth-first on the device (dotg_karatsuba_batch_host).
inline Limbs karatsuba_mul(const Limbs& a, const Limbs& b, KaratsubaConfig cfg = {}) {
    if (cfg.theta < 1) throw std::invalid_argument("karatsuba: threshold must be at least 1");
    auto sig = [](const Limbs& x) {
        std::size_t n = x.size();
        while (n > 0 && x[n - 1] == 0) --n;
        return n;
    };
    const std::size_t na = sig(a), nb = sig(b);
    if (na == 0 || nb == 0) return {};
    const std::size_t m = na > nb ? na : nb;
    Limbs pa(a.begin(), a.begin() + na), pb(b.begin(), b.begin() + nb);
    pa.resize(m, 0);
    pb.resize(m, 0);
    Limbs out(2 * m);
    detail::check(dotg_karatsuba_batch_host(out.data(), pa.data(), pb.data(), m, 1, cfg.theta));
    out.resize(sig(out));
    return out;
}

// Batched extensions (no reference equivalent; one call instead of a loop over pairs):
// row-major host arrays [batch][m]; flags[batch] may be empty.
inline void dot_add_batch(std::span<limb_t> out, std::span<const limb_t> a, std::span<const limb_t> b,
                          std::span<std::uint32_t> flags, std::size_t m) {
    if (m == 0 || a.size() % m || a.size() != b.size() || out.size() != a.size())
        throw std::invalid_argument("dot add batch: shapes differ");
    detail::check(dotg_add_batch_host(out.data(), a.data(), b.data(), flags.empty() ? nullptr : flags.data(), m,
                                      a.size() / m));
}
inline void dot_sub_batch(std::span<limb_t> out, std::span<const limb_t> a, std::span<const limb_t> b,
                          std::span<std::uint32_t> flags, std::size_t m) {
    if (m == 0 || a.size() % m || a.size() != b.size() || out.size() != a.size())
        throw std::invalid_argument("dot sub batch: shapes differ");
    detail::check(dotg_sub_batch_host(out.data(), a.data(), b.data(), flags.empty() ? nullptr : flags.data(), m,
                                      a.size() / m));
}
inline void dot_mul_batch(std::span<limb_t> out, std::span<const limb_t> a, std::span<const limb_t> b,
                          std::size_t m) {
    if (m == 0 || a.size() % m || a.size() != b.size() || out.size() != 2 * a.size())
        throw std::invalid_argument("dot mul batch: shapes differ");
    detail::check(dotg_mul_batch_host(out.data(), a.data(), b.data(), m, a.size() / m));
}

}  // namespace dot_b200
