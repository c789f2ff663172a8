// ref_shim.cpp - C-ABI wrapper around the UNMODIFIED reference (TEST INFRASTRUCTURE).
//
// Linked by oracle/Makefile with the reference's own translation units, compiled
// from where they lie under /root/reference/proj/src (nothing is copied). It lets
// Python load the reference through ctypes to (a) generate golden vectors,
// (b) pin oracle/dot_oracle.c, and (c) serve as the CPU baseline
// (bench.py cpu_baseline / --impl reference, kind "reference").
//
// Only the reference's public API is called (include/dot/*.hpp):
//   dot_add_words / dot_sub_words span + value forms   addsub.hpp:95-109
//   add_w_limbs / sub_w_limbs                           addsub.hpp:86-89
//   dot_mul_words                                       mul.hpp:75-76
//   oracle_add / oracle_sub / oracle_mul                oracle.hpp:18-23
//   dispatch_note                                       addsub.hpp:41-43
// std::invalid_argument is caught and turned into return code -1 (message kept).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "dot/addsub.hpp"
#include "dot/limbs.hpp"
#include "dot/mul.hpp"
#include "dot/oracle.hpp"

using dot::limb_t;
using dot::Limbs;

namespace {
thread_local std::string g_err;

dot::Width width_of(int w) {
    switch (w) {
        case 0: return dot::Width::scalar;
        case 2: return dot::Width::w2;
        case 4: return dot::Width::w4;
        case 8: return dot::Width::w8;
        default: return static_cast<dot::Width>(w);  // lets validate_width throw
    }
}

template <class F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return -1;
    }
}
}  // namespace

extern "C" {

const char* dotref_last_error() { return g_err.c_str(); }

const char* dotref_dispatch_note(int w) {
    static std::string s;
    s = std::string(dot::dispatch_note(width_of(w)));
    return s.c_str();
}

// Span form. Returns the carry/borrow (0/1) or -1 on std::invalid_argument.
int dotref_words(int sub, limb_t* out, size_t mo, const limb_t* a, size_t ma, const limb_t* b,
                 size_t mb, int width, uint64_t* chunks, uint64_t* fires) {
    return guarded([&] {
        dot::AddSubStats st;
        std::span<limb_t> so(out, mo);
        std::span<const limb_t> sa(a, ma), sb(b, mb);
        unsigned c = sub ? dot::dot_sub_words(so, sa, sb, width_of(width), &st)
                         : dot::dot_add_words(so, sa, sb, width_of(width), &st);
        if (chunks) *chunks = st.chunks_processed;
        if (fires) *fires = st.phase4_triggers;
        return int(c);
    });
}

// Value form (zero-pads to the longer operand). out must hold max(ma, mb) limbs.
int dotref_words_value(int sub, limb_t* out, const limb_t* a, size_t ma, const limb_t* b,
                       size_t mb, int width) {
    return guarded([&] {
        const Limbs va(a, a + ma), vb(b, b + mb);
        const dot::WordsResult r = sub ? dot::dot_sub_words(va, vb, width_of(width))
                                       : dot::dot_add_words(va, vb, width_of(width));
        std::copy(r.limbs.begin(), r.limbs.end(), out);
        return int(r.flag);
    });
}

// Chunk API: returns carry_out, *phase4 = phase4_fired, sums written to out[0..w).
int dotref_chunk(int sub, limb_t* out, const limb_t* a, const limb_t* b, size_t len,
                 unsigned carry_in, unsigned w, int* phase4) {
    return guarded([&] {
        std::span<const limb_t> sa(a, len), sb(b, len);
        const dot::ChunkResult r = sub ? dot::sub_w_limbs(sa, sb, carry_in, w)
                                       : dot::add_w_limbs(sa, sb, carry_in, w);
        std::copy(r.sums.begin(), r.sums.begin() + std::min<size_t>(w, 8), out);
        if (phase4) *phase4 = r.phase4_fired ? 1 : 0;
        return int(r.carry_out);
    });
}

// dot_mul_words: writes exactly 2m limbs. Returns 0 or -1.
int dotref_mul_words(limb_t* out, const limb_t* a, size_t ma, const limb_t* b, size_t mb) {
    return guarded([&] {
        const Limbs r = dot::dot_mul_words(Limbs(a, a + ma), Limbs(b, b + mb));
        std::copy(r.begin(), r.end(), out);
        return int(r.size());
    });
}

// The column pipeline stages one by one (mul.hpp:32-67, mul.cpp:12-90), so the device
// stages (dotg_gather_columns ... dotg_carry_pass) are pinned to the reference's own
// outputs. u128 values cross the ABI as (low 64, high 64) pairs.
namespace {
dot::RadixConfig radix_of(int bits) { return bits == 52 ? dot::kUnsaturated : dot::kSaturated; }
}  // namespace

// gather_columns: m_a / m_b receive the m*m gathered limbs (column order). Returns m*m.
int dotref_gather_columns(limb_t* m_a, limb_t* m_b, const limb_t* a, const limb_t* b, size_t m) {
    return guarded([&] {
        const dot::ColumnBuffers buf = dot::gather_columns(Limbs(a, a + m), Limbs(b, b + m));
        std::copy(buf.m_a.begin(), buf.m_a.end(), m_a);
        std::copy(buf.m_b.begin(), buf.m_b.end(), m_b);
        return int(buf.m_a.size());
    });
}

// compute_partials over n gathered pairs (any n; the reference only reads m_a / m_b).
int dotref_compute_partials(limb_t* p_lo, limb_t* p_hi, const limb_t* m_a, const limb_t* m_b, size_t n,
                            int limb_bits, int width) {
    return guarded([&] {
        dot::ColumnBuffers buf;
        buf.m_a.assign(m_a, m_a + n);
        buf.m_b.assign(m_b, m_b + n);
        buf.p_lo.assign(n, 0);
        buf.p_hi.assign(n, 0);
        dot::compute_partials(buf, radix_of(limb_bits), width_of(width));
        std::copy(buf.p_lo.begin(), buf.p_lo.end(), p_lo);
        std::copy(buf.p_hi.begin(), buf.p_hi.end(), p_hi);
        return 0;
    });
}

// align_and_reduce of the m*m partials of an m-limb product: 2m u128 column sums.
int dotref_align_and_reduce(limb_t* columns, const limb_t* p_lo, const limb_t* p_hi, size_t m) {
    return guarded([&] {
        dot::ColumnBuffers buf;
        buf.m = m;
        buf.p_lo.assign(p_lo, p_lo + m * m);
        buf.p_hi.assign(p_hi, p_hi + m * m);
        buf.col_lo.assign(2 * m, 0);
        const std::span<const dot::u128> cols = dot::align_and_reduce(buf);
        for (size_t c = 0; c < cols.size(); ++c) {
            columns[2 * c] = limb_t(cols[c]);
            columns[2 * c + 1] = limb_t(cols[c] >> 64);
        }
        return int(cols.size());
    });
}

// carry_pass over ncols arbitrary u128 columns; out must hold ncols + 3 limbs. Returns the
// number of limbs written (ncols plus the residual limbs, if any).
int dotref_carry_pass(limb_t* out, const limb_t* columns, size_t ncols, int limb_bits) {
    return guarded([&] {
        std::vector<dot::u128> cols(ncols);
        for (size_t c = 0; c < ncols; ++c) cols[c] = (dot::u128(columns[2 * c + 1]) << 64) | columns[2 * c];
        const Limbs r = dot::carry_pass(std::span<const dot::u128>(cols.data(), cols.size()), radix_of(limb_bits));
        std::copy(r.begin(), r.end(), out);
        return int(r.size());
    });
}

// 52-bit radix routes (mul.hpp:73-85): dot_mul_words(kUnsaturated), dot_mul_5x5,
// dot_mul_4x4, and the repacking helpers (limbs.hpp:111-117). Return the output length.
int dotref_mul_words52(limb_t* out, const limb_t* a, size_t ma, const limb_t* b, size_t mb) {
    return guarded([&] {
        const Limbs r = dot::dot_mul_words(Limbs(a, a + ma), Limbs(b, b + mb), dot::kUnsaturated);
        std::copy(r.begin(), r.end(), out);
        return int(r.size());
    });
}

int dotref_mul_5x5(limb_t* out, const limb_t* a, size_t ma, const limb_t* b, size_t mb) {
    return guarded([&] {
        const Limbs r = dot::dot_mul_5x5(Limbs(a, a + ma), Limbs(b, b + mb));
        std::copy(r.begin(), r.end(), out);
        return int(r.size());
    });
}

int dotref_mul_4x4(limb_t* out, const limb_t* a, size_t ma, const limb_t* b, size_t mb) {
    return guarded([&] {
        const Limbs r = dot::dot_mul_4x4(Limbs(a, a + ma), Limbs(b, b + mb));
        std::copy(r.begin(), r.end(), out);
        return int(r.size());
    });
}

int dotref_pack_64_to_52(limb_t* out, const limb_t* a, size_t m) {
    return guarded([&] {
        const Limbs r = dot::pack_64_to_52(Limbs(a, a + m));
        std::copy(r.begin(), r.end(), out);
        return int(r.size());
    });
}

int dotref_unpack_52_to_64(limb_t* out, const limb_t* a, size_t m) {
    return guarded([&] {
        const Limbs r = dot::unpack_52_to_64(Limbs(a, a + m));
        std::copy(r.begin(), r.end(), out);
        return int(r.size());
    });
}

int dotref_oracle_addsub(int sub, limb_t* out, const limb_t* a, size_t ma, const limb_t* b,
                         size_t mb) {
    return guarded([&] {
        const Limbs va(a, a + ma), vb(b, b + mb);
        const dot::WordsResult r = sub ? dot::oracle_sub(va, vb) : dot::oracle_add(va, vb);
        std::copy(r.limbs.begin(), r.limbs.end(), out);
        return int(r.flag);
    });
}

// oracle_mul: out must hold ma+mb limbs; writes the trimmed result, zero-pads the rest,
// returns the trimmed length.
int dotref_oracle_mul(limb_t* out, const limb_t* a, size_t ma, const limb_t* b, size_t mb) {
    return guarded([&] {
        const Limbs r = dot::oracle_mul(Limbs(a, a + ma), Limbs(b, b + mb));
        std::fill(out, out + ma + mb, limb_t(0));
        std::copy(r.begin(), r.end(), out);
        return int(r.size());
    });
}

// Batched CPU baseline over [batch][m] row-major operands with a static partition
// of pairs across nthreads std::threads (the reference functions are pure and
// reentrant). op: 0 add, 1 sub, 2 mul. impl: 0 = the DoT path, 2 = its
// value form for add/sub
// (span-form dot_add_words/dot_sub_words at Width::w8, dot_mul_words), 1 = oracle.
// flags may be null for mul. out is [batch][m] (add/sub) or [batch][2m] (mul).
int dotref_batch(int op, int impl, limb_t* out, const limb_t* a, const limb_t* b, uint32_t* flags,
                 size_t m, size_t batch, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    std::vector<std::thread> pool;
    std::vector<int> status(size_t(nthreads), 0);
    auto work = [&](int t) {
        const size_t lo = batch * size_t(t) / size_t(nthreads);
        const size_t hi = batch * size_t(t + 1) / size_t(nthreads);
        status[size_t(t)] = guarded([&] {
            for (size_t p = lo; p < hi; ++p) {
                const limb_t* pa = a + p * m;
                const limb_t* pb = b + p * m;
                if (op == 2) {
                    limb_t* po = out + p * 2 * m;
                    const Limbs va(pa, pa + m), vb(pb, pb + m);
                    if (impl == 0) {
                        const Limbs r = dot::dot_mul_words(va, vb);
                        std::copy(r.begin(), r.end(), po);
                    } else {
                        const Limbs r = dot::oracle_mul(va, vb);
                        std::fill(po, po + 2 * m, limb_t(0));
                        std::copy(r.begin(), r.end(), po);
                    }
                } else {
                    limb_t* po = out + p * m;
                    unsigned f;
                    if (impl == 0) {
                        std::span<limb_t> so(po, m);
                        std::span<const limb_t> sa(pa, m), sb(pb, m);
                        f = op ? dot::dot_sub_words(so, sa, sb, dot::Width::w8)
                               : dot::dot_add_words(so, sa, sb, dot::Width::w8);
                    } else if (impl == 2) {  // value form (allocates the result, bench.cpp:95-104)
                        const Limbs va(pa, pa + m), vb(pb, pb + m);
                        const dot::WordsResult r = op ? dot::dot_sub_words(va, vb, dot::Width::w8)
                                                      : dot::dot_add_words(va, vb, dot::Width::w8);
                        std::copy(r.limbs.begin(), r.limbs.end(), po);
                        f = r.flag;
                    } else {
                        const Limbs va(pa, pa + m), vb(pb, pb + m);
                        const dot::WordsResult r = op ? dot::oracle_sub(va, vb) : dot::oracle_add(va, vb);
                        std::copy(r.limbs.begin(), r.limbs.end(), po);
                        f = r.flag;
                    }
                    if (flags) flags[p] = f;
                }
            }
            return 0;
        });
    };
    for (int t = 1; t < nthreads; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    for (int s : status)
        if (s != 0) return s;
    return 0;
}

}  // extern "C"
