/* dot_oracle.c - CPU restatement of the reference's limb arithmetic (TEST INFRASTRUCTURE).
 *
 * See dot_oracle.h for the role of this file and how it is pinned. Each function
 * cites the reference routine (paths under /root/reference/proj) whose algorithm it
 * restates; no reference source is copied.
 */
#include "dot_oracle.h"

#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* oracle.cpp:16-31 - carry threaded limb by limb; at most one of the two wraps
 * of a limb can happen, so the carry stays 0/1. */
unsigned dotor_add(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m) {
    unsigned c = 0;
    for (size_t i = 0; i < m; ++i) {
        uint64_t r = a[i] + (uint64_t)c;
        unsigned w = r < (uint64_t)c;
        r += b[i];
        w += r < b[i];
        out[i] = r;
        c = w;
    }
    return c;
}

/* oracle.cpp:33-48 */
unsigned dotor_sub(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m) {
    unsigned bw = 0;
    for (size_t i = 0; i < m; ++i) {
        const uint64_t ai = a[i], bi = b[i];
        uint64_t r = ai - (uint64_t)bw;
        unsigned nb = r > ai;
        nb += r < bi;
        out[i] = r - bi;
        bw = nb;
    }
    return bw;
}

static size_t sig_limbs(const uint64_t* a, size_t m) { /* limbs.cpp:35-39 */
    while (m > 0 && a[m - 1] == 0) --m;
    return m;
}

/* oracle.cpp:50-63 */
size_t dotor_mul(uint64_t* out, const uint64_t* a, size_t ma, const uint64_t* b, size_t mb) {
    if (ma == 0 || mb == 0) return 0;
    memset(out, 0, sizeof(uint64_t) * (ma + mb));
    for (size_t i = 0; i < ma; ++i) {
        uint64_t carry = 0;
        for (size_t j = 0; j < mb; ++j) {
            const u128 t = (u128)a[i] * b[j] + out[i + j] + carry;
            out[i + j] = (uint64_t)t;
            carry = (uint64_t)(t >> 64);
        }
        out[i + mb] = carry;
    }
    return sig_limbs(out, ma + mb);
}

/* addsub.cpp:21-84 (chunk_generic, untimed). Phase 1 lane sums; phase 2 lane carry
 * mask, top-lane capture, shift-in of carry_in (LaneMask::shifted_in, limbs.hpp:71-73);
 * phase 3 aligned carry add plus secondary overflow mask; phase 4 (only if the
 * secondary mask is non-zero) settles every cascade with one mask addition. */
unsigned dotor_chunk(int sub, uint64_t* out, const uint64_t* a, const uint64_t* b,
                     unsigned carry_in, unsigned t, int* phase4) {
    uint64_t av[8], bv[8], r[8], f[8];
    const uint32_t lane_bits = (1u << t) - 1u;
    for (unsigned i = 0; i < t; ++i) { av[i] = a[i]; bv[i] = b[i]; }
    for (unsigned i = 0; i < t; ++i) r[i] = sub ? av[i] - bv[i] : av[i] + bv[i];

    uint32_t c = 0;
    for (unsigned i = 0; i < t; ++i)
        c |= (uint32_t)(sub ? av[i] < bv[i] : r[i] < av[i]) << i;
    unsigned flag_out = (c >> (t - 1)) & 1u;
    c = ((c << 1) | (carry_in & 1u)) & lane_bits;

    for (unsigned i = 0; i < t; ++i) {
        const uint64_t bit = (c >> i) & 1u;
        f[i] = sub ? r[i] - bit : r[i] + bit;
    }
    uint32_t sec = 0;
    for (unsigned i = 0; i < t; ++i)
        sec |= (uint32_t)(sub ? f[i] > r[i] : f[i] < r[i]) << i;
    const int fired = sec != 0;
    if (fired) {
        uint32_t prop = 0;
        for (unsigned i = 0; i < t; ++i)
            prop |= (uint32_t)(sub ? f[i] == 0 : f[i] == ~(uint64_t)0) << i;
        const uint32_t settled = (sec << 1) + prop;
        flag_out |= (settled >> t) & 1u;
        const uint32_t adjust = (settled ^ prop) & lane_bits;
        for (unsigned i = 0; i < t; ++i) {
            const uint64_t bit = (adjust >> i) & 1u;
            f[i] = sub ? f[i] - bit : f[i] + bit;
        }
    }
    for (unsigned i = 0; i < t; ++i) out[i] = f[i];
    if (phase4) *phase4 = fired;
    return flag_out;
}

/* addsub.cpp:136-170 (run_words): full chunks, then one masked tail of m % lanes. */
unsigned dotor_words(int sub, uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m,
                     unsigned lanes, uint64_t* chunks, uint64_t* fires) {
    unsigned carry = 0;
    uint64_t nch = 0, nf = 0;
    size_t i = 0;
    int p4 = 0;
    for (; i + lanes <= m; i += lanes) {
        carry = dotor_chunk(sub, out + i, a + i, b + i, carry, lanes, &p4);
        ++nch;
        nf += (uint64_t)p4;
    }
    if (i < m) {
        carry = dotor_chunk(sub, out + i, a + i, b + i, carry, (unsigned)(m - i), &p4);
        ++nch;
        nf += (uint64_t)p4;
    }
    if (chunks) *chunks += nch;
    if (fires) *fires += nf;
    return carry;
}

/* mul.cpp:12-103 at k = 64 (kSaturated). The gather order (column c ascending, i
 * ascending, mul.cpp:24-33) only fixes evaluation order; columns are u128 sums of
 * low halves in c and high halves in c+1 (mul.cpp:54-68); the carry pass folds a
 * wrapped 128-bit add back in at weight 2^64 (mul.cpp:70-90). */
void dotor_mul_columns(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m) {
    const size_t ncol = 2 * m;
    u128 col_buf[512];
    u128* col = col_buf;
    u128* heap = 0;
    if (ncol > 512) {
        heap = (u128*)malloc(sizeof(u128) * ncol);
        col = heap;
    }
    for (size_t c = 0; c < ncol; ++c) col[c] = 0;
    for (size_t c = 0; c + 1 < ncol; ++c) {
        const size_t i_lo = c + 1 >= m ? c + 1 - m : 0;
        const size_t i_hi = c < m - 1 ? c : m - 1;
        for (size_t i = i_lo; i <= i_hi; ++i) {
            const u128 p = (u128)a[i] * b[c - i];
            col[c] += (uint64_t)p;
            col[c + 1] += (uint64_t)(p >> 64);
        }
    }
    u128 carry = 0;
    for (size_t c = 0; c < ncol; ++c) {
        const u128 v = col[c] + carry;
        const u128 wrapped = v < col[c] ? ((u128)1 << 64) : 0;
        out[c] = (uint64_t)v;
        carry = (v >> 64) + wrapped;
    }
    if (heap) {
        free(heap);
    }
}

/* limbs.cpp:46-53 */
int dotor_compare(const uint64_t* a, size_t ma, const uint64_t* b, size_t mb) {
    const size_t na = sig_limbs(a, ma), nb = sig_limbs(b, mb);
    if (na != nb) return na < nb ? -1 : 1;
    for (size_t i = na; i-- > 0;)
        if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
}

void dotor_addsub_batch(int op, uint64_t* out, const uint64_t* a, const uint64_t* b,
                        uint32_t* flags, size_t m, size_t batch) {
    for (size_t p = 0; p < batch; ++p) {
        const size_t o = p * m;
        flags[p] = op ? dotor_sub(out + o, a + o, b + o, m) : dotor_add(out + o, a + o, b + o, m);
    }
}

void dotor_mul_batch(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch) {
    for (size_t p = 0; p < batch; ++p) {
        uint64_t* o = out + p * 2 * m;
        if (m == 0) continue;
        (void)dotor_mul(o, a + p * m, m, b + p * m, m);
    }
}

static uint64_t splitmix64_at(uint64_t seed, uint64_t k) {
    uint64_t z = seed + k * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

void dotor_fill_splitmix64(uint64_t* out, size_t n, uint64_t seed, uint64_t offset) {
    for (size_t i = 0; i < n; ++i) out[i] = splitmix64_at(seed, offset + i + 1);
}

/* dot_mul_words at k = 52 (RadixConfig kUnsaturated; mul.cpp:38-90): low halves of every
 * 52x52-bit product into column c, high halves (>> 52) into c + 1, carry pass in radix
 * 2^52. Writes exactly 2m limbs, each < 2^52. Inputs must be < 2^52 (caller checks). */
void dotor_mul_columns52(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m) {
    const uint64_t mask = ((uint64_t)1 << 52) - 1;
    const size_t ncol = 2 * m;
    u128* col = (u128*)calloc(ncol, sizeof(u128));
    for (size_t i = 0; i < m; ++i)
        for (size_t j = 0; j < m; ++j) {
            const u128 p = (u128)a[i] * b[j];
            col[i + j] += (uint64_t)p & mask;
            col[i + j + 1] += (uint64_t)(p >> 52);
        }
    u128 carry = 0;
    for (size_t c = 0; c < ncol; ++c) {
        const u128 v = col[c] + carry;
        out[c] = (uint64_t)v & mask;
        carry = v >> 52;
    }
    free(col);
}

/* ---- the column pipeline as separate stages (mul.hpp:32-67, mul.cpp:12-90) ---- */

/* gather_columns (mul.cpp:12-36): column order, c ascending, i ascending. */
size_t dotor_gather_columns(uint64_t* m_a, uint64_t* m_b, const uint64_t* a, const uint64_t* b, size_t m) {
    size_t t = 0;
    for (size_t c = 0; c + 1 < 2 * m; ++c) {
        const size_t i_lo = c + 1 >= m ? c + 1 - m : 0;
        const size_t i_hi = c < m - 1 ? c : m - 1;
        for (size_t i = i_lo; i <= i_hi; ++i, ++t) {
            m_a[t] = a[i];
            m_b[t] = b[c - i];
        }
    }
    return t;
}

/* compute_partials (mul.cpp:38-52): split each product at bit k (k = 64 or 52). */
void dotor_compute_partials(uint64_t* p_lo, uint64_t* p_hi, const uint64_t* m_a, const uint64_t* m_b, size_t n,
                            unsigned k) {
    const uint64_t mask = k >= 64 ? ~(uint64_t)0 : (((uint64_t)1 << k) - 1);
    for (size_t t = 0; t < n; ++t) {
        const u128 p = (u128)m_a[t] * m_b[t];
        p_lo[t] = (uint64_t)p & mask;
        p_hi[t] = (uint64_t)(p >> k);
    }
}

/* align_and_reduce (mul.cpp:54-68): 2m u128 column sums as (low, high) word pairs. */
void dotor_align_and_reduce(uint64_t* columns, const uint64_t* p_lo, const uint64_t* p_hi, size_t m) {
    u128* col = (u128*)calloc(2 * m, sizeof(u128));
    size_t t = 0;
    for (size_t c = 0; c + 1 < 2 * m; ++c) {
        const size_t lo = c + 1 >= m ? c + 1 - m : 0, hi = c < m - 1 ? c : m - 1;
        for (size_t i = lo; i <= hi; ++i, ++t) {
            col[c] += p_lo[t];
            col[c + 1] += p_hi[t];
        }
    }
    for (size_t c = 0; c < 2 * m; ++c) {
        columns[2 * c] = (uint64_t)col[c];
        columns[2 * c + 1] = (uint64_t)(col[c] >> 64);
    }
    free(col);
}

/* carry_pass (mul.cpp:70-90): serial renormalisation to base 2^k with the 128-bit wrap
 * fold, then residual limbs. out holds ncols + 3 limbs; returns the limbs written. */
size_t dotor_carry_pass(uint64_t* out, const uint64_t* columns, size_t ncols, unsigned k) {
    const uint64_t mask = k >= 64 ? ~(uint64_t)0 : (((uint64_t)1 << k) - 1);
    u128 carry = 0;
    size_t n = 0;
    for (size_t c = 0; c < ncols; ++c) {
        const u128 col = ((u128)columns[2 * c + 1] << 64) | columns[2 * c];
        const u128 v = col + carry;
        const u128 wrapped = v < col ? ((u128)1 << (128 - k)) : 0;
        out[n++] = (uint64_t)v & mask;
        carry = (v >> k) + wrapped;
    }
    while (carry != 0) {
        out[n++] = (uint64_t)carry & mask;
        carry >>= k;
    }
    return n;
}
