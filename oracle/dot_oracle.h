/* dot_oracle.h - CPU restatement of the reference's limb arithmetic (TEST INFRASTRUCTURE).
 *
 * This directory is the parity checker, never the product: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load it. The product path (paper_2604_21566_b200/) never links or calls it.
 *
 * Every function restates one routine of the reference (paths relative to
 * /root/reference/proj). Parity of this restatement is pinned two ways:
 *   1. against golden vectors produced by the reference itself
 *      (tests/golden/, made by tests/golden/make_golden.py through oracle/_ref);
 *   2. directly against oracle/_ref/libdotref.so (the reference's own TUs,
 *      compiled from /root/reference by oracle/Makefile) when that library exists.
 *
 * Limbs are little-endian uint64 words, index 0 least significant (limbs.hpp:1-18).
 */
#ifndef DOT_ORACLE_H
#define DOT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* oracle_add (src/oracle.cpp:16-31): limb-serial add, returns the carry. */
unsigned dotor_add(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m);
/* oracle_sub (src/oracle.cpp:33-48): limb-serial subtract, returns the borrow. */
unsigned dotor_sub(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m);
/* oracle_mul (src/oracle.cpp:50-63): row-wise schoolbook with 128-bit intermediates.
 * Writes ma+mb limbs (zero-padded) to out and returns the trimmed length
 * (normalized(), src/limbs.cpp:40-44). Empty operand -> returns 0, writes nothing. */
size_t dotor_mul(uint64_t* out, const uint64_t* a, size_t ma, const uint64_t* b, size_t mb);

/* chunk_generic<Sub,false> (src/addsub.cpp:21-84): the four DoT phases over t lanes
 * (1 <= t <= 8). Returns the chunk carry/borrow; *phase4 = whether phase 4 fired. */
unsigned dotor_chunk(int sub, uint64_t* out, const uint64_t* a, const uint64_t* b,
                     unsigned carry_in, unsigned t, int* phase4);
/* run_words (src/addsub.cpp:136-170) over chunk_generic with `lanes` lanes per chunk
 * (lane_count(w): 8 for scalar/w8, 2, 4). Optional counters mirror AddSubStats
 * chunks_processed / phase4_triggers (addsub.hpp:53-56). out may alias a or b. */
unsigned dotor_words(int sub, uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m,
                     unsigned lanes, uint64_t* chunks, uint64_t* fires);

/* dot_mul_words (src/mul.cpp:96-103): gather_columns (12-36), compute_partials at
 * k=64 (38-52), align_and_reduce (54-68), carry_pass (70-90). Writes exactly 2m limbs. */
void dotor_mul_columns(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m);

/* dot_mul_words(a, b, kUnsaturated) (mul.cpp:38-90 at k = 52): exactly 2m limbs < 2^52. */
void dotor_mul_columns52(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m);

/* The column pipeline stage by stage (u128 columns as (low, high) uint64 pairs):
 * gather_columns (mul.cpp:12-36) -> returns m*m; compute_partials at k in {64, 52}
 * (mul.cpp:38-52); align_and_reduce (mul.cpp:54-68) -> 2m columns; carry_pass
 * (mul.cpp:70-90) over any ncols columns, out holds ncols + 3 limbs, returns the count. */
size_t dotor_gather_columns(uint64_t* m_a, uint64_t* m_b, const uint64_t* a, const uint64_t* b, size_t m);
void dotor_compute_partials(uint64_t* p_lo, uint64_t* p_hi, const uint64_t* m_a, const uint64_t* m_b, size_t n,
                            unsigned k);
void dotor_align_and_reduce(uint64_t* columns, const uint64_t* p_lo, const uint64_t* p_hi, size_t m);
size_t dotor_carry_pass(uint64_t* out, const uint64_t* columns, size_t ncols, unsigned k);

/* compare (src/limbs.cpp:46-53): -1 / 0 / +1 ignoring high zero limbs. */
int dotor_compare(const uint64_t* a, size_t ma, const uint64_t* b, size_t mb);

/* Batched row-major helpers ([batch][m] operands, flags[batch]); loops over the
 * functions above, for fast parity checking from Python. op: 0 add, 1 sub. */
void dotor_addsub_batch(int op, uint64_t* out, const uint64_t* a, const uint64_t* b,
                        uint32_t* flags, size_t m, size_t batch);
/* [batch][m] x [batch][m] -> [batch][2m] via dotor_mul (zero-padded to 2m). */
void dotor_mul_batch(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch);

/* Seeded input generator shared with the device (dotg_fill_splitmix64 in the product
 * library): out[i] = splitmix64 output for counter (offset + i + 1). Not part of the
 * reference; it only makes multi-GiB inputs reproducible on host and device. */
void dotor_fill_splitmix64(uint64_t* out, size_t n, uint64_t seed, uint64_t offset);

#ifdef __cplusplus
}
#endif

#endif
