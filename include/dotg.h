/* dotg.h - C ABI of the B200 (sm_100a) limb-arithmetic path.
 *
 * This is the drop-in boundary for the reference's hot path (DigitsOnTurbo,
 * /root/reference/proj). The reference exposes C++ only; each entry point below
 * names the reference interface it replaces (file:line under proj/). Nothing here
 * throws: every function returns a dotg_status and dotg_last_error() describes the
 * last failure on the calling thread. There is no CPU fallback: without a usable
 * sm_100 device every compute entry point returns DOTG_ECUDA.
 *
 * Data model (include/dot/limbs.hpp:1-31): a number is m little-endian uint64 limbs,
 * index 0 least significant. Flags are uint32 0/1 of weight 2^(64m).
 *
 * Pointer conventions:
 *   *_batch / *_words  : DEVICE pointers, stream-ordered on `stream` (a cudaStream_t,
 *                        NULL = legacy default stream). Returns once enqueued.
 *   *_host             : HOST pointers (pinned or pageable). The call stages through
 *                        device memory with copy/compute overlap and returns after the
 *                        results are back in host memory (synchronous, like the
 *                        reference's span forms).
 *
 * Aliasing (addsub.hpp:95-97): out may alias a or b exactly; partial overlap is
 * rejected with DOTG_EINVAL (the reference leaves it undefined).
 *
 * Layouts for batches of independent pairs:
 *   DOTG_ROW_MAJOR    pair p, limb i at [p*m + i]     (the reference's Limbs, back to back)
 *   DOTG_INTERLEAVED  pair p, limb i at [i*batch + p] (batch-interleaved, north star)
 */
#ifndef DOTG_H
#define DOTG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    DOTG_OK = 0,
    DOTG_EINVAL = 1,  /* std::invalid_argument in the reference */
    DOTG_ECUDA = 2,   /* CUDA runtime error / no sm_100 device */
    DOTG_ENOMEM = 3,  /* device or host allocation failed */
    DOTG_ENOTSUP = 4, /* argument combination not supported */
    DOTG_ENCCL = 5    /* NCCL missing or a collective failed (sharded entry points) */
} dotg_status;

typedef enum { DOTG_ROW_MAJOR = 0, DOTG_INTERLEAVED = 1 } dotg_layout;

typedef void* dotg_stream_t; /* cudaStream_t */

/* Reference: Width selector (addsub.hpp:30-36). Accepted for drop-in validation
 * (0 scalar, 2, 4, 8); the device path has one kernel family, results are identical. */
int dotg_validate_width(int width);

const char* dotg_last_error(void);
const char* dotg_version(void);
/* Number of SMs of the current device, or -1. Loads the CUDA runtime. */
int dotg_device_sms(void);

/* ---------------------------------------------------------------------------
 * Batched add/sub of independent pairs.
 * Replaces: a loop of dot_add_words / dot_sub_words span calls
 *   (addsub.hpp:98-103, addsub.cpp:286-294 -> run_words 136-170), one per pair, as in
 *   the reference bench's exec_case (bench.cpp:95-104).
 * out[p] = a[p] +/- b[p] mod 2^(64m); flags[p] = carry/borrow (flags may be NULL).
 * m = 0 is legal: flags are set to 0 (addsub.cpp:139-170 with m = 0).
 * ------------------------------------------------------------------------- */
int dotg_add_batch(uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags,
                   size_t m, size_t batch, int layout, dotg_stream_t stream);
int dotg_sub_batch(uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags,
                   size_t m, size_t batch, int layout, dotg_stream_t stream);
/* Row-pitched form (the stride_limbs of SURVEY.md §8(b)): pair p's limb i at
 * a[p * lda + i], b[p * ldb + i], out[p * ldo + i] (pitches in limbs, >= m when
 * batch > 1), so callers can pass views of wider arrays without a copy. Pitches equal to m
 * take the dense kernels; other pitches run a thread per pair. out may alias a or b
 * exactly (same pointer and pitch). */
int dotg_addsub_batch_strided(int sub, uint64_t* out, size_t ldo, const uint64_t* a, size_t lda, const uint64_t* b,
                              size_t ldb, uint32_t* flags, size_t m, size_t batch, dotg_stream_t stream);
/* Row-pitched multiply: a[p * lda + i], b[p * ldb + i], out[p * ldo + k] (k < 2m); pitches
 * in limbs (lda, ldb >= m and ldo >= 2m when batch > 1). Non-dense pitches gather the rows
 * into scratch and scatter the product (two extra passes). out must not overlap a or b. */
int dotg_mul_batch_strided(uint64_t* out, size_t ldo, const uint64_t* a, size_t lda, const uint64_t* b, size_t ldb,
                           size_t m, size_t batch, dotg_stream_t stream);

/* ---------------------------------------------------------------------------
 * Grouped batched add/sub: up to any number of INDEPENDENT problems (sizes may differ)
 * in as few launches as possible - one persistent launch for every row-major,
 * power-of-two m <= 256 problem (up to 32 per launch). No problem's out may overlap
 * another problem's operands or output. Replaces a loop of span calls over pairs of
 * several sizes (e.g. the reference corpus sweep, testgen.cpp:61-66 sizes).
 * ------------------------------------------------------------------------- */
typedef struct {
    int op;          /* 0 add, 1 sub */
    int layout;      /* dotg_layout */
    uint64_t* out;
    const uint64_t* a;
    const uint64_t* b;
    uint32_t* flags; /* may be NULL */
    size_t m;
    size_t batch;
} dotg_addsub_problem;
int dotg_addsub_grouped(const dotg_addsub_problem* problems, int n, dotg_stream_t stream);

/* ---------------------------------------------------------------------------
 * Batched column multiplication.
 * Replaces: dot_mul_words(a, b, kSaturated, w) per pair (mul.hpp:75-76, mul.cpp:96-103).
 * out[p] = a[p] * b[p], exactly 2m limbs (high limbs may be 0). Requires
 * 1 <= m <= 2^24 (kMaxMulLimbs, mul.hpp:30; mul.cpp:13-18). ROW_MAJOR out is
 * [batch][2m]; INTERLEAVED out is [2m][batch].
 * ------------------------------------------------------------------------- */
int dotg_mul_batch(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                   int layout, dotg_stream_t stream);

/* Which pipe dotg_mul_batch (and everything built on it) takes the partial products on.
 * AUTO (row-major): m <= 16 on the IMAD column kernels (exact-size register kernels for
 * m = 3 ... 15 off the powers of two); m in {20, 24, 28, 32, 48, 64, 80, 96, 112, 128} on
 * the integer tensor pipe (radix-2^8 IMMA column sums), other 16 < m < 128 zero-extended
 * to the next of those (odd rows loaded directly, even rows through the bulk-copy ring);
 * 128 < m < 256 as one Karatsuba level over 80 / 96 / 112 / 128-limb tensor-pipe leaves;
 * 256 <= m <= 65536 on the 5th-generation tensor core (tcgen05.mma kind::i8, column sums
 * in tensor memory; rows padded to a multiple of 16 limbs); m > 65536 as padded Karatsuba
 * down to tcgen05 leaves (environment: DOTG_MUL_UMMA=0 keeps the mma.sync leaves,
 * DOTG_UMMA_LEAF / DOTG_UMMA_DIRECT pick the leaf size and the direct limit).
 * Interleaved: m <= 16 on register kernels in place, 16 < m <= 128 on the tensor pipe in
 * place, larger m transposed around the row-major route.
 * IMMA also covers m in {8, 16} (slower there than IMAD; taken only when forced).
 * IMAD / IMMA force one side where it applies (IMMA falls back to IMAD for shapes it
 * does not cover). Both are bit-exact; the knob exists for A/B measurement and for
 * parity tests of both kernels. Process-wide. Returns the previous route (>= 0), or
 * -DOTG_EINVAL (negative, distinct from every route) for an unknown value. */
#define DOTG_MUL_AUTO 0
#define DOTG_MUL_IMAD 1
#define DOTG_MUL_IMMA 2
int dotg_set_mul_route(int route);

/* Unsaturated 52-bit radix (RadixConfig kUnsaturated): dot_mul_words(a, b, kUnsaturated)
 * and dot_mul_5x5 (mul.hpp:73-85, mul.cpp:38-90, 127-150). Host row-major arrays; every
 * limb must be < 2^52 (check_limbs, limbs.cpp:26-33 -> DOTG_EINVAL); exactly 2m output
 * limbs, each < 2^52. */
int dotg_mul52_batch_host(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch);
/* Device-pointer form (stream-ordered): the caller guarantees every limb < 2^52 (the host
 * form above validates them like check_limbs); a wider limb yields an unspecified
 * product. Row-major [batch][m] -> [batch][2m]. */
int dotg_mul52_batch(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                     dotg_stream_t stream);

/* ---------------------------------------------------------------------------
 * Batched Karatsuba (reference karatsuba_mul / kara_rec, mul.hpp:87-102,
 * mul.cpp:161-233): equal-length row-major pairs, exactly 2m output limbs, recursion
 * until m <= theta (theta >= 1), odd levels zero-padded, base case = the column multiply
 * (bit-identical to dot_mul_4x4 / dot_mul_words). Breadth-first on the device: one
 * batched launch per recursion level. Scratch from the stream-ordered allocator.
 * ------------------------------------------------------------------------- */
int dotg_karatsuba_batch(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                         size_t theta, dotg_stream_t stream);
int dotg_karatsuba_batch_host(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                              size_t theta);

/* ---------------------------------------------------------------------------
 * One long number on one GPU (config 5 at G = 1, and the span form at any m).
 * Replaces: dot_add_words / dot_sub_words span form (addsub.hpp:98-103).
 * carry_out is a DEVICE pointer to one uint32 (may be NULL). Scratch is taken from
 * the stream-ordered allocator of `stream`'s device.
 * ------------------------------------------------------------------------- */
int dotg_add_words(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m,
                   uint32_t* carry_out, dotg_stream_t stream);
int dotg_sub_words(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m,
                   uint32_t* carry_out, dotg_stream_t stream);

/* ---------------------------------------------------------------------------
 * One long number sharded by limb range across ranks (config 5, G > 1).
 * Each rank holds limbs [r*n/G, (r+1)*n/G) of a, b, out and calls:
 *   1. dotg_shard_local   - streaming pass over the shard with an unknown carry-in X;
 *                           writes every output limb that does not depend on X and the
 *                           shard aggregate agg[0..1] = {G, P} (device uint32[2]):
 *                           G = carry-out if X = 0, P = 1 iff every limb propagates.
 *   2. exchange agg across ranks (8 bytes per rank; e.g. ncclAllGather / torch
 *      all_gather_into_tensor) into all_aggs = uint32[world][2] on the device.
 *   3. dotg_shard_finish  - carry-in X_r = exclusive scan of (G, P) over ranks < r,
 *                           then the boundary fix-up; carry_out (device uint32, may be
 *                           NULL) receives the carry of the WHOLE number (rank-independent).
 * `state` is a device scratch of dotg_shard_state_bytes(m) bytes that must stay alive
 * between the two calls. Single GPU: world = 1 with all_aggs = agg.
 * ------------------------------------------------------------------------- */
size_t dotg_shard_state_bytes(size_t m);
int dotg_shard_local(int sub, uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m,
                     void* state, uint32_t* agg, dotg_stream_t stream);
int dotg_shard_finish(int sub, uint64_t* out, size_t m, void* state, const uint32_t* all_aggs,
                      int rank, int world, uint32_t* carry_out, dotg_stream_t stream);

/* ---------------------------------------------------------------------------
 * The same protocol driven from C++ in one call per rank (SURVEY.md §8(b)
 * dotg_add_words_sharded; §8(e)). Replaces: the serial chunk chain of one long number,
 * dot_add_words / dot_sub_words span form over m limbs (addsub.cpp:136-170, 286-294),
 * when the number's limbs are spread over the GPUs of one node.
 *   dotg_add_words_sharded(out, a, b, m_local, carry_out, comm, stream)
 * enqueues on `stream`: dotg_shard_local -> ncclAllGather of the 8-byte {G, P} -> the
 * boundary fix-up; no host synchronisation (CUDA-graph capturable). out/a/b are this
 * rank's m_local limbs (rank order = limb order, any split, m_local = 0 allowed);
 * carry_out (device uint32, may be NULL) receives the carry/borrow of the WHOLE number.
 * A dotg_comm wraps an NCCL communicator: created here from an NCCL unique id (rank 0
 * calls dotg_comm_get_unique_id and the caller broadcasts the dotg_comm_id_bytes()
 * bytes by any means), or wrapped around a caller-owned ncclComm_t (dotg_comm_wrap; not
 * destroyed by dotg_comm_destroy). NCCL is loaded at run time; without it these calls
 * return DOTG_ENCCL. The current device must be the communicator's device.
 * ------------------------------------------------------------------------- */
typedef struct dotg_comm dotg_comm;
size_t dotg_comm_id_bytes(void);
int dotg_comm_get_unique_id(void* id);
int dotg_comm_init_rank(dotg_comm** comm, int world, const void* id, int rank);
int dotg_comm_wrap(dotg_comm** comm, void* nccl_comm);
int dotg_comm_destroy(dotg_comm* comm);
int dotg_comm_rank(const dotg_comm* comm);
int dotg_comm_size(const dotg_comm* comm);
int dotg_add_words_sharded(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m_local,
                           uint32_t* carry_out, const dotg_comm* comm, dotg_stream_t stream);
int dotg_sub_words_sharded(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m_local,
                           uint32_t* carry_out, const dotg_comm* comm, dotg_stream_t stream);

/* ---------------------------------------------------------------------------
 * Host-buffer entry points (the reference-facing call: host spans in, host out).
 * Replace: dot_add_words / dot_sub_words span forms (addsub.hpp:98-103) and
 * dot_mul_words (mul.hpp:75-76) over a batch of row-major host arrays. Inputs are
 * streamed to the device in slices on two streams so host->device copies, kernels
 * and device->host copies overlap; the call returns when out/flags are filled.
 * Pinned host memory (cudaHostAlloc) reaches full PCIe bandwidth.
 * ------------------------------------------------------------------------- */
int dotg_add_batch_host(uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags,
                        size_t m, size_t batch);
int dotg_sub_batch_host(uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags,
                        size_t m, size_t batch);
int dotg_mul_batch_host(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m,
                        size_t batch);
/* Several independent row-major problems through ONE copy/compute pipeline (no drain
 * between problems); host pointers; layout must be DOTG_ROW_MAJOR. */
int dotg_addsub_grouped_host(const dotg_addsub_problem* problems, int n);
/* Single number, host spans (the literal span form). *carry receives the flag. */
int dotg_add_words_host(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m,
                        uint32_t* carry);
int dotg_sub_words_host(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m,
                        uint32_t* carry);

/* ---------------------------------------------------------------------------
 * Instrumentation parity with AddSubStats (addsub.hpp:53-72): after out = a +/- b has
 * been computed, counts the reference's w-limb chunks (w = lane_count(width): 8 for
 * scalar/w8, 2, 4) and how many of them would have taken the rare Phase 4
 * (addsub.cpp:48-79). Derived on the device from a, b and out; off the hot path.
 * counters: DEVICE uint64[2] {chunks_processed, phase4_triggers}, ACCUMULATED into.
 * ------------------------------------------------------------------------- */
int dotg_addsub_stats(int sub, const uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m,
                      size_t batch, int layout, int width, uint64_t* counters, dotg_stream_t stream);
/* Span form with stats on host spans: out = a +/- b (m limbs), *carry = flag and the two
 * counters ADDED to *chunks / *fires (AddSubStats semantics). */
int dotg_words_host_stats(int sub, uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m,
                          int width, uint32_t* carry, uint64_t* chunks, uint64_t* fires);

/* Phase ticks (AddSubStats::collect_ticks, addsub.hpp:57-63; the reference's PhaseTimer
 * laps, kernels.hpp:20-37, and the phase-% / carry-to-add pass of bench.cpp:227-247):
 * runs the batched add/sub with per-phase %clock64 laps compiled into the same team
 * kernel and ADDS SM-clock cycles, summed over warps, into ticks[6] in AddSubStats order
 * {load, add, carry_gen, carry_add, store, overflow} (overflow stays 0: cascades are
 * resolved by the same mask addition as every other carry). out/flags are computed as by
 * dotg_add_batch / dotg_sub_batch. Row-major, power-of-two m <= 256 (else DOTG_ENOTSUP).
 * Device form: device pointers, ticks a device uint64[6]. Host form: host arrays, ticks a
 * host uint64[6]. Off the hot path (the laps serialise each warp's phases). */
int dotg_addsub_phase_ticks(int sub, uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags, size_t m,
                            size_t batch, uint64_t* ticks, dotg_stream_t stream);
int dotg_addsub_phase_ticks_host(int sub, uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags,
                                 size_t m, size_t batch, uint64_t* ticks);

/* ---------------------------------------------------------------------------
 * Batched comparison. Replaces: compare(a, b) per pair (limbs.hpp:84, limbs.cpp:46-53),
 * the a >= b check of the sub configs. out[p] = -1 / 0 / +1 for a[p] < = > b[p] (equal
 * lengths: the first difference from the top). Device pointers, stream-ordered.
 * ------------------------------------------------------------------------- */
int dotg_compare_batch(int32_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch, int layout,
                       dotg_stream_t stream);
/* Host-memory form (row-major), backing the C++ drop-in's compare(a, b) (which zero-pads
 * unequal lengths first: high zero limbs do not change the order, limbs.cpp:46-53). */
int dotg_compare_host(int32_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch);

/* ---------------------------------------------------------------------------
 * Chunk-level operations. Replaces: add_w_limbs / sub_w_limbs (addsub.hpp:78-89,
 * addsub.cpp:172-190). One chunk = w limbs, 1 <= w <= 8 (the reference's masked-tail form
 * for w < 8). Batched device form: chunk p at a/b/sums + p*w, carry_in[p] (NULL = all 0),
 * carry_out[p], phase4_fired[p] (NULL = not wanted; 1 iff the reference's Phase 4 fires
 * for that chunk). A carry_in entry > 1 (the reference throws) sets carry_out[p] to
 * 0xFFFFFFFF and leaves that chunk's sums unwritten. sums may alias a or b exactly.
 * Host form: one chunk from host memory, carry_in > 1 is DOTG_EINVAL.
 * ------------------------------------------------------------------------- */
int dotg_chunk_batch(int sub, uint64_t* sums, uint32_t* carry_out, uint32_t* phase4_fired, const uint64_t* a,
                     const uint64_t* b, const uint32_t* carry_in, unsigned w, size_t batch, dotg_stream_t stream);
int dotg_chunk_host(int sub, uint64_t* sums, uint32_t* carry_out, uint32_t* phase4_fired, const uint64_t* a,
                    const uint64_t* b, uint32_t carry_in, unsigned w);

/* ---------------------------------------------------------------------------
 * The column pipeline as separate stages. Replaces: gather_columns, compute_partials,
 * align_and_reduce, carry_pass (mul.hpp:32-67, mul.cpp:12-90) - the stages dot_mul_words
 * chains (mul.cpp:96-103; dotg_mul_batch fuses them). Same buffers, bit for bit:
 *   gather:   m_a / m_b [batch][m*m] in column order (i + j ascending, i ascending);
 *             1 <= m <= 2^24 (m*m buffers: device memory bounds it far lower).
 *   partials: p_lo = (m_a*m_b) mod 2^k, p_hi = floor(m_a*m_b / 2^k) truncated to 64 bits,
 *             limb_bits k in {64, 52} (n entries, any grouping).
 *   reduce:   columns [batch][2m] u128 sums as (low 64, high 64) pairs of uint64.
 *   carry:    out [batch][out_cap] limbs, out_limbs[p] = limbs written (ncols plus a
 *             residual of at most 2): out_cap >= ncols + 2.
 * Host forms (one operand set, host pointers) back the C++ drop-in.
 * ------------------------------------------------------------------------- */
int dotg_gather_columns(uint64_t* m_a, uint64_t* m_b, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                        dotg_stream_t stream);
int dotg_compute_partials(uint64_t* p_lo, uint64_t* p_hi, const uint64_t* m_a, const uint64_t* m_b, size_t n,
                          int limb_bits, dotg_stream_t stream);
int dotg_align_and_reduce(uint64_t* columns, const uint64_t* p_lo, const uint64_t* p_hi, size_t m, size_t batch,
                          dotg_stream_t stream);
int dotg_carry_pass(uint64_t* out, uint32_t* out_limbs, size_t out_cap, const uint64_t* columns, size_t ncols,
                    size_t batch, int limb_bits, dotg_stream_t stream);
int dotg_gather_columns_host(uint64_t* m_a, uint64_t* m_b, const uint64_t* a, const uint64_t* b, size_t m);
int dotg_compute_partials_host(uint64_t* p_lo, uint64_t* p_hi, const uint64_t* m_a, const uint64_t* m_b, size_t n,
                               int limb_bits);
int dotg_align_and_reduce_host(uint64_t* columns, const uint64_t* p_lo, const uint64_t* p_hi, size_t m);
int dotg_carry_pass_host(uint64_t* out, uint32_t* out_limbs, size_t out_cap, const uint64_t* columns, size_t ncols,
                         int limb_bits);

/* ---------------------------------------------------------------------------
 * Carry statistics (acceptance criterion 4, acceptance.cpp:157-170). Replaces:
 * carry_census(k) (oracle.cpp:65-78): counts[0] = pairs (x, y) in [0, 2^k)^2 with
 * x + y = 2^k - 1, counts[1] = pairs with x + y >= 2^k, 1 <= k <= 16 (exhaustive, on the
 * device); and run_stats' Monte-Carlo carry frequency (bench.cpp:278-287): *carries =
 * carry-outs of `samples` random 64-bit additions (splitmix64 stream of `seed`).
 * Host pointers; synchronous.
 * ------------------------------------------------------------------------- */
int dotg_carry_census(unsigned k, uint64_t* counts);
int dotg_mc_carry(uint64_t samples, uint64_t seed, uint64_t* carries);

/* Workload setup (not the hot path): out[i] = splitmix64 output for counter
 * offset + i + 1 (device pointer, stream-ordered). Host twin: oracle/dot_oracle.c. */
int dotg_fill_splitmix64(uint64_t* out, size_t n, uint64_t seed, uint64_t offset,
                         dotg_stream_t stream);

/* Diagnostics: number of kernels this library launched since load (all threads). */
uint64_t dotg_kernel_launches(void);

#ifdef __cplusplus
}
#endif

#endif /* DOTG_H */
