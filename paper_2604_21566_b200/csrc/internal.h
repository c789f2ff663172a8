// internal.h - launcher declarations shared between the kernel TUs and the C ABI.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstddef>
#include <cstdint>
#include <string>

namespace dotg {

// Launch counter reported by dotg_kernel_launches() (diagnostics for the bench's
// gpu_launches claim).
extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// One independent batched add/sub problem as the grouped kernel sees it.
struct AddSubProblem {
    uint64_t* out;
    const uint64_t* a;
    const uint64_t* b;
    uint32_t* flags;
    uint64_t batch;
    uint64_t task_begin;  // first warp task of this problem in the group's task space
    uint32_t m;
    uint32_t sub;
};
constexpr int kMaxGroup = 32;
struct AddSubGroup {  // passed by value as a __grid_constant__ kernel parameter
    uint64_t total_tasks;
    int n;
    AddSubProblem p[kMaxGroup];
};

// Grouped batched add/sub: every problem independent; layouts[i] per problem.
cudaError_t launch_addsub_group(const AddSubProblem* probs, const int* layouts, int n, cudaStream_t stream);

// Batched add/sub with the phase-tick laps compiled in (row-major, power-of-two m <= 256):
// ticks = device uint64[6] {load, add, carry_gen, carry_add, store, overflow}, accumulated.
cudaError_t launch_addsub_timed(bool sub, uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags,
                                size_t m, size_t batch, uint64_t* ticks, cudaStream_t st);

// Batched add/sub. layout 0 = row-major [batch][m], 1 = interleaved [m][batch].
cudaError_t launch_addsub_batch(bool sub, uint64_t* out, const uint64_t* a, const uint64_t* b,
                                uint32_t* flags, size_t m, size_t batch, int layout,
                                cudaStream_t stream);

// Long-number (tiled) add/sub, shard-capable. See addsub_long.cu.
size_t long_state_bytes(size_t m);
cudaError_t launch_long_local(bool sub, uint64_t* out, const uint64_t* a, const uint64_t* b,
                              size_t m, void* state, uint32_t* agg, cudaStream_t stream);
cudaError_t launch_long_finish(bool sub, uint64_t* out, size_t m, void* state,
                               const uint32_t* all_aggs, int rank, int world,
                               uint32_t* carry_out, cudaStream_t stream);

// Empty shard aggregate {0, 1}; whole-number carry from gathered aggregates (comm.cu).
cudaError_t launch_shard_identity(uint32_t* agg, cudaStream_t stream);
cudaError_t launch_compose_aggs(const uint32_t* all_aggs, int world, uint32_t* carry_out, cudaStream_t stream);

// Shared C-ABI helpers (capi.cu): set dotg_last_error and return code; the sm_100 check;
// the span-form argument checks of one long add/sub (null operands, partial aliasing).
int api_fail(int code, const std::string& msg);
int api_check_device();
int api_check_addsub_words(const uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m);

// A batch of long numbers (row-major, m >= 1 tile): the tiled passes with grid.y = number.
cudaError_t launch_addsub_pitched(bool sub, uint64_t* out, size_t ldo, const uint64_t* a, size_t lda,
                                  const uint64_t* b, size_t ldb, uint32_t* flags, size_t m, size_t batch,
                                  cudaStream_t stream);
cudaError_t launch_mul_pitched(uint64_t* out, size_t ldo, const uint64_t* a, size_t lda, const uint64_t* b,
                               size_t ldb, size_t m, size_t batch, cudaStream_t st);
cudaError_t launch_long_batch(bool sub, uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags,
                              size_t m, size_t batch, cudaStream_t stream);

// Batched multiplication (exactly 2m output limbs per pair).
cudaError_t launch_mul_batch(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m,
                             size_t batch, int layout, cudaStream_t stream);

// Integer tensor-pipe column multiply (mul_imma.cu), row-major, m in {8,16,32,64}.
bool mul_imma_supported(size_t m);
cudaError_t launch_mul_imma(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                            cudaStream_t st);
// Even 16 < m < 128, 16-byte aligned rows: zero-extended to the next tensor-pipe size.
cudaError_t launch_mul_imma_rt(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                               cudaStream_t st);
// Interleaved [m][batch] operands / product in place: even 16 < m <= 128.
cudaError_t launch_mul_imma_il(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                               cudaStream_t st);
// Wide operands on the 5th-generation tensor core (mul_umma.cu): row-major, 16-byte
// aligned rows, 256 <= m <= 16384, m % 16 == 0 (DOTG_MUL_UMMA=0 disables the route).
bool mul_umma_supported(size_t m);
cudaError_t launch_mul_umma(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                            cudaStream_t st);
// Karatsuba leaf size above the direct tcgen05 range for a batch of m-limb products
// (DOTG_UMMA_LEAF overrides; by batch x m: 65536 up to 2^17 limbs, 16384 up to 2^18, 4096).
size_t mul_umma_leaf(size_t m, size_t batch);
// Largest m taken directly (DOTG_UMMA_DIRECT, default 65536); Karatsuba above.
size_t mul_umma_direct_max();
// Route for launch_mul_batch: 0 auto, 1 IMAD only, 2 IMMA where supported.
extern std::atomic<int> g_mul_route;

// Unsaturated 52-bit radix product (row-major, limbs < 2^52, exactly 2m limbs out).
cudaError_t launch_mul52_batch(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                               cudaStream_t st);

// Breadth-first batched Karatsuba over the column multiply (karatsuba.cu).
cudaError_t launch_karatsuba_batch(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                                   size_t theta, cudaStream_t st);
// m padded to base * 2^L (base a tensor-pipe size); L = 0 pads the rows and multiplies.
cudaError_t launch_karatsuba_padded(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                                    size_t base, cudaStream_t st);
// Rows copied into aligned temporaries zero-extended to mp >= m limbs, multiplied there,
// low 2m limbs of each product kept (any alignment of out / a / b).
cudaError_t mul_padded_rows(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch, size_t mp,
                            cudaStream_t st);
// Keep freed stream-ordered scratch cached in the device pool (per host thread, device).
void retain_stream_pool();

// Batched compare (compare.cu): out[p] in {-1, 0, 1}.
cudaError_t launch_compare_batch(int32_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                                 int layout, cudaStream_t st);

// AddSubStats parity counters (stats.cu): counters = device uint64[2] {chunks, fires}.
cudaError_t launch_addsub_stats(bool sub, const uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m,
                                size_t batch, int layout, unsigned lanes, uint64_t* counters, cudaStream_t st);

// Chunk-level add_w_limbs / sub_w_limbs, batched (chunk.cu).
cudaError_t launch_chunk_batch(bool sub, uint64_t* sums, uint32_t* carry_out, uint32_t* fired, const uint64_t* a,
                               const uint64_t* b, const uint32_t* carry_in, unsigned w, size_t batch,
                               cudaStream_t st);

// The reference's column pipeline as separate stages (columns.cu).
cudaError_t launch_gather_columns(uint64_t* ma, uint64_t* mb, const uint64_t* a, const uint64_t* b, size_t m,
                                  size_t batch, cudaStream_t st);
cudaError_t launch_partials(uint64_t* plo, uint64_t* phi, const uint64_t* ma, const uint64_t* mb, size_t n,
                            unsigned k, cudaStream_t st);
cudaError_t launch_align_reduce(uint64_t* cols, const uint64_t* plo, const uint64_t* phi, size_t m, size_t batch,
                                cudaStream_t st);
cudaError_t launch_carry_pass(uint64_t* out, uint32_t* nout, size_t cap, const uint64_t* cols, size_t ncols,
                              size_t batch, unsigned k, cudaStream_t st);

// Carry statistics (run_stats / carry_census, stats.cu).
cudaError_t launch_carry_census(unsigned k, uint64_t* counts, cudaStream_t st);
cudaError_t launch_mc_carry(uint64_t samples, uint64_t seed, uint64_t* carries, cudaStream_t st);

// Workload setup: splitmix64 counter fill (util.cu).
cudaError_t launch_fill_splitmix64(uint64_t* out, size_t n, uint64_t seed, uint64_t offset, cudaStream_t st);

}  // namespace dotg
