// mul_batch.cu - batched "vertical and crosswise" (column) multiplication on sm_100a.
//
// Replaces dot_mul_words (include/dot/mul.hpp:75-76, src/mul.cpp:96-103): gather pairs
// into columns (mul.cpp:12-36), independent partial products (38-52), column
// reduction (54-68), one carry pass (70-90), exactly 2m output limbs.
//
// B200 restatement: limbs are split into 32-bit words
// (n = 2m words), every 32x32->64 partial product of a column is accumulated into a
// 96-bit column accumulator with ONE IMAD.WIDE.U32 carrying out into a predicate plus
// half an IADD3.X (ptxas fuses mad.lo.cc + madc.hi.cc + addc; measured 32 products /
// clk / SM on B200 - tools/imad_peak.cu). A column of <= n products sums below
// n * 2^64, so 96 bits cover every m up to the reference cap kMaxMulLimbs = 2^24
// (mul.hpp:26-30). The carry pass is deferred to once per column / output block: the
// accumulator's low word is final, the upper 64 bits carry into the next column.
//
// Kernels (the route per size / layout / alignment is launch_mul_batch at the bottom):
//   k_mul_regs<M>   M <= 4 and the interleaved layout: thread per pair, operands in
//                   registers, columns scanned in order.
//   k_mul_kara16    M = 16 (config 3): one in-register Karatsuba level over three
//                   16 x 16-word column products (768 instead of 1024 IMAD.WIDE).
//   k_mul_regblk<M> M = 8: registers, output blocks of 16 columns; with RT also
//                   4 < m < 16 on zero-extended operands, any alignment.
//   k_mul_imma<NB>  (mul_imma.cu) m in {32, 64, 128} and even sizes between: the integer
//                   tensor pipe - the default for those sizes (config 4).
//   padded Karatsuba (karatsuba.cu) m > 128, and copy-padded odd 16 < m < 128.
//   k_transpose_u64 interleaved m > 16: to row-major and back around the row route.
//   k_mul_smem<M>   M in {32, 64, 128} when the IMAD route is forced: persistent, thread per pair, operands staged in
//                   XOR-swizzled shared memory (2 CTAs per SM fill it) by coalesced
//                   256-bit loads, output produced in blocks
//                   of K = 16 columns: for every (output block, a-block) pair a 16x16
//                   block of products is accumulated into 16 independent column
//                   accumulators (ILP 16; triangular edge blocks skip the zero
//                   products, so exactly 4m^2 products are issued) (config 4: M = 64).
//   k_mul_strided   any m / layout: thread per pair, operands read through L1.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <cstdlib>

#include "device.cuh"
#include "internal.h"

namespace dotg {

namespace {

// acc(96) += x * y
__device__ __forceinline__ void mac(uint32_t& lo, uint32_t& mid, uint32_t& hi, uint32_t x, uint32_t y) {
    asm("mad.lo.cc.u32 %0, %3, %4, %0;\n\t"
        "madc.hi.cc.u32 %1, %3, %4, %1;\n\t"
        "addc.u32 %2, %2, 0;"
        : "+r"(lo), "+r"(mid), "+r"(hi)
        : "r"(x), "r"(y));
}

// (lo,mid,hi) += (c0,c1,c2)
__device__ __forceinline__ void add96(uint32_t& lo, uint32_t& mid, uint32_t& hi, uint32_t c0, uint32_t c1,
                                      uint32_t c2) {
    asm("add.cc.u32 %0, %0, %3;\n\t"
        "addc.cc.u32 %1, %1, %4;\n\t"
        "addc.u32 %2, %2, %5;"
        : "+r"(lo), "+r"(mid), "+r"(hi)
        : "r"(c0), "r"(c1), "r"(c2));
}

__device__ __forceinline__ uint32_t lo32(uint64_t x) { return uint32_t(x); }
__device__ __forceinline__ uint32_t hi32(uint64_t x) { return uint32_t(x >> 32); }

// ---------------------------------------------------------------------------
// M <= 16: everything in registers.
// ---------------------------------------------------------------------------
// LAYOUT 0: row-major, 1: interleaved, 2: row-major staged through shared memory (odd M:
// the CTA's 128 rows of a and b are loaded, and its products stored, as contiguous
// coalesced runs instead of per-thread strided limbs; r02: m = 5 / 7 / 9 / 11 / 13 / 15
// row-major ran 39-69 us per 2^22 limbs unstaged against 24-42 us interleaved).
template <int M, int LAYOUT>
__global__ void __launch_bounds__(128) k_mul_regs(uint64_t* out, const uint64_t* a, const uint64_t* b,
                                                  size_t batch) {
    constexpr int N = 2 * M;  // words per operand
    constexpr bool STG = LAYOUT == 2;
    __shared__ uint64_t stage[STG ? 2 * 128 * M : 1];  // a rows | b rows, later the 2M-limb products
    const size_t pidx = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t p0 = size_t(blockIdx.x) * blockDim.x;
    const int np = STG ? int(batch - p0 < 128 ? batch - p0 : 128) : 0;
    if constexpr (STG) {
        for (int e = threadIdx.x; e < np * M; e += 128) {
            stage[e] = __ldcs(a + p0 * M + e);
            stage[128 * M + e] = __ldcs(b + p0 * M + e);
        }
        __syncthreads();
    } else if (pidx >= batch) {
        return;
    }
    const bool act = pidx < batch;
    uint32_t A[N], B[N];
    if constexpr (STG) {
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const uint64_t x = act ? stage[threadIdx.x * M + i] : 0, y = act ? stage[128 * M + threadIdx.x * M + i] : 0;
            A[2 * i] = lo32(x);
            A[2 * i + 1] = hi32(x);
            B[2 * i] = lo32(y);
            B[2 * i + 1] = hi32(y);
        }
        __syncthreads();  // the operand rows are in registers: the buffer takes the products
    } else if constexpr (LAYOUT == 0 && M % 4 == 0) {
#pragma unroll
        for (int v = 0; v < M / 4; ++v) {
            uint64_t x[4], y[4];
            ld_stream<4>(a + pidx * M + 4 * v, x);
            ld_stream<4>(b + pidx * M + 4 * v, y);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                A[8 * v + 2 * k] = lo32(x[k]);
                A[8 * v + 2 * k + 1] = hi32(x[k]);
                B[8 * v + 2 * k] = lo32(y[k]);
                B[8 * v + 2 * k + 1] = hi32(y[k]);
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const size_t off = LAYOUT == 0 ? pidx * M + i : size_t(i) * batch + pidx;
            const uint64_t x = a[off], y = b[off];
            A[2 * i] = lo32(x);
            A[2 * i + 1] = hi32(x);
            B[2 * i] = lo32(y);
            B[2 * i + 1] = hi32(y);
        }
    }
    uint32_t lo = 0, mid = 0, hi = 0;
    uint64_t o[4];
    uint32_t prev = 0;
#pragma unroll
    for (int c = 0; c < 2 * N; ++c) {
        if (c < 2 * N - 1) {
#pragma unroll
            for (int i = (c - N + 1 > 0 ? c - N + 1 : 0); i <= (c < N - 1 ? c : N - 1); ++i)
                mac(lo, mid, hi, A[i], B[c - i]);
        }
        const uint32_t w = lo;
        lo = mid;
        mid = hi;
        hi = 0;
        if (c & 1) {
            const int limb = c >> 1;
            const uint64_t v = uint64_t(prev) | (uint64_t(w) << 32);
            if constexpr (STG) {
                stage[threadIdx.x * (2 * M) + limb] = v;
            } else if constexpr (LAYOUT == 0 && (2 * M) % 4 == 0) {
                o[limb & 3] = v;
                if ((limb & 3) == 3) st_stream<4>(out + pidx * (2 * M) + (limb - 3), o);
            } else {
                const size_t off = LAYOUT == 0 ? pidx * (2 * M) + limb : size_t(limb) * batch + pidx;
                out[off] = v;
            }
        } else {
            prev = w;
        }
    }
    if constexpr (STG) {
        __syncthreads();
        for (int e = threadIdx.x; e < np * 2 * M; e += 128) __stcs(out + p0 * (2 * M) + e, stage[e]);
    }
}

// ---------------------------------------------------------------------------
// M in {32, 64, 128}: shared-memory operands, K = 16 output blocks.
// ---------------------------------------------------------------------------
constexpr int kK = 16;
enum StepMode { kFull = 0, kLower = 1, kUpper = 2 };

// acc[x] += sum_u A[u] * W[K + x - u]  (W[e] = b'_{(d-1)K + e}); kLower keeps x >= u
// (d = 0: j = x - u must be >= 0), kUpper keeps x < u (d = NB: j < n).
template <int MODE, int K = kK>
__device__ __forceinline__ void mul_step(uint32_t (&acc)[K][3], const uint32_t (&A)[K],
                                         const uint32_t (&W)[2 * K]) {
#pragma unroll
    for (int u = 0; u < K; ++u) {
#pragma unroll
        for (int x = 0; x < K; ++x) {
            if (MODE == kLower && x < u) continue;
            if (MODE == kUpper && x >= u) continue;
            mac(acc[x][0], acc[x][1], acc[x][2], A[u], W[K + x - u]);
        }
    }
}

// Shared-window byte addresses (computed once per kernel from __cvta_generic_to_shared;
// converting a generic pointer per access costs an S2UR + ULEA chain on sm_100).
__device__ __forceinline__ void lds4(uint32_t addr, uint32_t& x, uint32_t& y, uint32_t& z, uint32_t& w) {
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(addr));
}
__device__ __forceinline__ void sts4(uint32_t addr, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(x), "r"(y), "r"(z), "r"(w)
                 : "memory");
}

template <int M>
struct SmemCfg {
    static constexpr int N = 2 * M;          // words per operand
    static constexpr int NB = N / kK;        // a-blocks
    static constexpr int NS = 2 * N / kK;    // output blocks
    static constexpr int CH = N / 4;         // 16-byte chunks per operand per pair
    static constexpr size_t PAIR_BYTES = size_t(2) * N * sizeof(uint32_t);
};

// Physical word offset of logical word w of pair p: 16-byte chunks XOR-swizzled by
// (p & 7) so that 8 consecutive threads reading the same logical chunk hit 8 distinct
// bank groups (conflict-free ld.shared.v4) without padding.
// Byte offset of logical word w (w % 4 == 0) of pair p.
template <int N>
__device__ __forceinline__ uint32_t swz(int p, int w) {
    return uint32_t(p * N * 4) + (uint32_t((w >> 2) ^ (p & 7)) << 4);
}

// Persistent: each CTA (blockDim.x = pairs per group) loops over groups of pairs:
// stage the group's operands (coalesced 256-bit loads -> swizzled smem), then every
// thread multiplies its pair. Groups per CTA are balanced so the last round is full.
template <int M>
__global__ void __launch_bounds__(128) k_mul_smem(uint64_t* out, const uint64_t* a, const uint64_t* b,
                                                  size_t batch) {
    using C = SmemCfg<M>;
    extern __shared__ __align__(16) uint32_t smem[];
    const int P = int(blockDim.x);
    const uint32_t sa = uint32_t(__cvta_generic_to_shared(smem));
    const uint32_t sb = sa + uint32_t(P * C::N * 4);
    const int tid = int(threadIdx.x);
    const size_t ngroups = (batch + size_t(P) - 1) / size_t(P);
    constexpr int VPP = M / 4;  // 256-bit vectors per pair per operand

    for (size_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
        const size_t p0 = g * size_t(P);
        __syncthreads();  // previous group's smem reads are done
#pragma unroll 4
        for (int v = tid; v < P * VPP; v += P) {
            const int pr = v / VPP, ch = v % VPP;
            const size_t gp = p0 + size_t(pr);
            uint64_t x[4] = {0, 0, 0, 0}, y[4] = {0, 0, 0, 0};
            if (gp < batch) {
                ld_stream<4>(a + gp * M + 4 * ch, x);
                ld_stream<4>(b + gp * M + 4 * ch, y);
            }
            sts4(sa + swz<C::N>(pr, 8 * ch), lo32(x[0]), hi32(x[0]), lo32(x[1]), hi32(x[1]));
            sts4(sa + swz<C::N>(pr, 8 * ch + 4), lo32(x[2]), hi32(x[2]), lo32(x[3]), hi32(x[3]));
            sts4(sb + swz<C::N>(pr, 8 * ch), lo32(y[0]), hi32(y[0]), lo32(y[1]), hi32(y[1]));
            sts4(sb + swz<C::N>(pr, 8 * ch + 4), lo32(y[2]), hi32(y[2]), lo32(y[3]), hi32(y[3]));
        }
        __syncthreads();

        const size_t gp = p0 + size_t(tid);
        if (gp >= batch) continue;
        uint32_t cr0 = 0, cr1 = 0, cr2 = 0;  // carry into the next output block
#pragma unroll 1
        for (int s = 0; s < C::NS; ++s) {
            uint32_t acc[kK][3];
#pragma unroll
            for (int x = 0; x < kK; ++x) acc[x][0] = acc[x][1] = acc[x][2] = 0;
            const int i_lo = s - C::NB > 0 ? s - C::NB : 0;
            const int i_hi = s < C::NB - 1 ? s : C::NB - 1;
#pragma unroll 1
            for (int I = i_lo; I <= i_hi; ++I) {
                const int d = s - I;  // 0 .. NB
                uint32_t A[kK], W[2 * kK];
#pragma unroll
                for (int q = 0; q < kK / 4; ++q)
                    lds4(sa + swz<C::N>(tid, I * kK + 4 * q), A[4 * q], A[4 * q + 1], A[4 * q + 2], A[4 * q + 3]);
                // W[e] = b'_{(d-1)K + e}; blocks outside [0, N) read as zero.
#pragma unroll
                for (int q = 0; q < 2 * kK / 4; ++q) {
                    const int j = (d - 1) * kK + 4 * q;
                    if (j >= 0 && j < C::N)
                        lds4(sb + swz<C::N>(tid, j), W[4 * q], W[4 * q + 1], W[4 * q + 2], W[4 * q + 3]);
                    else
                        W[4 * q] = W[4 * q + 1] = W[4 * q + 2] = W[4 * q + 3] = 0;
                }
                if (d == 0) mul_step<kLower>(acc, A, W);
                else if (d == C::NB) mul_step<kUpper>(acc, A, W);
                else mul_step<kFull>(acc, A, W);
            }
            // Deferred normalisation of this block: 16 columns -> 16 final words.
            uint32_t w[kK];
#pragma unroll
            for (int x = 0; x < kK; ++x) {
                add96(acc[x][0], acc[x][1], acc[x][2], cr0, cr1, cr2);
                w[x] = acc[x][0];
                cr0 = acc[x][1];
                cr1 = acc[x][2];
                cr2 = 0;
            }
            uint64_t o0[4], o1[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                o0[k] = uint64_t(w[2 * k]) | (uint64_t(w[2 * k + 1]) << 32);
                o1[k] = uint64_t(w[8 + 2 * k]) | (uint64_t(w[8 + 2 * k + 1]) << 32);
            }
            uint64_t* po = out + gp * (2 * M) + size_t(s) * (kK / 2);
            st_stream<4>(po, o0);
            st_stream<4>(po + 4, o1);
        }
    }
}

// ---------------------------------------------------------------------------
// M in {8, 16} (config 3): operands in registers, output in blocks of K = 16 columns
// with 16 independent column accumulators (ILP 16; one accumulator per column would
// leave the IMAD.WIDE carry chain latency-bound - tools/mac_sweep.cu: 1 accumulator
// tops out at ~22 products/clk/SM, 16 accumulators at ~29 of the 32 peak).
// ---------------------------------------------------------------------------
// Flat grid, one pair per thread. (Measured on B200, r01: 8-column output blocks (42.9 us,
// same), 6 / 7 CTAs per SM forced through launch bounds (80 / 72 registers with spills:
// 45.9 / 55.9 us - ncu: the FMA-heavy pipe at ~80%, stalls split between math-pipe
// throttle and fixed-latency waits), one-warp CTAs with the resident
// warps per SM capped so the batch ends just below a whole wave (43.9 us), a persistent
// loop with an exactly balanced pair range per CTA (48.2 us: the 2.77 pairs/thread
// quantisation moves into the warps as partial last iterations), a persistent thread-stride
// loop, and prefetching the next pair into L2 or into shared memory with cp.async, were
// all slower than this - 48-54 us vs 43.6 us for config 3 - and a compute-only variant
// with no loads ran at the same 43.5 us, i.e. the kernel is IMAD-issue bound, not
// memory bound: ~25.5 products/clk/SM while SMs are active.)
// RT: the pairs are mr < M limbs (rows of mr limbs, any 8-byte alignment), computed as
// M-limb products of zero-extended operands; only the 2 mr product limbs are stored.
template <int M, bool RT = false>
__global__ void __launch_bounds__(128) k_mul_regblk(uint64_t* out, const uint64_t* a, const uint64_t* b,
                                                    size_t batch, int mr = M) {
    constexpr int N = 2 * M;         // words per operand
    constexpr int NB = N / kK;       // a-blocks
    constexpr int NS = 2 * N / kK;   // output blocks
    static_assert(N % kK == 0, "M must be a multiple of 8");
    const size_t pidx = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (pidx >= batch) return;
    {
        uint32_t A[N], B[N];
        if constexpr (RT) {
#pragma unroll
            for (int i = 0; i < M; ++i) {
                const uint64_t x = i < mr ? __ldg(a + pidx * mr + i) : 0ull;
                const uint64_t y = i < mr ? __ldg(b + pidx * mr + i) : 0ull;
                A[2 * i] = lo32(x);
                A[2 * i + 1] = hi32(x);
                B[2 * i] = lo32(y);
                B[2 * i + 1] = hi32(y);
            }
        } else {
#pragma unroll
            for (int v = 0; v < M / 4; ++v) {
                uint64_t x[4], y[4];
                ld_stream<4>(a + pidx * M + 4 * v, x);
                ld_stream<4>(b + pidx * M + 4 * v, y);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    A[8 * v + 2 * k] = lo32(x[k]);
                    A[8 * v + 2 * k + 1] = hi32(x[k]);
                    B[8 * v + 2 * k] = lo32(y[k]);
                    B[8 * v + 2 * k + 1] = hi32(y[k]);
                }
            }
        }
        uint32_t cr0 = 0, cr1 = 0, cr2 = 0;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        uint32_t acc[kK][3];
#pragma unroll
        for (int x = 0; x < kK; ++x) acc[x][0] = acc[x][1] = acc[x][2] = 0;
#pragma unroll
        for (int I = 0; I < NB; ++I) {
            const int d = s - I;
            if (d < 0 || d > NB) continue;
            uint32_t Ab[kK], W[2 * kK];
#pragma unroll
            for (int u = 0; u < kK; ++u) Ab[u] = A[I * kK + u];
#pragma unroll
            for (int e = 0; e < 2 * kK; ++e) {
                const int j = (d - 1) * kK + e;
                W[e] = (j >= 0 && j < N) ? B[j < 0 ? 0 : (j >= N ? N - 1 : j)] : 0u;
            }
            if (d == 0) mul_step<kLower>(acc, Ab, W);
            else if (d == NB) mul_step<kUpper>(acc, Ab, W);
            else mul_step<kFull>(acc, Ab, W);
        }
        uint32_t w[kK];
#pragma unroll
        for (int x = 0; x < kK; ++x) {
            add96(acc[x][0], acc[x][1], acc[x][2], cr0, cr1, cr2);
            w[x] = acc[x][0];
            cr0 = acc[x][1];
            cr1 = acc[x][2];
            cr2 = 0;
        }
        uint64_t o0[4], o1[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            o0[k] = uint64_t(w[2 * k]) | (uint64_t(w[2 * k + 1]) << 32);
            o1[k] = uint64_t(w[8 + 2 * k]) | (uint64_t(w[8 + 2 * k + 1]) << 32);
        }
        if constexpr (RT) {
            uint64_t* po = out + pidx * (2 * size_t(mr));
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int limb = s * (kK / 2) + k;
                if (limb < 2 * mr) po[limb] = k < 4 ? o0[k] : o1[k - 4];
            }
        } else {
            uint64_t* po = out + pidx * (2 * M) + size_t(s) * (kK / 2);
            st_stream<4>(po, o0);
            st_stream<4>(po + 4, o1);
        }
    }
    }
}

// ---------------------------------------------------------------------------
// M = 16 (config 3) with one in-register Karatsuba level: three 16 x 16-word column
// products (768 instead of 1024 IMAD.WIDE) - z0 = lo*lo, z2 = hi*hi, z1 = |a_hi - a_lo| *
// |b_hi - b_lo| - and mid = z0 + z2 -+ z1 (reference kara_rec, mul.cpp:176-233, the
// subtractive form), recombined with 32-bit carry chains on the ALU pipe.
// ---------------------------------------------------------------------------
// Z = A * B for 16-word operands: one 16-column block below (kLower) and one above (kUpper).
template <int K>
__device__ __forceinline__ void mulK_words(const uint32_t (&A)[K], const uint32_t (&B)[K], uint32_t (&Z)[2 * K]) {
    uint32_t cr0 = 0, cr1 = 0, cr2 = 0;
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        uint32_t acc[K][3];
#pragma unroll
        for (int x = 0; x < K; ++x) acc[x][0] = acc[x][1] = acc[x][2] = 0;
        uint32_t W[2 * K];
#pragma unroll
        for (int e = 0; e < 2 * K; ++e) {
            const int j = (s - 1) * K + e;
            W[e] = (j >= 0 && j < K) ? B[j < 0 ? 0 : (j >= K ? K - 1 : j)] : 0u;
        }
        if (s == 0) mul_step<kLower, K>(acc, A, W);
        else mul_step<kUpper, K>(acc, A, W);
#pragma unroll
        for (int x = 0; x < K; ++x) {
            add96(acc[x][0], acc[x][1], acc[x][2], cr0, cr1, cr2);
            Z[s * K + x] = acc[x][0];
            cr0 = acc[x][1];
            cr1 = acc[x][2];
            cr2 = 0;
        }
    }
}

// D = |X - Y| (K words), returns X < Y.
template <int K>
__device__ __forceinline__ uint32_t absdiff(const uint32_t (&X)[K], const uint32_t (&Y)[K], uint32_t (&D)[K]) {
    uint32_t bw = 0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        const uint64_t t = uint64_t(X[i]) - uint64_t(Y[i]) - bw;
        D[i] = uint32_t(t);
        bw = uint32_t(t >> 63);
    }
    // negative: D = -D (two's complement over K words)
    const uint32_t mask = 0u - bw;
    uint32_t c = bw;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        const uint64_t t = uint64_t(D[i] ^ mask) + c;
        D[i] = uint32_t(t);
        c = uint32_t(t >> 32);
    }
    return bw;
}

// (A second Karatsuba level - nine 8 x 8-word products, 576 IMAD.WIDE - needs 168
// registers and ran 44.2 us; one level stays.)
__device__ __forceinline__ void mul16_words(const uint32_t (&A)[kK], const uint32_t (&B)[kK], uint32_t (&Z)[2 * kK]) {
    mulK_words<kK>(A, B, Z);
}
__device__ __forceinline__ uint32_t absdiff16(const uint32_t (&X)[kK], const uint32_t (&Y)[kK], uint32_t (&D)[kK]) {
    return absdiff<kK>(X, Y, D);
}

// 128 registers, 16 warps/SM. One warp per CTA (16 CTAs/SM) trims the partial last wave:
// C3 38.5 us vs 39.7 us with 128-thread CTAs (tools/k16var.sh). Capping registers for 20
// warps/SM (96 registers) spills 236 B and runs 44-46 us; uncapped, ptxas takes 186
// registers (8 warps/SM) and runs 54-56 us.
#ifndef DOTG_K16_TPB
#define DOTG_K16_TPB 32
#endif
#ifndef DOTG_K16_MINB
#define DOTG_K16_MINB 16
#endif
// IL = true: the interleaved [m][batch] layout (limb i of pair p at i * batch + p), every
// load / store coalesced across the warp's 32 consecutive pairs.
template <bool IL>
__device__ __forceinline__ void kara16_pair(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t batch,
                                            size_t pidx) {
    // output limbs [l0, l0 + 4) of this pair
    auto put4 = [&](size_t l0, const uint64_t (&o)[4]) {
        if constexpr (IL) {
#pragma unroll
            for (int k = 0; k < 4; ++k) __stcs(out + (l0 + k) * batch + pidx, o[k]);
        } else {
            st_stream<4>(out + pidx * 32 + l0, o);
        }
    };
    uint32_t Al[kK], Ah[kK], Bl[kK], Bh[kK];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
        uint64_t x[4], y[4];
        if constexpr (IL) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                x[k] = __ldcs(a + size_t(4 * v + k) * batch + pidx);
                y[k] = __ldcs(b + size_t(4 * v + k) * batch + pidx);
            }
        } else {
            ld_stream<4>(a + pidx * 16 + 4 * v, x);
            ld_stream<4>(b + pidx * 16 + 4 * v, y);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int w = 8 * v + 2 * k;  // word index 0..31
            uint32_t* pa = w < kK ? &Al[w] : &Ah[w - kK];
            uint32_t* pb = w < kK ? &Bl[w] : &Bh[w - kK];
            pa[0] = lo32(x[k]);
            pa[1] = hi32(x[k]);
            pb[0] = lo32(y[k]);
            pb[1] = hi32(y[k]);
        }
    }
    uint32_t Da[kK], Db[kK];
    const uint32_t sa = absdiff16(Ah, Al, Da), sb = absdiff16(Bh, Bl, Db);
    uint32_t Z1[2 * kK], Z0[2 * kK], Z2[2 * kK];
    mul16_words(Da, Db, Z1);
    mul16_words(Al, Bl, Z0);
    mul16_words(Ah, Bh, Z2);
    {  // R[0, 16) = z0[0, 16)
        uint64_t o0[4], o1[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            o0[k] = uint64_t(Z0[2 * k]) | (uint64_t(Z0[2 * k + 1]) << 32);
            o1[k] = uint64_t(Z0[8 + 2 * k]) | (uint64_t(Z0[8 + 2 * k + 1]) << 32);
        }
        put4(0, o0);
        put4(4, o1);
    }
    // mid = z0 + z2 - z1 (same signs) or + z1 (33 words; the true value is < 2^1025)
    const uint32_t neg = sa == sb ? 1u : 0u, mask = 0u - neg;
    uint32_t mid[2 * kK + 1];
    {
        uint32_t c = neg;
#pragma unroll
        for (int i = 0; i < 2 * kK; ++i) {
            const uint64_t t = uint64_t(Z0[i]) + Z2[i] + (Z1[i] ^ mask) + c;
            mid[i] = uint32_t(t);
            c = uint32_t(t >> 32);
        }
        mid[2 * kK] = c + mask;
    }
    // R[16, 64) = (z0[16, 32) | z2 << 512) + mid
    uint32_t c = 0;
#pragma unroll
    for (int q = 0; q < 6; ++q) {  // 6 x 8 words = 48 words = 24 limbs
        uint32_t r[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int i = 8 * q + e;
            const uint32_t base = i < kK ? Z0[kK + i] : Z2[i - kK];
            const uint32_t add = i <= 2 * kK ? mid[i <= 2 * kK ? i : 0] : 0u;
            const uint64_t t = uint64_t(base) + add + c;
            r[e] = uint32_t(t);
            c = uint32_t(t >> 32);
        }
        uint64_t o[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) o[k] = uint64_t(r[2 * k]) | (uint64_t(r[2 * k + 1]) << 32);
        put4(size_t(8 + 4 * q), o);
    }
}

template <bool IL>
__global__ void __launch_bounds__(DOTG_K16_TPB, DOTG_K16_MINB) k_mul_kara16(uint64_t* out, const uint64_t* a,
                                                                           const uint64_t* b, size_t batch) {
    const size_t pidx = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (pidx >= batch) return;
    kara16_pair<IL>(out, a, b, batch, pidx);
}

// ---------------------------------------------------------------------------
// C3 hybrid: the Karatsuba middle product z1 = |a_hi - a_lo| * |b_hi - b_lo| (512 x 512
// bits) on the otherwise idle FP64 pipe, z0 and z2 on the IMAD pipe as above. Exact 52 x
// 52-bit products on FP64 (tools/dfma_sweep.cu, 2^20 cases checked): with x, y < 2^52,
//   h = fma.rz(x, y, 2^104)  -> bits(h) = bits(2^104) + floor(xy / 2^52)
//   l = fma.rn(x, y, (2^104 + 2^52) - h) -> bits(l) = bits(2^52) + (xy mod 2^52)
// so the raw bit patterns are accumulated as 64-bit integers into radix-2^52 columns and
// the constant biases (a compile-time count per column) are subtracted once. Per pair the
// IMAD pipe issues 512 column MACs instead of 768; the FP64 pipe takes 100 products.
// ---------------------------------------------------------------------------
template <int V>
__device__ __forceinline__ void ld_cached(const uint64_t* p, uint64_t (&v)[V]) {
    static_assert(V == 4, "V = 4");
    asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3]) : "l"(p));
}

// Z = X * Y for 16-word (512-bit) operands, on the FP64 pipe. Z has 32 words.
__device__ __forceinline__ void mul16_words_fp64(const uint32_t (&X)[16], const uint32_t (&Y)[16],
                                                 uint32_t (&Z)[32]) {
    constexpr uint64_t kM52 = (uint64_t(1) << 52) - 1;
    constexpr int NL = 10;  // 52-bit limbs per 512-bit operand
    double x[NL], y[NL];
#pragma unroll
    for (int k = 0; k < NL; ++k) {
        const int o = 52 * k, w = o / 32, sh = o % 32;
        auto word = [](const uint32_t (&W)[16], int i) -> uint64_t { return i < 16 ? W[i < 16 ? i : 0] : 0u; };
        const uint64_t vx = ((word(X, w) | (word(X, w + 1) << 32)) >> sh | (sh ? word(X, w + 2) << (64 - sh) : 0)) & kM52;
        const uint64_t vy = ((word(Y, w) | (word(Y, w + 1) << 32)) >> sh | (sh ? word(Y, w + 2) << (64 - sh) : 0)) & kM52;
        x[k] = double(vx);  // exact: < 2^52
        y[k] = double(vy);
    }
    const double C104 = 20282409603651670423947251286016.0;                     // 2^104
    const double C104p52 = 20282409603651670423947251286016.0 + 4503599627370496.0;  // 2^104 + 2^52
    uint64_t col[2 * NL];
#pragma unroll
    for (int c = 0; c < 2 * NL; ++c) col[c] = 0;
#pragma unroll
    for (int i = 0; i < NL; ++i)
#pragma unroll
        for (int j = 0; j < NL; ++j) {
            double h, cc, l;
            asm("fma.rz.f64 %0, %1, %2, %3;" : "=d"(h) : "d"(x[i]), "d"(y[j]), "d"(C104));
            asm("sub.rn.f64 %0, %1, %2;" : "=d"(cc) : "d"(C104p52), "d"(h));
            asm("fma.rn.f64 %0, %1, %2, %3;" : "=d"(l) : "d"(x[i]), "d"(y[j]), "d"(cc));
            col[i + j] += uint64_t(__double_as_longlong(l));
            col[i + j + 1] += uint64_t(__double_as_longlong(h));
        }
    // remove the biases (mod 2^64: the true column sums are < 20 * 2^52), carry in radix 2^52
    constexpr uint64_t kB52 = 0x4330000000000000ull, kB104 = 0x4670000000000000ull;
    uint64_t r[2 * NL];
    uint64_t carry = 0;
#pragma unroll
    for (int c = 0; c < 2 * NL; ++c) {
        const int nlo = c < NL ? c + 1 : (c <= 2 * NL - 2 ? 2 * NL - 1 - c : 0);  // pairs with i + j = c
        const int nhi = c == 0 ? 0 : (c - 1 < NL ? c : 2 * NL - c);            // pairs with i + j = c - 1
        const uint64_t v = col[c] - uint64_t(nlo) * kB52 - uint64_t(nhi) * kB104 + carry;
        r[c] = v & kM52;
        carry = v >> 52;
    }
    // repack 20 x 52 bits into 32 words (the product is < 2^1024)
#pragma unroll
    for (int w = 0; w < 32; ++w) {
        const int o = 32 * w, k = o / 52, sh = o % 52;
        uint64_t v = r[k] >> sh;
        if (k + 1 < 2 * NL) v |= r[k + 1 < 2 * NL ? k + 1 : 0] << (52 - sh);
        Z[w] = uint32_t(v);
    }
}

#ifndef DOTG_K16H_MINB
#define DOTG_K16H_MINB 16
#endif
__global__ void __launch_bounds__(32, DOTG_K16H_MINB) k_mul_kara16h(uint64_t* out, const uint64_t* a, const uint64_t* b,
                                                                   size_t batch) {
    const size_t pidx = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (pidx >= batch) return;
    const uint64_t* pa = a + pidx * 16;
    const uint64_t* pb = b + pidx * 16;
    // z1 first, from |a_hi - a_lo| and |b_hi - b_lo|; the halves are reloaded (L1) later
    uint32_t Z1[2 * kK];
    uint32_t sa, sb;
    {
        uint32_t Al[kK], Ah[kK], Bl[kK], Bh[kK];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            uint64_t x[4], y[4];
            ld_cached<4>(pa + 4 * v, x);
            ld_cached<4>(pb + 4 * v, y);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int w = 8 * v + 2 * k;
                uint32_t* qa = w < kK ? &Al[w] : &Ah[w - kK];
                uint32_t* qb = w < kK ? &Bl[w] : &Bh[w - kK];
                qa[0] = lo32(x[k]);
                qa[1] = hi32(x[k]);
                qb[0] = lo32(y[k]);
                qb[1] = hi32(y[k]);
            }
        }
        uint32_t Da[kK], Db[kK];
        sa = absdiff16(Ah, Al, Da);
        sb = absdiff16(Bh, Bl, Db);
        mul16_words_fp64(Da, Db, Z1);
    }
    auto load_half = [&](const uint64_t* p, int half, uint32_t (&W)[kK]) {
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            uint64_t x[4];
            ld_cached<4>(p + 8 * half + 4 * v, x);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                W[8 * v + 2 * k] = lo32(x[k]);
                W[8 * v + 2 * k + 1] = hi32(x[k]);
            }
        }
    };
    uint32_t Z0[2 * kK], Z2[2 * kK];
    {
        uint32_t X[kK], Y[kK];
        load_half(pa, 0, X);
        load_half(pb, 0, Y);
        mul16_words(X, Y, Z0);
    }
    uint64_t* po = out + pidx * 32;
    {  // R[0, 16) = z0[0, 16)
        uint64_t o0[4], o1[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            o0[k] = uint64_t(Z0[2 * k]) | (uint64_t(Z0[2 * k + 1]) << 32);
            o1[k] = uint64_t(Z0[8 + 2 * k]) | (uint64_t(Z0[8 + 2 * k + 1]) << 32);
        }
        st_stream<4>(po, o0);
        st_stream<4>(po + 4, o1);
    }
    {
        uint32_t X[kK], Y[kK];
        load_half(pa, 1, X);
        load_half(pb, 1, Y);
        mul16_words(X, Y, Z2);
    }
    // mid = z0 + z2 - z1 (same signs) or + z1, then R[16, 64) as in k_mul_kara16
    const uint32_t neg = sa == sb ? 1u : 0u, mask = 0u - neg;
    uint32_t mid[2 * kK + 1];
    {
        uint32_t c = neg;
#pragma unroll
        for (int i = 0; i < 2 * kK; ++i) {
            const uint64_t t = uint64_t(Z0[i]) + Z2[i] + (Z1[i] ^ mask) + c;
            mid[i] = uint32_t(t);
            c = uint32_t(t >> 32);
        }
        mid[2 * kK] = c + mask;
    }
    uint32_t c = 0;
#pragma unroll
    for (int q = 0; q < 6; ++q) {
        uint32_t r[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int i = 8 * q + e;
            const uint32_t base = i < kK ? Z0[kK + i] : Z2[i - kK];
            const uint32_t add = i <= 2 * kK ? mid[i <= 2 * kK ? i : 0] : 0u;
            const uint64_t t = uint64_t(base) + add + c;
            r[e] = uint32_t(t);
            c = uint32_t(t >> 32);
        }
        uint64_t o[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) o[k] = uint64_t(r[2 * k]) | (uint64_t(r[2 * k + 1]) << 32);
        st_stream<4>(po + 8 + 4 * q, o);
    }
}

// ---------------------------------------------------------------------------
// Generic: any m, any layout (pair p, limb i at p*sp + i*si; out limb k at p*so + k*sio).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t word_at(const uint64_t* base, size_t si, size_t w) {
    const uint64_t limb = base[(w >> 1) * si];
    return (w & 1) ? hi32(limb) : lo32(limb);
}

__global__ void __launch_bounds__(256) k_mul_strided(uint64_t* out, const uint64_t* a, const uint64_t* b,
                                                     size_t m, size_t batch, size_t sp, size_t si,
                                                     size_t so, size_t sio) {
    const size_t pidx = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (pidx >= batch) return;
    const uint64_t* pa = a + pidx * sp;
    const uint64_t* pb = b + pidx * sp;
    uint64_t* po = out + pidx * so;
    const size_t n = 2 * m;
    uint32_t lo = 0, mid = 0, hi = 0, prev = 0;
    for (size_t c = 0; c < 2 * n; ++c) {
        if (c + 1 < 2 * n) {
            const size_t i0 = c + 1 > n ? c + 1 - n : 0;
            const size_t i1 = c < n - 1 ? c : n - 1;
            for (size_t i = i0; i <= i1; ++i) mac(lo, mid, hi, word_at(pa, si, i), word_at(pb, si, c - i));
        }
        const uint32_t w = lo;
        lo = mid;
        mid = hi;
        hi = 0;
        if (c & 1) po[(c >> 1) * sio] = uint64_t(prev) | (uint64_t(w) << 32);
        else prev = w;
    }
}

template <int M, int LAYOUT>
cudaError_t run_regs(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t batch, cudaStream_t st) {
    const size_t blocks = (batch + 127) / 128;
    k_mul_regs<M, LAYOUT><<<unsigned(blocks), 128, 0, st>>>(out, a, b, batch);
    count_launch();
    return cudaGetLastError();
}

template <int M>
cudaError_t run_regblk(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t batch, cudaStream_t st) {
    const size_t blocks = (batch + 127) / 128;
    k_mul_regblk<M><<<unsigned(blocks), 128, 0, st>>>(out, a, b, batch);
    count_launch();
    return cudaGetLastError();
}

template <int M>
cudaError_t run_regblk_rt(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                          cudaStream_t st) {
    const size_t blocks = (batch + 127) / 128;
    k_mul_regblk<M, true><<<unsigned(blocks), 128, 0, st>>>(out, a, b, batch, int(m));
    count_launch();
    return cudaGetLastError();
}

// Pairs per group (= threads per CTA) chosen so that two CTAs fill the SM's shared
// memory and the batch splits into whole rounds of groups across all SMs.
template <int M>
cudaError_t run_smem(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t batch, cudaStream_t st) {
    using C = SmemCfg<M>;
    // per (host thread, device): the smem opt-in is a per-device function attribute
    static thread_local struct { int dev = -1, sms = 0, max_smem = 0; } di;
    int dev = 0;
    cudaGetDevice(&dev);
    // two CTAs per SM, 1 KB reserved per CTA
    auto pairs_per_cta = [](int max_smem) {
        int P = int((size_t(max_smem) / 2 - 1024) / C::PAIR_BYTES);
        return P > 128 ? 128 : (P < 1 ? 1 : P);
    };
    if (di.dev != dev) {
        cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&di.max_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        cudaError_t e = cudaFuncSetAttribute(k_mul_smem<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(size_t(pairs_per_cta(di.max_smem)) * C::PAIR_BYTES));
        if (e != cudaSuccess) return e;
        di.dev = dev;
    }
    const int P = pairs_per_cta(di.max_smem);
    const size_t smem = size_t(P) * C::PAIR_BYTES;
    const int sms = di.sms;
    const size_t groups = (batch + size_t(P) - 1) / size_t(P);
    const size_t slots = size_t(sms) * 2;
    // balanced rounds: every CTA gets ceil(groups / slots) or one fewer groups
    const size_t rounds = (groups + slots - 1) / slots;
    const size_t grid = (groups + rounds - 1) / rounds;
    k_mul_smem<M><<<unsigned(grid), unsigned(P), smem, st>>>(out, a, b, batch);
    count_launch();
    return cudaGetLastError();
}

cudaError_t run_strided(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                        int layout, cudaStream_t st) {
    const size_t blocks = (batch + 255) / 256;
    if (layout == 0)
        k_mul_strided<<<unsigned(blocks), 256, 0, st>>>(out, a, b, m, batch, m, 1, 2 * m, 1);
    else
        k_mul_strided<<<unsigned(blocks), 256, 0, st>>>(out, a, b, m, batch, 1, batch, 1, batch);
    count_launch();
    return cudaGetLastError();
}

bool aligned32(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 31u) == 0; }
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ---------------------------------------------------------------------------
// Unsaturated 52-bit radix (RadixConfig kUnsaturated, limbs.hpp:39-49): the generic
// pipeline at k = 52 (mul.cpp:38-90) and the fixed 5x5 route (mul.cpp:127-150): every
// 52x52-bit product splits at bit 52, low half into column c, high half into c + 1,
// then one carry pass in radix 2^52. Thread per pair, 128-bit column accumulators
// (a column of m pairs sums below 2m * 2^52). Exactly 2m output limbs, each < 2^52.
// ---------------------------------------------------------------------------
// Small m (dot_mul_5x5's m = 5, the 4x4 route's 5 after repacking, up to 16): thread per
// pair with both operands in registers (staged by the CTA through shared memory) and
// every 52 x 52-bit product taken ONCE (mul.lo /
// mul.hi of the 64-bit limbs, split at bit 52: low part into column i + j, high part into
// i + j + 1). A column of M low parts plus M high parts is < 2M * 2^52, so plain 64-bit
// column sums are exact; one radix-2^52 carry pass (mul.cpp:70-90 at k = 52). Rows are
// zero-extended to M limbs (zero limbs add nothing), only 2m limbs are stored.
// FP = true: the 52 x 52-bit products on the FP64 pipe, exactly (the fma.rz / fma.rn pair
// of k_mul_kara16h below: bits(h) = bits(2^104) + floor(xy / 2^52), bits(l) = bits(2^52) +
// (xy mod 2^52)), the raw bit patterns summed per column and the biases removed once -
// three FP64 operations per product instead of a 64-bit multiply and multiply-high on the
// IMAD pipe.
template <int M, bool FP>
__global__ void __launch_bounds__(128) k_mul52_regs(uint64_t* __restrict__ out, const uint64_t* __restrict__ a,
                                                    const uint64_t* __restrict__ b, int m, size_t batch) {
    // the CTA's 128 rows of a and b (and later its 128 products) are contiguous: staged
    // through shared memory with coalesced loads / stores (rows of 5 limbs are 40 bytes)
    __shared__ uint64_t buf[2 * 128 * M];  // a rows | b rows, then the products
    uint64_t* sa = buf;
    uint64_t* sb = buf + 128 * M;
    uint64_t* so = buf;
    const size_t p0 = size_t(blockIdx.x) * 128;
    const size_t np = batch - p0 < 128 ? batch - p0 : 128;
    const size_t nin = np * size_t(m), nout = 2 * nin;
    if (np == 128 && m == M) {
        // a full CTA: every load of the tile in flight at once (2M per thread), then the
        // shared-memory stores (the plain loop waits for each pair of loads)
        uint64_t va[M], vb[M];
#pragma unroll
        for (int k = 0; k < M; ++k) {
            va[k] = __ldcs(a + p0 * M + threadIdx.x + 128 * k);
            vb[k] = __ldcs(b + p0 * M + threadIdx.x + 128 * k);
        }
#pragma unroll
        for (int k = 0; k < M; ++k) {
            sa[threadIdx.x + 128 * k] = va[k];
            sb[threadIdx.x + 128 * k] = vb[k];
        }
    } else {
        for (size_t i = threadIdx.x; i < nin; i += 128) {
            sa[i] = __ldcs(a + p0 * size_t(m) + i);
            sb[i] = __ldcs(b + p0 * size_t(m) + i);
        }
    }
    __syncthreads();
    constexpr uint64_t kMask = (uint64_t(1) << 52) - 1;
    uint64_t x[M], y[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
        x[i] = (threadIdx.x < np && i < m) ? sa[threadIdx.x * m + i] : 0ull;
        y[i] = (threadIdx.x < np && i < m) ? sb[threadIdx.x * m + i] : 0ull;
    }
    __syncthreads();  // the operand rows are in registers: the buffer takes the products
    if (threadIdx.x < np) {
        uint64_t col[2 * M];
#pragma unroll
        for (int c = 0; c < 2 * M; ++c) col[c] = 0;
        if constexpr (FP) {
            const double C104 = 20282409603651670423947251286016.0;                          // 2^104
            const double C104p52 = 20282409603651670423947251286016.0 + 4503599627370496.0;  // 2^104 + 2^52
            double xd[M], yd[M];
#pragma unroll
            for (int i = 0; i < M; ++i) xd[i] = double(x[i]), yd[i] = double(y[i]);  // exact below 2^52
#pragma unroll
            for (int i = 0; i < M; ++i)
#pragma unroll
                for (int j = 0; j < M; ++j) {
                    double h, cc, l;
                    asm("fma.rz.f64 %0, %1, %2, %3;" : "=d"(h) : "d"(xd[i]), "d"(yd[j]), "d"(C104));
                    asm("sub.rn.f64 %0, %1, %2;" : "=d"(cc) : "d"(C104p52), "d"(h));
                    asm("fma.rn.f64 %0, %1, %2, %3;" : "=d"(l) : "d"(xd[i]), "d"(yd[j]), "d"(cc));
                    col[i + j] += uint64_t(__double_as_longlong(l));
                    col[i + j + 1] += uint64_t(__double_as_longlong(h));
                }
            // biases: column c holds one bits(2^52) per pair with i + j = c and one
            // bits(2^104) per pair with i + j = c - 1 (mod 2^64; the true sums are < 2M 2^52)
            constexpr uint64_t kB52 = 0x4330000000000000ull, kB104 = 0x4670000000000000ull;
#pragma unroll
            for (int c = 0; c < 2 * M; ++c) {
                const int nlo = c < M ? c + 1 : (c <= 2 * M - 2 ? 2 * M - 1 - c : 0);
                const int nhi = c == 0 ? 0 : (c - 1 < M ? c : 2 * M - c);
                col[c] -= uint64_t(nlo) * kB52 + uint64_t(nhi) * kB104;
            }
        } else {
#pragma unroll
            for (int i = 0; i < M; ++i)
#pragma unroll
                for (int j = 0; j < M; ++j) {
                    const uint64_t lo = x[i] * y[j], hi = __umul64hi(x[i], y[j]);
                    col[i + j] += lo & kMask;
                    col[i + j + 1] += (hi << 12) | (lo >> 52);  // floor(product / 2^52) < 2^52
                }
        }
        uint64_t carry = 0;
#pragma unroll
        for (int c = 0; c < 2 * M; ++c) {
            const uint64_t v = col[c] + carry;  // < 2^(52 + log2(2M) + 1): no wrap
            if (c < 2 * m) so[threadIdx.x * 2 * m + c] = v & kMask;
            carry = v >> 52;
        }
    }
    __syncthreads();
    for (size_t i = threadIdx.x; i < nout; i += 128) __stcs(out + p0 * 2 * size_t(m) + i, so[i]);
}

__global__ void __launch_bounds__(128) k_mul52(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m,
                                               size_t batch) {
    const size_t p = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= batch) return;
    const uint64_t* pa = a + p * m;
    const uint64_t* pb = b + p * m;
    uint64_t* po = out + p * 2 * m;
    constexpr uint64_t kMask = (uint64_t(1) << 52) - 1;
    typedef unsigned __int128 u128;
    u128 carry = 0;
    for (size_t c = 0; c < 2 * m; ++c) {
        u128 col = carry;
        // low halves of column c, high halves of column c - 1
        const size_t i0 = c + 1 > m ? c + 1 - m : 0, i1 = c < m - 1 ? c : m - 1;
        for (size_t i = i0; i <= i1 && c + 1 < 2 * m; ++i) col += uint64_t(u128(pa[i]) * pb[c - i]) & kMask;
        if (c >= 1) {
            const size_t d = c - 1;
            const size_t j0 = d + 1 > m ? d + 1 - m : 0, j1 = d < m - 1 ? d : m - 1;
            for (size_t i = j0; i <= j1; ++i) col += uint64_t((u128(pa[i]) * pb[d - i]) >> 52);
        }
        po[c] = uint64_t(col) & kMask;
        carry = col >> 52;
    }
}

}  // namespace

cudaError_t launch_mul52_batch(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                               cudaStream_t st) {
    if (batch == 0) return cudaSuccess;
    const unsigned grid = unsigned((batch + 127) / 128);
    static const bool fp = [] {  // A/B knob: 52 x 52-bit products on the FP64 pipe (1) or the IMAD pipe (0)
        const char* e = std::getenv("DOTG_MUL52_FP");
        return e ? std::atoi(e) != 0 : true;
    }();
    if (m > 16) k_mul52<<<grid, 128, 0, st>>>(out, a, b, m, batch);
    else if (fp) {
        if (m <= 4) k_mul52_regs<4, true><<<grid, 128, 0, st>>>(out, a, b, int(m), batch);
        else if (m <= 5) k_mul52_regs<5, true><<<grid, 128, 0, st>>>(out, a, b, int(m), batch);
        else if (m <= 8) k_mul52_regs<8, true><<<grid, 128, 0, st>>>(out, a, b, int(m), batch);
        else k_mul52_regs<16, true><<<grid, 128, 0, st>>>(out, a, b, int(m), batch);
    } else {
        if (m <= 4) k_mul52_regs<4, false><<<grid, 128, 0, st>>>(out, a, b, int(m), batch);
        else if (m <= 5) k_mul52_regs<5, false><<<grid, 128, 0, st>>>(out, a, b, int(m), batch);
        else if (m <= 8) k_mul52_regs<8, false><<<grid, 128, 0, st>>>(out, a, b, int(m), batch);
        else k_mul52_regs<16, false><<<grid, 128, 0, st>>>(out, a, b, int(m), batch);
    }
    count_launch();
    return cudaGetLastError();
}

std::atomic<int> g_mul_route{0};

// dst[c][r] = src[r][c] for a rows x cols u64 matrix: 32 x 32 tiles through shared
// memory (coalesced on both sides; the 33-word row pitch keeps the column reads
// conflict-free).
static __global__ void __launch_bounds__(256) k_transpose_u64(const uint64_t* __restrict__ src, size_t rows, size_t cols,
                                                       uint64_t* __restrict__ dst) {
    __shared__ uint64_t tile[32][33];
    const size_t r0 = size_t(blockIdx.y) * 32, c0 = size_t(blockIdx.x) * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
#pragma unroll
    for (int k = 0; k < 32; k += 8) {
        const size_t r = r0 + ty + k, c = c0 + tx;
        if (r < rows && c < cols) tile[ty + k][tx] = __ldg(src + r * cols + c);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 32; k += 8) {
        const size_t c = c0 + ty + k, r = r0 + tx;
        if (r < rows && c < cols) dst[c * rows + r] = tile[tx][ty + k];
    }
}

static cudaError_t transpose_u64(const uint64_t* src, size_t rows, size_t cols, uint64_t* dst, cudaStream_t st) {
    const dim3 grid(unsigned((cols + 31) / 32), unsigned((rows + 31) / 32));
    if (grid.y > 65535u) return cudaErrorInvalidConfiguration;
    k_transpose_u64<<<grid, 256, 0, st>>>(src, rows, cols, dst);
    count_launch();
    return cudaGetLastError();
}

// Interleaved [m][batch] products for m > 16 go through the row-major kernels: the
// thread-per-pair kernel reading the interleaved layout directly is compute-serial per
// pair (8-18x slower at m = 32 / 64, tools/mul_layout_timing.py), while three transposes
// cost one extra pass over the operands and the product.
static cudaError_t mul_interleaved_via_rows(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                                     cudaStream_t st) {
    retain_stream_pool();
    uint64_t *ta = nullptr, *tb = nullptr, *to = nullptr;
    cudaError_t e = cudaMallocAsync(&ta, batch * m * 8, st);
    if (e == cudaSuccess) e = cudaMallocAsync(&tb, batch * m * 8, st);
    if (e == cudaSuccess) e = cudaMallocAsync(&to, batch * 2 * m * 8, st);
    if (e == cudaSuccess) e = transpose_u64(a, m, batch, ta, st);
    if (e == cudaSuccess) e = transpose_u64(b, m, batch, tb, st);
    if (e == cudaSuccess) e = launch_mul_batch(to, ta, tb, m, batch, 0, st);
    if (e == cudaSuccess) e = transpose_u64(to, batch, 2 * m, out, st);
    for (void* q : {static_cast<void*>(ta), static_cast<void*>(tb), static_cast<void*>(to)})
        if (q != nullptr) cudaFreeAsync(q, st);
    return e;
}

cudaError_t launch_mul_batch(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                             int layout, cudaStream_t stream) {
    if (batch == 0) return cudaSuccess;
    const bool al = aligned32(out) && aligned32(a) && aligned32(b);
    // interleaved even 16 < m <= 128: the tensor-pipe kernel reads and writes the
    // interleaved layout in place (tools/mul_layout_timing.py)
    if (layout == 1 && m > 16 && m <= 128 && g_mul_route.load(std::memory_order_relaxed) != 1)
        return launch_mul_imma_il(out, a, b, m, batch, stream);
    // Small sizes off the powers of two (m = 3 ... 15) on a register kernel of exactly m
    // limbs (no zero-extended columns; tools/mul_sweep.py, profiles/r02_mul_exact_ab.jsonl):
    // interleaved rows are coalesced as they are (the transposes around the row-major route
    // below cost 3-5x: m = 3 ... 15 at 24-42 us per 2^22 limbs, were 114-145); even row-major
    // m too (m = 6 24 vs 45 us, m = 10-14 30-38 vs 63-66 zero-extended); odd row-major rows
    // are staged through shared memory so loads and stores stay coalesced (unstaged they ran
    // 39-69 us, no faster than zero-extension). DOTG_MUL_EXACT=0 (A/B) takes the old routes,
    // =3 the exact kernel without staging.
    static const int exact = [] {
        const char* e = std::getenv("DOTG_MUL_EXACT");
        return e ? std::atoi(e) : 1;
    }();
    if (exact && g_mul_route.load(std::memory_order_relaxed) != 1 && m >= 3 && m <= 15 && (m & (m - 1)) != 0) {
        const int L = layout == 1 ? 1 : (m % 2 == 1 && exact != 3 ? 2 : 0);  // odd rows: staged
        switch (m) {
#define DOTG_EXACT(MM)                                                                                           \
    case MM:                                                                                                     \
        return L == 1 ? run_regs<MM, 1>(out, a, b, batch, stream)                                               \
                      : (L == 2 ? run_regs<MM, 2>(out, a, b, batch, stream) : run_regs<MM, 0>(out, a, b, batch, stream));
            DOTG_EXACT(3) DOTG_EXACT(5) DOTG_EXACT(6) DOTG_EXACT(7) DOTG_EXACT(9) DOTG_EXACT(10)
            DOTG_EXACT(11) DOTG_EXACT(12) DOTG_EXACT(13) DOTG_EXACT(14) DOTG_EXACT(15)
#undef DOTG_EXACT
            default: break;
        }
    }
    // other interleaved m > 16, and 4 < m < 16 off the powers of two (no interleaved register
    // kernel for those): transpose around the row-major route
    if (layout == 1 && (m > 16 || (m > 4 && (m & (m - 1)) != 0)) && g_mul_route.load(std::memory_order_relaxed) != 1 &&
        batch <= (size_t(65535) * 32))
        return mul_interleaved_via_rows(out, a, b, m, batch, stream);
    // Tensor pipe where it beats the IMAD kernels (tools/mul_timing.py on B200: m = 32
    // 1.27x, 64 2.26x, 128 3.8x; at m = 8 / 16 the per-pair warp overhead loses to the
    // thread-per-pair IMAD kernels, so only a forced IMMA route takes them there).
    const int route = g_mul_route.load(std::memory_order_relaxed);
    if (layout == 0 && mul_imma_supported(m) && route != 1 && (route == 2 || m >= 32))
        return al ? launch_mul_imma(out, a, b, m, batch, stream) : mul_padded_rows(out, a, b, m, batch, m, stream);
    // Sizes without a dedicated kernel: 16 < m < 128 zero-pads to the next tensor-pipe
    // size; m > 128 runs padded Karatsuba down to m = 128 tensor-pipe leaves (the generic
    // thread-per-pair kernel would be 100x slower there: tools/kara_timing.py). Both copy
    // the rows, so any alignment works.
    if (layout == 0 && route != 1 && m > 16 && m < 128 &&
        (m % 2 == 1 || (aligned16(out) && aligned16(a) && aligned16(b))))  // odd rows: direct loads
        return launch_mul_imma_rt(out, a, b, m, batch, stream);
    // m >= 256: the tcgen05 column kernel (mul_umma.cu) up to 16384 limbs (rows padded to a
    // multiple of 16 limbs when needed), Karatsuba down to its leaves above that.
    if (layout == 0 && route != 1 && m >= 256 && ((m + 15) & ~size_t(15)) <= mul_umma_direct_max() &&
        mul_umma_supported((m + 15) & ~size_t(15))) {
        if (m % 16 == 0 && aligned16(a) && aligned16(b)) return launch_mul_umma(out, a, b, m, batch, stream);
        return mul_padded_rows(out, a, b, m, batch, (m + 15) & ~size_t(15), stream);
    }
    if (layout == 0 && route != 1 && m > mul_umma_direct_max() && mul_umma_supported(mul_umma_leaf(m, batch)))
        return launch_karatsuba_padded(out, a, b, m, batch, mul_umma_leaf(m, batch), stream);
    if (layout == 0 && route != 1 && m > 16 && !mul_imma_supported(m)) {
        // rows copy-padded to the next tensor-pipe size: a multiple of 16 limbs up to 128
        // (DOTG_IMMA_FINE=0: the next power of two), padded Karatsuba above
        static const int fine = [] {
            const char* e = std::getenv("DOTG_IMMA_FINE");
            return e ? std::atoi(e) : 1;
        }();
        size_t base = m > 128 ? 128 : (fine ? (m + 15) & ~size_t(15) : (m <= 32 ? 32 : (m <= 64 ? 64 : 128)));
        // 128 < m < 256: one Karatsuba level over the smallest tensor-pipe leaf of 80 / 96 /
        // 112 / 128 limbs that covers m (m = 129 padded to 160 instead of 256: 1.5x the
        // products instead of 3.9x)
        if (fine && m > 128 && m < 256) base = m <= 160 ? 80 : (m <= 192 ? 96 : (m <= 224 ? 112 : 128));
        return launch_karatsuba_padded(out, a, b, m, batch, base < 32 ? 32 : base, stream);
    }
    // 4 < m < 16 off the power-of-two kernels, or misaligned rows of 5..16: the register
    // kernels of the next size with zero-extended operands, any alignment
    // (tools/odd_m_mul_timing.py: m = 12 92 us vs 492 us thread-per-pair generic).
    if (layout == 0 && route != 1 && m > 4 && m <= 16 && (!al || (m & (m - 1)) != 0))
        return m <= 8 ? run_regblk_rt<8>(out, a, b, m, batch, stream) : run_regblk_rt<16>(out, a, b, m, batch, stream);
    if (layout == 1) {
        switch (m) {
            case 1: return run_regs<1, 1>(out, a, b, batch, stream);
            case 2: return run_regs<2, 1>(out, a, b, batch, stream);
            case 4: return run_regs<4, 1>(out, a, b, batch, stream);
            case 8: return run_regs<8, 1>(out, a, b, batch, stream);
            case 16:
                if (route != 1) {  // the C3 kernel on the interleaved layout (one Karatsuba level)
                    k_mul_kara16<true><<<unsigned((batch + DOTG_K16_TPB - 1) / DOTG_K16_TPB), DOTG_K16_TPB, 0,
                                         stream>>>(out, a, b, batch);
                    count_launch();
                    return cudaGetLastError();
                }
                return run_regs<16, 1>(out, a, b, batch, stream);
            default: return run_strided(out, a, b, m, batch, 1, stream);
        }
    }
    switch (m) {
        case 1: return run_regs<1, 0>(out, a, b, batch, stream);
        case 2:
            if (al) return run_regs<2, 0>(out, a, b, batch, stream);
            break;
        case 4:
            if (al) return run_regs<4, 0>(out, a, b, batch, stream);
            break;
        case 8:
            if (al) return run_regblk<8>(out, a, b, batch, stream);
            break;
        case 16:
            if (al) {  // C3: 40.0 us vs 42.1 us for the plain 16-column kernel (tools/mul_timing.py)
                // A/B knob: DOTG_K16_HYBRID=1 takes z1 on the FP64 pipe (k_mul_kara16h).
                // Measured r02 (tools/c3_probe.py): 41.6 vs 39.4 us at 2^18 pairs, 0.873 vs
                // 0.903 of the roofline at 2^21 - the kernel is latency-bound at 16 warps/SM,
                // not IMAD-pipe-bound, so moving a third of the MACs to another pipe loses
                // to the extra instructions. Default off.
                static const int hybrid = [] {
                    const char* e = std::getenv("DOTG_K16_HYBRID");
                    return e ? std::atoi(e) : 0;
                }();
                if (hybrid)
                    k_mul_kara16h<<<unsigned((batch + 31) / 32), 32, 0, stream>>>(out, a, b, batch);
                else
                    k_mul_kara16<false><<<unsigned((batch + DOTG_K16_TPB - 1) / DOTG_K16_TPB), DOTG_K16_TPB, 0, stream>>>(
                        out, a, b, batch);
                count_launch();
                return cudaGetLastError();
            }
            break;
        case 32:
            if (al) return run_smem<32>(out, a, b, batch, stream);
            break;
        case 64:
            if (al) return run_smem<64>(out, a, b, batch, stream);
            break;
        case 128:
            if (al) return run_smem<128>(out, a, b, batch, stream);
            break;
        default:
            break;
    }
    return run_strided(out, a, b, m, batch, 0, stream);
}

}  // namespace dotg
