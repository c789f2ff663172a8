// mul_imma.cu - batched column multiplication on the integer tensor pipe (IMMA).
//
// Same contract as the IMAD column kernels in mul_batch.cu (dot_mul_words,
// include/dot/mul.hpp:75-76, src/mul.cpp:96-103: every column of partial products
// summed, one deferred carry pass, exactly 2m output limbs), but the partial products
// are taken in radix 2^8 on the tensor cores: BASELINE.json's north_star allows an
// 8-bit limb-split tensor variant when it beats the IMAD pipe. Measured on B200
// (tools/imma_peak.cu): mma.sync m16n8k32 u8 sustains 2048 byte-MACs/clk/SM = 128
// u32-product equivalents/clk/SM, 4x the 32/clk/SM of IMAD.WIDE.U32.
//
// Formulation (one warp per pair, operands of n = 32*NB bytes, NB 32-byte blocks):
//   column sum S[x] = sum_i a[i] * b[x - i]   (bytes, x < 2n; S < 2^27 for n <= 1024)
// One m16n8k32 MMA computes D[r][c] += sum_k A[r][k] * B[k][c] with
//   A[r][k] = bpad[H + r + k]                 Hankel window of b (bpad[y] = b[y - 31])
//   B[k][c] = a[32*(c0 + c - beta) + 31 - k]  a-block (c0 + c - beta), byte-reversed
//   H = R0 + 32*beta
// Every product term lands in column x = R0 + r + 32*(c0 + c), independent of beta
// and k, so the tensor core itself sums a whole column: accumulator tile (R0, c0)
// iterates beta over the blocks and finishes holding exact column sums - no partial
// sums leave the registers. Tiles: R0 in {0, 16}, c0 in {0, 8, ...} (2n/256 of them).
//
// Operand delivery (no per-MMA shared-memory round trips for B):
//   * b is staged once per pair as 4 byte-shifted copies in shared memory, so every
//     4-byte Hankel window is one aligned LDS.32 (lane (g,t) always reads copy g & 3);
//     windows at 16j + g + 4t (+8) serve tiles R0 = 0 and 16 of consecutive beta.
//   * the a-blocks a lane ever needs (block g - m for m = beta - c0) are loaded once per
//     pair into registers Q[m], indexed by the compile-time m: the lane-dependent block
//     index is folded into which word each lane loads, not into register indexing.
// Epilogue: D tiles -> per-warp shared column array (conflict-free padded index), each
// lane folds 8 columns per output limb into a 128-bit value, and one warp-ballot carry
// lookahead (device.cuh) resolves the inter-limb carries - the same generate/propagate
// algebra as the add kernel, used as the deferred carry-normalisation pass. (Measured
// r01: the epilogue is ~17 of C4's 85 us. A shared-memory-free version - Hankel rows
// permuted so a lane holds adjacent byte columns, limbs assembled by two shuffle
// butterflies and a lane permutation - was bit-exact but no faster at m = 64 (84.7 us),
// 5% faster at m = 32 and spilled at m = 128 (92.8 vs 63 us).)
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "device.cuh"
#include "internal.h"

namespace dotg {

namespace {

__device__ __forceinline__ void imma(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                     uint32_t b1) {
    asm("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

template <int NB>
struct ImmaCfg {
    static constexpr int M = 4 * NB;              // limbs per operand
    static constexpr int NW = 8 * NB;             // u32 words per operand
    static constexpr int CL = NW + 16;            // words per shifted copy of bpad
    static constexpr int CLP = CL + ((8 - CL % 32) + 32) % 32;  // padded: CLP % 32 == 8
    static constexpr int COPY_WORDS = 4 * CLP;
    // a as 12-word blocks (8 words + 4 pad: conflict-free Q loads), 7 zero blocks each
    // side so every lane's block g - m is a valid (possibly zero) block
    static constexpr int A_WORDS = 12 * (NB + 14);
    static constexpr int NCOL = 64 * NB;          // product bytes = column sums
    static constexpr int S_WORDS = NCOL + 4 * (NCOL / 32);  // padded index x + 4 (x >> 5)
#ifndef DOTG_IMMA_ST_BIG
#define DOTG_IMMA_ST_BIG 4
#endif
    static constexpr int ST = M >= 64 ? DOTG_IMMA_ST_BIG : 8;  // bulk-copy ring stages per warp
    static constexpr int RAW_WORDS = ST * 2 * NW; // ring of raw (a, b) pairs
    static constexpr int WARP_WORDS = RAW_WORDS + COPY_WORDS + A_WORDS + S_WORDS;
    static constexpr int NC0 = (2 * NB + 7) / 8;  // accumulator tiles per R0
    static constexpr int NQ = NB + 7;             // Q[m], m in [-(NB-1), 7]
    static constexpr int OUT_LIMBS = 2 * M;
    static constexpr int LPL = OUT_LIMBS >= 32 ? (OUT_LIMBS + 31) / 32 : 1;  // output limbs per lane
    static constexpr int LANES = OUT_LIMBS >= 32 ? 32 : OUT_LIMBS;  // lane l: limbs l + 32k (< OUT_LIMBS)
    static constexpr int VW = (NW + 31) / 32;                        // operand words per lane
    static constexpr int LD_LANES = NW / VW;
    static_assert(LANES <= 32, "limb split");
    static_assert(NW % VW == 0 && NW / VW <= 32, "operand split");  // VW of 3, 5, 6, 7: scalar moves
};

constexpr int kImmaWarps = 4;

// ---- bulk async copies (TMA engine, no tensor map) into a per-warp mbarrier ring
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ int aidx(int w) { return 12 * ((w >> 3) + 7) + (w & 7); }

// Shared-memory vector moves of VW consecutive, VW-aligned words.
template <int VW, int N>
__device__ __forceinline__ void lds_vec(const uint32_t* p, uint32_t (&w)[N]) {
    if constexpr (VW == 8) {
        const uint4 v = *reinterpret_cast<const uint4*>(p);
        const uint4 u = *reinterpret_cast<const uint4*>(p + 4);
        w[0] = v.x, w[1] = v.y, w[2] = v.z, w[3] = v.w;
        w[4] = u.x, w[5] = u.y, w[6] = u.z, w[7] = u.w;
    } else if constexpr (VW == 4) {
        const uint4 v = *reinterpret_cast<const uint4*>(p);
        w[0] = v.x, w[1] = v.y, w[2] = v.z, w[3] = v.w;
    } else if constexpr (VW == 2) {
        const uint2 v = *reinterpret_cast<const uint2*>(p);
        w[0] = v.x, w[1] = v.y;
    } else if constexpr (VW == 1) {
        w[0] = *p;
    } else {
#pragma unroll
        for (int e = 0; e < VW; ++e) w[e] = p[e];
    }
}
template <int VW>
__device__ __forceinline__ void sts_vec(uint32_t* p, const uint32_t (&w)[VW]) {
    if constexpr (VW == 8) {
        *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
        *reinterpret_cast<uint4*>(p + 4) = make_uint4(w[4], w[5], w[6], w[7]);
    } else if constexpr (VW == 4) {
        *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
    } else if constexpr (VW == 2) {
        *reinterpret_cast<uint2*>(p) = make_uint2(w[0], w[1]);
    } else if constexpr (VW == 1) {
        *p = w[0];
    } else {
#pragma unroll
        for (int e = 0; e < VW; ++e) p[e] = w[e];
    }
}

// Persistent: every warp walks pairs gw, gw + nwarps, ... with the next ST pairs'
// operands in flight through the bulk-copy ring. (Measured r01: software-pipelining the
// warp - pair k-1's epilogue and pair k+1's staging placed inside pair k's unrolled beta
// loop, two staging buffers, column sums aliasing the dead buffer - is bit-exact but
// slower at every size: C4 99.1 us vs 83.1 us, 128 registers.)
#ifndef DOTG_IMMA_MINB16
#define DOTG_IMMA_MINB16 1
#endif
// IL = true: the batch-interleaved layout [m][batch] (limb i of pair p at i * batch + p),
// read and written in place - no transposes. A CTA takes kGP = 16 consecutive pairs at a
// time (4 per warp): it loads their [m][16] operand tiles with whole 128-byte rows (16
// threads per limb row) into one padded shared tile, each warp runs its 4 pairs from
// their tile columns and writes each product back into its own pair's column (2m limbs:
// the operand rows it replaces are already staged), and the CTA stores the [2m][16]
// product tile with whole rows. Two barriers per 16 pairs. (r02: a [m][4] tile per 4
// pairs, 32-byte rows, two barriers per 4 pairs: 105 us at m = 64; every warp loading
// its own pair: 139 us, L1 92% busy.) Row-major (IL = false) uses the per-warp mbarrier
// ring of cp.async.bulk copies.
#ifndef DOTG_IMMA_GP16
#define DOTG_IMMA_GP16 16
#endif
#ifndef DOTG_IMMA_IL_PREFETCH
#define DOTG_IMMA_IL_PREFETCH 1  // the next group's tile loads in flight during this one (0: load on arrival)
#endif
#ifndef DOTG_IMMA_IL_MINB16
#define DOTG_IMMA_IL_MINB16 3  // 150 registers for the prefetch (4 CTAs/SM would spill)
#endif
// pairs per interleaved CTA group (NB = 16: DOTG_IMMA_GP16) and words per tile row (2 per
// pair + 1 pad: odd, so the warps' column reads are conflict-free)
template <int NB> __host__ __device__ constexpr int il_gp() { return NB == 16 ? DOTG_IMMA_GP16 : 16; }
template <int NB> __host__ __device__ constexpr int il_pitch() { return 2 * il_gp<NB>() + 1; }
template <int NB, bool IL>
__global__ void __launch_bounds__(kImmaWarps * 32, NB == 16 ? (IL ? DOTG_IMMA_IL_MINB16 : DOTG_IMMA_MINB16) : 1) k_mul_imma(uint64_t* __restrict__ out,
                                                              const uint64_t* __restrict__ a,
                                                              const uint64_t* __restrict__ b, size_t batch,
                                                              int mr) {
    // mr < M: rows of mr limbs (mr even, 16-byte aligned rows), zero-extended in the raw
    // ring to M limbs - only the first 8 mr bytes of a slot are ever loaded, the rest stays
    // zero - and only 2 mr product limbs are stored.
    using C = ImmaCfg<NB>;
    extern __shared__ __align__(16) uint32_t smem_dyn[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    uint32_t* raw = smem_dyn + size_t(warp) * (IL ? C::WARP_WORDS - C::RAW_WORDS : C::WARP_WORDS);
    uint32_t* cp = raw + (IL ? 0 : C::RAW_WORDS);            // 4 shifted copies of bpad
    uint32_t* sa = cp + C::COPY_WORDS;                        // byte-reversed a words
    int* S = reinterpret_cast<int*>(sa + C::A_WORDS);         // column sums
    __shared__ uint64_t bars[kImmaWarps][C::ST];
    uint64_t* bar = bars[warp];
    // IL tile: rows [0, M) operand a, [M, 2M) operand b, later rows [0, 2M) the products
    constexpr int kGP = il_gp<NB>(), kTileP = il_pitch<NB>();
    __shared__ uint32_t tile[IL ? 2 * C::M * kTileP : 1];
    for (int i = lane; i < C::COPY_WORDS + C::A_WORDS; i += 32) cp[i] = 0;  // padding stays zero
    if (!IL && mr < C::M)
        for (int i = lane; i < C::RAW_WORDS; i += 32) raw[i] = 0;
    __syncwarp();
    // the zero-fill is a generic-proxy write; the bulk copies below write the same ring
    // through the async proxy: order the former before the latter
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");

    const size_t nwarps = size_t(gridDim.x) * kImmaWarps;
    const size_t first = size_t(blockIdx.x) * kImmaWarps + warp;
    const uint32_t kOpBytes = uint32_t(mr) * 8u;  // bytes per operand row
    auto issue = [&](int stage, size_t p) {  // lane 0 only
        uint32_t* dst = raw + stage * 2 * C::NW;
        mbar_expect_tx(&bar[stage], 2 * kOpBytes);
        bulk_load(dst, a + p * size_t(mr), kOpBytes, &bar[stage]);
        bulk_load(dst + C::NW, b + p * size_t(mr), kOpBytes, &bar[stage]);
    };
    // odd mr: rows are not 16-byte aligned, so no bulk copies - each warp loads its pair's
    // words straight from global memory (coalesced 32-bit loads, zero past 2 mr words)
    const bool direct = !IL && (mr & 1) != 0;
    if (!IL && !direct && lane == 0) {
        for (int st = 0; st < C::ST; ++st) mbar_init(&bar[st]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int st = 0; st < C::ST; ++st)
            if (first + size_t(st) * nwarps < batch) issue(st, first + size_t(st) * nwarps);
    }
    __syncwarp();

    // ---- stage: copy_s[i] = bytes bpad[4i + s ..], bpad[y] = b[y - 31]; word j of b feeds
    // copy index i = j + 8 (with word j + 1), and i = 7 takes (0, b[0]). av / bv: the lane's
    // VW operand words (lanes < LD_LANES).
    auto stage_pair = [&](uint32_t (&av)[C::VW], uint32_t (&bv)[C::VW + 1]) {
        const uint32_t nxt = __shfl_down_sync(0xffffffffu, bv[0], 1);
        if (lane < C::LD_LANES) {
            bv[C::VW] = lane + 1 < C::LD_LANES ? nxt : 0u;
            const int j0 = lane * C::VW;  // copy index j0 + 8 is VW-aligned
            uint32_t c0[C::VW], c1[C::VW], c2[C::VW], c3[C::VW], sv[C::VW];
#pragma unroll
            for (int e = 0; e < C::VW; ++e) {
                const uint32_t lo = bv[e], hi = bv[e + 1];
                c0[e] = __funnelshift_r(lo, hi, 8);
                c1[e] = __funnelshift_r(lo, hi, 16);
                c2[e] = __funnelshift_r(lo, hi, 24);
                c3[e] = hi;
                sv[e] = bswap32(av[e]);
            }
            sts_vec<C::VW>(cp + 0 * C::CLP + j0 + 8, c0);
            sts_vec<C::VW>(cp + 1 * C::CLP + j0 + 8, c1);
            sts_vec<C::VW>(cp + 2 * C::CLP + j0 + 8, c2);
            sts_vec<C::VW>(cp + 3 * C::CLP + j0 + 8, c3);
            if constexpr ((C::VW & (C::VW - 1)) == 0) {
                sts_vec<C::VW>(sa + aidx(j0), sv);  // VW-aligned: inside one 8-word block
            } else {
#pragma unroll
                for (int e = 0; e < C::VW; ++e) sa[aidx(j0 + e)] = sv[e];
            }
            if (lane == 0) {
                cp[0 * C::CLP + 7] = bv[0] << 24;
                cp[1 * C::CLP + 7] = bv[0] << 16;
                cp[2 * C::CLP + 7] = bv[0] << 8;
                cp[3 * C::CLP + 7] = bv[0];
            }
        }
        __syncwarp();
    };

    // ---- tensor-core column sums of the staged pair, then the deferred carry pass:
    // lo[k] = product limb lane + 32 k (lanes < LANES)
    const bool active = lane < C::LANES;
    auto multiply_staged = [&](uint64_t (&lo)[C::LPL]) {
        // a-blocks in registers: Q[m] = block (g - m), words 7 - t and 3 - t
        uint32_t Q0[C::NQ], Q1[C::NQ];
        const uint32_t* qb = sa + 12 * (g + 7 + NB - 1) + 3 - t;  // block g - m, m = q - (NB - 1)
#pragma unroll
        for (int q = 0; q < C::NQ; ++q) {
            Q0[q] = qb[4 - 12 * q];
            Q1[q] = qb[-12 * q];
        }
        int D[2][C::NC0][4];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int c = 0; c < C::NC0; ++c) D[r][c][0] = D[r][c][1] = D[r][c][2] = D[r][c][3] = 0;
        const uint32_t* wb = cp + (g & 3) * C::CLP + (g >> 2) + t;  // W(16j + g + 4t) = wb[4j]
#pragma unroll
        for (int be = 0; be <= NB; ++be) {
            const uint32_t x0 = wb[8 * be], x1 = wb[8 * be + 2];       // j = 2 be
            const uint32_t y0 = wb[8 * be + 4], y1 = wb[8 * be + 6];   // j = 2 be + 1
            const uint32_t z0 = wb[8 * be + 8], z1 = wb[8 * be + 10];  // j = 2 be + 2
#pragma unroll
            for (int c = 0; c < C::NC0; ++c) {
                const int c0 = 8 * c;
                if (be < c0 - NB + 1 || be > c0 + 7) continue;
                const int q = be - c0 + NB - 1;
                imma(D[0][c], x0, x1, y0, y1, Q0[q], Q1[q]);
                imma(D[1][c], y0, y1, z0, z1, Q0[q], Q1[q]);
            }
        }
        // column sums to shared memory: tile (R0 = 16 r, c0 = 8 c): d0 -> x, d1 -> x + 32,
        // d2 -> x + 8, d3 -> x + 40, x = R0 + g + 32 (c0 + 2t); padded index x + 4 (x >> 5)
        // keeps these stores and the limb reads below conflict-free.
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int c = 0; c < C::NC0; ++c) {
                const int x = 16 * r + g + 32 * (8 * c + 2 * t);
                if (x < C::NCOL) {
                    const int p = x + 4 * (x >> 5);
                    S[p] = D[r][c][0];
                    S[p + 36] = D[r][c][1];
                    S[p + 8] = D[r][c][2];
                    S[p + 44] = D[r][c][3];
                }
            }
        __syncwarp();
        // deferred carry normalisation. Lane l owns limbs L = l + 32k; limb value
        // sum_e S[8L + e] 2^(8e) < 2^83 as (lo, hi); t_L = lo_L + hi_{L-1} with generate =
        // carry out of that add and propagate = (t_L == ~0), then one ballot lookahead per
        // 32-limb segment, segments chained through their carry-out.
        typedef unsigned __int128 u128;
        uint64_t hi[C::LPL];
#pragma unroll
        for (int k = 0; k < C::LPL; ++k) {
            const int L = lane + 32 * k;
            u128 v = 0;
            if (active && L < C::OUT_LIMBS) {
                const int base = 8 * L + 4 * (L >> 2);
                const int4 s0 = *reinterpret_cast<const int4*>(S + base);
                const int4 s1 = *reinterpret_cast<const int4*>(S + base + 4);
                const uint64_t low = uint64_t(uint32_t(s0.x)) + (uint64_t(uint32_t(s0.y)) << 8) +
                                     (uint64_t(uint32_t(s0.z)) << 16) + (uint64_t(uint32_t(s0.w)) << 24) +
                                     (uint64_t(uint32_t(s1.x)) << 32);  // < 2^59
                v = u128(low) + (u128(uint32_t(s1.y)) << 40) + (u128(uint32_t(s1.z)) << 48) +
                    (u128(uint32_t(s1.w)) << 56);
            }
            lo[k] = uint64_t(v);
            hi[k] = uint64_t(v >> 64);
        }
        __syncwarp();  // S is rewritten by the next pair
        uint32_t cseg = 0;  // carry into the current 32-limb segment
#pragma unroll
        for (int k = 0; k < C::LPL; ++k) {
            uint64_t h = __shfl_up_sync(0xffffffffu, hi[k], 1);
            const uint64_t hwrap = k > 0 ? __shfl_sync(0xffffffffu, hi[k > 0 ? k - 1 : 0], 31) : 0ull;
            if (lane == 0) h = hwrap;
            uint64_t sv = lo[k] + h;
            const bool ak = active && lane + 32 * k < C::OUT_LIMBS;  // last segment may be partial
            const uint32_t gk = ak && sv < h, pk = ak && sv == ~0ull;
            const uint32_t Gm = __ballot_sync(0xffffffffu, gk), Pm = __ballot_sync(0xffffffffu, pk);
            const uint64_t y = ((uint64_t(Gm) << 1) | cseg) + uint64_t(Pm);
            const uint32_t Cm = uint32_t(y) ^ Pm;
            cseg = uint32_t(y >> 32);
            sv += (Cm >> lane) & 1u;
            lo[k] = sv;
        }
    };

    if constexpr (IL) {
        // IL: lane's VW operand words of a pair = limbs VW/2 * lane ... (VW even for m >= 32)
        static_assert(C::VW % 2 == 0, "interleaved route needs two or more words per lane");
        constexpr int LL = C::VW / 2;                       // limbs per lane
        constexpr int NE = 2 * C::M * kGP / (kImmaWarps * 32);  // tile elements per thread
        static_assert((2 * C::M * kGP) % (kImmaWarps * 32) == 0, "tile split");
        const size_t ngroups = (batch + kGP - 1) / kGP;
        // element e = threadIdx.x + 128 i of a tile: row e / 16, pair column e % 16 (16
        // consecutive threads: one 128-byte limb row)
        uint64_t v[NE];
        auto fetch = [&](size_t grp) {
#pragma unroll
            for (int i = 0; i < NE; ++i) {
                const int e = threadIdx.x + kImmaWarps * 32 * i;
                const int r = e / kGP, col = e % kGP;
                const int lr = r < C::M ? r : r - C::M;  // rows [0, M): a, [M, 2M): b
                const size_t pr = grp * kGP + size_t(col);
                v[i] = (grp < ngroups && pr < batch && lr < mr) ? __ldg((r < C::M ? a : b) + size_t(lr) * batch + pr)
                                                                 : 0ull;
            }
        };
        if (DOTG_IMMA_IL_PREFETCH) fetch(blockIdx.x);
        for (size_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
            if (!DOTG_IMMA_IL_PREFETCH) fetch(grp);
#pragma unroll
            for (int i = 0; i < NE; ++i) {
                const int e = threadIdx.x + kImmaWarps * 32 * i;
                uint32_t* tp = tile + (e / kGP) * kTileP + 2 * (e % kGP);
                tp[0] = uint32_t(v[i]);
                tp[1] = uint32_t(v[i] >> 32);
            }
            __syncthreads();
            if (DOTG_IMMA_IL_PREFETCH) fetch(grp + gridDim.x);  // in flight during this group
#pragma unroll 1
            for (int j = 0; j < kGP / kImmaWarps; ++j) {
                const int col = warp * (kGP / kImmaWarps) + j;
                uint32_t bv[C::VW + 1], av[C::VW];
#pragma unroll
                for (int e = 0; e < LL; ++e) {
                    const int L = lane * LL + e;
                    av[2 * e] = tile[L * kTileP + 2 * col];
                    av[2 * e + 1] = tile[L * kTileP + 2 * col + 1];
                    bv[2 * e] = tile[(C::M + L) * kTileP + 2 * col];
                    bv[2 * e + 1] = tile[(C::M + L) * kTileP + 2 * col + 1];
                }
                stage_pair(av, bv);  // the column's operand rows are free from here on
                uint64_t lo[C::LPL];
                multiply_staged(lo);
                if (active)
#pragma unroll
                    for (int k = 0; k < C::LPL; ++k) {
                        uint32_t* to = tile + (lane + 32 * k) * kTileP + 2 * col;
                        to[0] = uint32_t(lo[k]);
                        to[1] = uint32_t(lo[k] >> 32);
                    }
            }
            __syncthreads();
            // the products, whole rows; the same element mapping as the load above, so the
            // next group's tile writes need no barrier after these reads
#pragma unroll
            for (int i = 0; i < NE; ++i) {
                const int e = threadIdx.x + kImmaWarps * 32 * i;
                const int r = e / kGP, col = e % kGP;
                const size_t pr = grp * kGP + size_t(col);
                if (pr < batch && r < 2 * mr) {
                    const uint32_t* tp = tile + r * kTileP + 2 * col;
                    out[size_t(r) * batch + pr] = uint64_t(tp[0]) | (uint64_t(tp[1]) << 32);
                }
            }
        }
    } else if (direct) {
        const uint32_t nw = 2u * uint32_t(mr);  // u32 words per operand row
        for (size_t pair = first; pair < batch; pair += nwarps) {
            const uint32_t* a32 = reinterpret_cast<const uint32_t*>(a + pair * size_t(mr));
            const uint32_t* b32 = reinterpret_cast<const uint32_t*>(b + pair * size_t(mr));
            uint32_t bv[C::VW + 1], av[C::VW];
            if (lane < C::LD_LANES) {
#pragma unroll
                for (int e = 0; e < C::VW; ++e) {
                    const uint32_t w = uint32_t(lane * C::VW + e);
                    av[e] = w < nw ? __ldg(a32 + w) : 0u;
                    bv[e] = w < nw ? __ldg(b32 + w) : 0u;
                }
            }
            stage_pair(av, bv);
            uint64_t lo[C::LPL];
            multiply_staged(lo);
            if (active) {
                uint64_t* po = out + pair * (2 * size_t(mr)) + lane;
#pragma unroll
                for (int k = 0; k < C::LPL; ++k)
                    if (lane + 32 * k < 2 * mr) po[32 * k] = lo[k];
            }
        }
    } else {
        int stage = 0;
        uint32_t parity = 0;
        for (size_t pair = first; pair < batch; pair += nwarps) {
            mbar_wait(&bar[stage], parity);
            {
                const uint32_t* ra = raw + stage * 2 * C::NW;
                const uint32_t* rb = ra + C::NW;
                uint32_t bv[C::VW + 1], av[C::VW];
                if (lane < C::LD_LANES) {
                    lds_vec<C::VW>(rb + lane * C::VW, bv);
                    lds_vec<C::VW>(ra + lane * C::VW, av);
                }
                stage_pair(av, bv);
            }
            // the raw slot is consumed: refill it with the pair ST steps ahead
            if (lane == 0) {
                const size_t ahead = pair + size_t(C::ST) * nwarps;
                if (ahead < batch) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    issue(stage, ahead);
                }
            }
            if (++stage == C::ST) {
                stage = 0;
                parity ^= 1u;
            }
            uint64_t lo[C::LPL];
            multiply_staged(lo);
            if (active) {
                uint64_t* po = out + pair * (2 * size_t(mr)) + lane;
#pragma unroll
                for (int k = 0; k < C::LPL; ++k)
                    if (lane + 32 * k < 2 * mr) po[32 * k] = lo[k];
            }
        }
    }
}

template <int NB, bool IL = false>
cudaError_t run_imma(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t batch, int mr, cudaStream_t st) {
    using C = ImmaCfg<NB>;
    const size_t smem = size_t(kImmaWarps) * (IL ? C::WARP_WORDS - C::RAW_WORDS : C::WARP_WORDS) * sizeof(uint32_t);
    // per (host thread, device): the smem opt-in is a per-device function attribute
    static thread_local struct { int dev = -1, grid_cap = 0; } di;
    int dev = 0;
    cudaGetDevice(&dev);
    if (di.dev != dev) {
        int sms = 0, per_sm = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        {  // dynamic + static (the interleaved tile) may pass the 48 KB default either way
            cudaError_t e = cudaFuncSetAttribute(k_mul_imma<NB, IL>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
            if (e != cudaSuccess) return e;
        }
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mul_imma<NB, IL>, kImmaWarps * 32, smem);
        if (e != cudaSuccess) return e;
        di.grid_cap = sms * (per_sm > 0 ? per_sm : 1);
        di.dev = dev;
    }
    const size_t need = (batch + kImmaWarps - 1) / kImmaWarps;
    const size_t grid = need < size_t(di.grid_cap) ? need : size_t(di.grid_cap);
    k_mul_imma<NB, IL><<<unsigned(grid), kImmaWarps * 32, smem, st>>>(out, a, b, batch, mr);
    count_launch();
    return cudaGetLastError();
}

}  // namespace

bool mul_imma_supported(size_t m) {
    return m == 8 || m == 16 || m == 20 || m == 24 || m == 28 || m == 32 || m == 48 || m == 64 || m == 80 ||
           m == 96 || m == 112 || m == 128;
}

cudaError_t launch_mul_imma(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                            cudaStream_t st) {
    if (batch == 0) return cudaSuccess;
    const int mr = int(m);
    switch (m) {
        case 8: return run_imma<2>(out, a, b, batch, mr, st);
        case 16: return run_imma<4>(out, a, b, batch, mr, st);
        case 20: return run_imma<5>(out, a, b, batch, mr, st);
        case 24: return run_imma<6>(out, a, b, batch, mr, st);
        case 28: return run_imma<7>(out, a, b, batch, mr, st);
        case 32: return run_imma<8>(out, a, b, batch, mr, st);
        case 48: return run_imma<12>(out, a, b, batch, mr, st);
        case 64: return run_imma<16>(out, a, b, batch, mr, st);
        case 80: return run_imma<20>(out, a, b, batch, mr, st);
        case 96: return run_imma<24>(out, a, b, batch, mr, st);
        case 112: return run_imma<28>(out, a, b, batch, mr, st);
        case 128: return run_imma<32>(out, a, b, batch, mr, st);
        default: return cudaErrorNotSupported;
    }
}

// Interleaved [m][batch] operands and product, read and written in place (m in {32, 64,
// 128}, and even 16 < m < 128 zero-extended in registers).
cudaError_t launch_mul_imma_il(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                               cudaStream_t st) {
    if (batch == 0) return cudaSuccess;
    if (m <= 16 || m > 128) return cudaErrorNotSupported;  // any m: tile rows past m load as zero
    const int mr = int(m);
    static const int fine = [] {
        const char* e = std::getenv("DOTG_IMMA_FINE");
        return e ? std::atoi(e) : 1;
    }();
    if (m <= 32) return run_imma<8, true>(out, a, b, batch, mr, st);
    if (m <= 64) return run_imma<16, true>(out, a, b, batch, mr, st);
    if (fine && m <= 96) return run_imma<24, true>(out, a, b, batch, mr, st);  // 6 words per lane (even)
    return run_imma<32, true>(out, a, b, batch, mr, st);
}

// Even 16 < m < 128 with 16-byte aligned rows: the next tensor-pipe size's kernel with the
// operand rows zero-extended in shared memory (no padded copies in HBM).
cudaError_t launch_mul_imma_rt(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                               cudaStream_t st) {
    if (batch == 0) return cudaSuccess;
    if (m <= 16 || m >= 128) return cudaErrorNotSupported;  // odd m: the kernel's direct loads
    const int mr = int(m);
    // next multiple of 4 limbs up to 32, of 16 above (DOTG_IMMA_FINE=0: the next power of
    // two, as in r01)
    static const int fine = [] {
        const char* e = std::getenv("DOTG_IMMA_FINE");
        return e ? std::atoi(e) : 1;
    }();
    if (fine && m <= 20) return run_imma<5>(out, a, b, batch, mr, st);
    if (fine && m <= 24) return run_imma<6>(out, a, b, batch, mr, st);
    if (fine && m <= 28) return run_imma<7>(out, a, b, batch, mr, st);
    if (m <= 32) return run_imma<8>(out, a, b, batch, mr, st);
    if (fine && m <= 48) return run_imma<12>(out, a, b, batch, mr, st);
    if (m <= 64) return run_imma<16>(out, a, b, batch, mr, st);
    if (fine && m <= 80) return run_imma<20>(out, a, b, batch, mr, st);
    if (fine && m <= 96) return run_imma<24>(out, a, b, batch, mr, st);
    if (fine && m <= 112) return run_imma<28>(out, a, b, batch, mr, st);
    return run_imma<32>(out, a, b, batch, mr, st);
}

}  // namespace dotg
