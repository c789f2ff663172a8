// mul_umma.cu - batched column multiplication of WIDE operands on the 5th-generation
// tensor core (tcgen05.mma kind::i8, accumulators in tensor memory).
//
// Same contract as every product kernel here (dot_mul_words, include/dot/mul.hpp:75-76,
// src/mul.cpp:96-103: all column sums, one deferred carry pass, exactly 2m limbs), for
// 256 <= m <= 65536 limbs (m % 16 == 0; other sizes are row-padded by the caller), and the
// leaves of the Karatsuba route above (mul_batch.cu, karatsuba.cu).
//
// Why tcgen05 here and mma.sync below 256 limbs: a UMMA with M = 128 reads its A tile
// (4 KB) from shared memory for every instruction, so it only pays when N (the columns
// sharing that tile) is large. One pair's column product offers N = number of a-chunks
// of 128 bytes sharing a b-window - 16 for m = 256, 64 for m = 1024, 256 from m = 4096
// (tools/umma_i8_probe.cu measured the small-N ceiling).
//
// Formulation (bytes; a, b of n = 8m bytes; x = i + j; S[x] = sum a[j] b[i]):
//   j = 128 J + 32 p + (31 - k)        J a-chunk, p in 0..3 its 32-byte block, k the MMA K
//   i = 128 s - 32 p + r + k - 31      s the b-window step, r in 0..127 the TMEM lane
//   => x = 128 (s + J) + r             independent of p and k
// MMA (s, p) over the D tile of output chunks [C0, C0 + NT):
//   A[r][k] = b[128 s - 32 p + r + k - 31]              (Hankel window of b)
//   B[k][c] = a[128 (C0 + c - s) + 32 p + 31 - k]       (a-block 4J + p, byte-reversed)
//   D[r][c] += sum_k A[r][k] B[k][c]    -> D[r][c] = S[128 (C0 + c) + r], no redundancy:
// every (i, j) byte pair is issued exactly once, into the one D entry of its column.
// Only the columns c whose a-chunk exists are issued (N' = that range rounded out to 16,
// zero-padded chunks), so a tile's MMAs are ~90-100 % useful.
//
// Shared-memory operands, K-major, no swizzle (core matrix = 8 rows x 16 bytes):
//   * A: core matrix (g, kk) of MMA (s, p) is C_t with t = 16 s - 4 p + g + 2 kk, where
//     C_t[rr][jj] = b[8 t + rr + jj - 31]. So the Hankel tiles of all (s, p) are windows
//     of ONE array of core matrices (SBO 128 B, LBO 256 B): 16x the b bytes, built per
//     block of kSB s-steps into a kSlots-slot ring by funnel shifts from b staged in
//     shared memory.
//   * B: per (p, kk) an array of 16-byte rows indexed by J (reversed half-blocks), so
//     shifting the a-chunk range by one (next s) is a 16-byte step of the start address
//     (SBO 128 B, LBO = the array length).
// Roles: warps 0-3 stage the operands and build ring slots (mbarrier `full`), warp 4
// issues each slot's MMAs from one elected lane and commits them to the slot's `empty`
// mbarrier. Work items are (pair, D tile, s-range split); m > 4096 splits s into ranges of
// <= 128 steps.
// Accumulation: s32 column sums < (b bytes per item) * 255^2 < 2^31 (<= 32 KB of b per item).
// Epilogue: tcgen05.ld (warp w holds lanes 32w..32w+31 = bytes of 4 limbs per chunk), a
// per-warp transpose through shared memory folds 8 byte columns per limb into lo64 + hi
// (< 2^25); unsplit items resolve every carry of the tile in the CTA (generate / propagate
// ballots, as the add kernel) and store the limbs; a second tile gets the first tile's
// carry word from k_umma_tile_carries; split items store partial limbs that
// k_umma_reduce adds before one batched add resolves LO + HI * 2^64.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "internal.h"

namespace dotg {

namespace {

constexpr int kPadJ = 16;            // zero a-chunks on each side of the B arrays
constexpr int kPadB = 160;           // zero bytes on each side of the staged b
constexpr int kSB = 4;               // s-steps per ring slot
constexpr int kTC = 16 * kSB + 16;   // core matrices per ring slot
constexpr int kSlots = 3;            // ring slots
constexpr int kWorkers = 128;        // builder / epilogue warps 0-3 (TMEM lane quarters)
constexpr int kThreads = 160;        // + warp 4: the MMA issuer
constexpr int kUmmaMaxM = 65536;     // largest m the kernel takes (s-range splits above 4096)
constexpr int kEpiLoBytes = 8 * 18;  // epilogue bytes per D column: 16 limbs (+2 pad) of LO
constexpr int kEpiHiBytes = 4 * 20;  // and 16 (+4 pad) of HI

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// Shared-memory matrix descriptor: K-major, no swizzle, version 1.
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
           (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46);
}
// Instruction descriptor kind::i8: u8 x u8 -> s32, both K-major, M = 128.
__device__ __forceinline__ uint32_t idesc_u8(uint32_t n) { return (2u << 4) | ((n >> 3) << 17) | ((128u >> 4) << 24); }

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\nUMMA_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra UMMA_WAIT_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

// Wait for warps off the critical path: suspended in hardware until the phase completes
// (or the hint elapses), so spinning waiters do not take issue slots from the MMA issuer.
__device__ __forceinline__ void mbar_sleep(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\nUMMA_SLEEP_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra UMMA_SLEEP_%=;\n}" ::"r"(bar),
        "r"(parity), "r"(1000000u)
        : "memory");
}

// The MMAs of one ring slot (s-steps s0 .. s1-1), issued by ONE elected lane of a
// converged warp. Descriptors are linear in the address (14-bit field, 16-byte units):
// A of (s, p) = slot base + 8 (16 (s - s0) + 12 - 4 p); B of (p, row j) = b_p0 + p b_dp + j.
__device__ __forceinline__ void issue_block(uint32_t slot_addr, int s0, int s1, int C0, int na, int nt, uint32_t dbase,
                                            uint64_t b_p0, uint64_t b_dp) {
    const uint64_t a_s0 = sdesc(slot_addr + 12 * 128, 256, 128);
    for (int s = s0; s < s1; ++s) {
        int lo = s - C0, hi = s - C0 + na;
        if (lo < 0) lo = 0;
        if (hi > nt) hi = nt;
        if (hi <= lo) continue;
        const int lo16 = lo & ~15, hi16 = (hi + 15) & ~15;
        const uint32_t id = idesc_u8(uint32_t(hi16 - lo16));
        const uint32_t dcol = dbase + uint32_t(lo16);
        const uint64_t ad = a_s0 + uint64_t(128 * (s - s0));
        const uint64_t bd = b_p0 + uint64_t(C0 + lo16 - s);
        asm volatile(
            "{\n\t.reg .pred pe;\n\t.reg .pred pa;\n\t"
            "elect.sync _|pe, 0xffffffff;\n\t"
            "setp.ne.b32 pa, %4, 0;\n\t"
            "@pe tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, pa;\n\t"
            "@pe tcgen05.mma.cta_group::1.kind::i8 [%0], %5, %6, %3, pa;\n\t"
            "@pe tcgen05.mma.cta_group::1.kind::i8 [%0], %7, %8, %3, pa;\n\t"
            "@pe tcgen05.mma.cta_group::1.kind::i8 [%0], %9, %10, %3, pa;\n\t}" ::"r"(dcol),
            "l"(ad), "l"(bd), "r"(id), "r"(1u), "l"(ad - 32), "l"(bd + b_dp), "l"(ad - 64), "l"(bd + 2 * b_dp),
            "l"(ad - 96), "l"(bd + 3 * b_dp)
            : "memory");
    }
}

__device__ __forceinline__ void commit_elect(uint32_t bar) {
    asm volatile(
        "{\n\t.reg .pred pe;\n\telect.sync _|pe, 0xffffffff;\n\t"
        "@pe tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
        : "memory");
}

// Work decomposition of one product size. An item is (pair, D tile of NT output chunks,
// split of the b-window steps s); m <= 4096 runs every s in one item (the CTA finishes the
// tile's limbs), larger m splits s into ranges of <= 128 steps (column sums of <= 16 KB of
// b per accumulator: < 2^31) whose folded partial limbs a second kernel adds.
struct UmmaPlan {
    int m, na, nt, tiles, splits, ss, cols;
    int jrows;        // a-chunk rows staged per B array (without pads)
    uint32_t la;      // bytes of one B array
    int bmax;         // b bytes staged at most
    uint32_t off_ring, off_b, smem;
};

// min_splits > 1 splits the s-range further (more items for a batch too small to fill the
// SMs); every split keeps >= 32 steps.
inline UmmaPlan umma_plan(int m, int min_splits = 1) {
    UmmaPlan g{};
    g.m = m;
    g.na = m / 16;
    g.nt = 2 * g.na < 256 ? (2 * g.na + 15) & ~15 : 256;
    g.tiles = (2 * g.na + g.nt - 1) / g.nt;
    g.cols = g.nt <= 32 ? 32 : (g.nt <= 64 ? 64 : (g.nt <= 128 ? 128 : 256));
    const int steps = g.na + 1;
    g.splits = g.na <= 256 ? 1 : (steps + 127) / 128;
    if (min_splits > g.splits) g.splits = min_splits < steps / 32 ? min_splits : (steps / 32 > g.splits ? steps / 32 : g.splits);
    g.ss = (steps + g.splits - 1) / g.splits;
    g.jrows = g.splits == 1 ? g.na : (g.na < g.nt + g.ss ? g.na : g.nt + g.ss);
    g.la = uint32_t(g.jrows + 2 * kPadJ) * 16;
    g.bmax = g.splits == 1 ? 8 * m : 128 * (g.ss + 1);
    g.off_ring = 8 * g.la;
    g.off_b = g.off_ring + kSlots * kTC * 128;
    g.smem = g.off_b + uint32_t(g.bmax + 2 * kPadB);
    const uint32_t epi = uint32_t((kEpiLoBytes + kEpiHiBytes) * g.nt + 4 * 16 * 36 * 4);  // LO, HI, transposes
    if (g.smem < epi) g.smem = epi;
    return g;
}

__global__ void __launch_bounds__(kThreads) k_mul_umma(uint64_t* __restrict__ out, uint64_t* __restrict__ carry_words,
                                                     uint64_t* __restrict__ part_lo, uint32_t* __restrict__ part_hi,
                                                     const uint64_t* __restrict__ a, const uint64_t* __restrict__ b,
                                                     const UmmaPlan G, unsigned items,
                                                     unsigned* __restrict__ next_item) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t full[kSlots], empty[kSlots], done;
    __shared__ uint32_t tbase_sh;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int m = G.m, na = G.na, nb = G.na, n = 8 * m;
    // barriers: full[q] (4 builder warps arrive), empty[q] (MMA commit), done (last commit)
    if (tid == 0) {
        for (int q = 0; q < kSlots; ++q) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(smem_u32(&full[q])) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[q])) : "memory");
        }
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase_sh)),
                     "r"(G.cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tbase_sh;
    unsigned it = 0;   // items done by this CTA (phase of `done`)
    unsigned qg = 0;   // ring blocks issued so far (phases of full / empty)
    // items: blockIdx.x first, then taken from a global counter (dynamic balance across SMs)
    __shared__ unsigned item_sh;
    for (unsigned item = blockIdx.x; item < items; ++it) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int split = int(item % unsigned(G.splits));
        const int C0 = int((item / unsigned(G.splits)) % unsigned(G.tiles)) * G.nt;
        const size_t pair = item / unsigned(G.splits * G.tiles);
        // this item's b-window steps, the a-chunks they pair with, the b bytes they read
        const int s_lo = split * G.ss, s_hi = s_lo + G.ss < nb + 1 ? s_lo + G.ss : nb + 1;
        const int j_lo = C0 - s_hi + 1 > 0 ? C0 - s_hi + 1 : 0;
        const int j_hi = C0 + G.nt - s_lo < na ? C0 + G.nt - s_lo : na;
        const int b_lo = 128 * s_lo - 128 > 0 ? 128 * s_lo - 128 : 0;
        const int b_hi = 128 * s_hi < n ? 128 * s_hi : n;
        const int nbs = b_hi - b_lo;  // staged b bytes (a multiple of 128)
        uint8_t* bh = sm;                       // 8 arrays [p][kk], rows J - j_lo + kPadJ of 16 B
        uint8_t* ring = sm + G.off_ring;        // kSlots slots x kTC core matrices
        uint8_t* bs = sm + G.off_b;             // kPadB zeros | b[b_lo, b_hi) | kPadB zeros
        const uint4* ga = reinterpret_cast<const uint4*>(a + pair * size_t(m));
        const uint4* gb = reinterpret_cast<const uint4*>(b + pair * size_t(m) + size_t(b_lo / 8));

        // a -> B arrays: 16-byte segment g of the operand is half (g & 1) of block 4J + p,
        // J = g / 8, p = (g / 2) % 4; stored byte-reversed as row J of array (p, kk = 1 - half).
        const int g_lo = 8 * j_lo, g_hi = j_hi > j_lo ? 8 * j_hi : g_lo;
        for (int g0 = g_lo + tid; g0 < g_hi; g0 += 4 * kThreads) {  // 4 loads in flight
            uint4 w[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) w[u] = g0 + u * kThreads < g_hi ? __ldg(ga + g0 + u * kThreads) : make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int g = g0 + u * kThreads;
                if (g >= g_hi) break;
                const int J = g >> 3, p = (g >> 1) & 3, kk = 1 - (g & 1);
                *reinterpret_cast<uint4*>(bh + (2 * p + kk) * G.la + (J - j_lo + kPadJ) * 16) =
                    make_uint4(bswap32(w[u].w), bswap32(w[u].z), bswap32(w[u].y), bswap32(w[u].x));
            }
        }
        const int rows = j_hi > j_lo ? j_hi - j_lo : 0;
        for (int e = tid; e < 8 * 2 * kPadJ; e += kThreads) {  // zero chunks on both sides
            const int arr = e / (2 * kPadJ), q = e % (2 * kPadJ);
            const int row = q < kPadJ ? q : rows + q;
            *reinterpret_cast<uint4*>(bh + arr * G.la + row * 16) = make_uint4(0, 0, 0, 0);
        }
        for (int g0 = tid; g0 < nbs / 16; g0 += 4 * kThreads) {
            uint4 w[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) w[u] = g0 + u * kThreads < nbs / 16 ? __ldg(gb + g0 + u * kThreads) : make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (g0 + u * kThreads < nbs / 16) reinterpret_cast<uint4*>(bs + kPadB)[g0 + u * kThreads] = w[u];
        }
        for (int e = tid; e < 2 * kPadB / 16; e += kThreads) {
            const int off = e < kPadB / 16 ? e * 16 : kPadB + nbs + (e - kPadB / 16) * 16;
            *reinterpret_cast<uint4*>(bs + off) = make_uint4(0, 0, 0, 0);
        }
        if (warp < 4) {  // zero the accumulator tile (every MMA accumulates)
            const uint32_t z = 0;
            for (int c = 0; c < G.nt; c += 16)
                asm volatile(
                    "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                        tm + (uint32_t(warp * 32) << 16) + uint32_t(c)),
                    "r"(z)
                    : "memory");
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();

        const int nblocks = (s_hi - s_lo + kSB - 1) / kSB;  // s = s_lo .. s_hi-1 in blocks of kSB steps
        if (warp < 4) {
            // builders: ring slot q % kSlots <- core matrices t = 16 s0 - 12 + (row / 8), row rr = row % 8
            const uint32_t* bw = reinterpret_cast<const uint32_t*>(bs);
            for (int q = 0; q < nblocks; ++q) {
                const unsigned qq = qg + unsigned(q);
                const int slot = int(qq % kSlots), s0 = s_lo + q * kSB;
                if (qq >= unsigned(kSlots)) mbar_sleep(smem_u32(&empty[slot]), (qq / kSlots - 1) & 1u);
                uint8_t* rs = ring + slot * (kTC * 128);
                const int t0 = 16 * s0 - 12;
#pragma unroll 2
                for (int row = tid; row < kTC * 8; row += kWorkers) {
                    const int o = 8 * (t0 + (row >> 3)) + (row & 7) - 31 - b_lo + kPadB;  // byte offset in bs
                    uint4 v = make_uint4(0, 0, 0, 0);
                    if (o + 16 > kPadB && o < kPadB + nbs) {
                        const int w0 = o >> 2, sh = (o & 3) * 8;
                        const uint32_t x0 = bw[w0], x1 = bw[w0 + 1], x2 = bw[w0 + 2], x3 = bw[w0 + 3], x4 = bw[w0 + 4];
                        v = make_uint4(__funnelshift_r(x0, x1, sh), __funnelshift_r(x1, x2, sh),
                                       __funnelshift_r(x2, x3, sh), __funnelshift_r(x3, x4, sh));
                    }
                    *reinterpret_cast<uint4*>(rs + row * 16) = v;
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[slot])) : "memory");
            }
        } else {
            // issuer: warp 4 (converged, one elected lane issues), MMAs of a slot once its 4
            // builder warps arrived
            // B row of chunk J is J - j_lo + kPadJ (issue_block adds J)
            const uint64_t b_p0 = sdesc(smem_u32(bh) + kPadJ * 16, G.la, 128) - uint64_t(j_lo);
            const uint64_t b_dp = uint64_t(2 * G.la / 16);
            for (int q = 0; q < nblocks; ++q) {
                const unsigned qq = qg + unsigned(q);
                const int slot = int(qq % kSlots), s0 = s_lo + q * kSB;
                mbar_wait(smem_u32(&full[slot]), (qq / kSlots) & 1u);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                issue_block(smem_u32(ring + slot * (kTC * 128)), s0, s0 + kSB < s_hi ? s0 + kSB : s_hi, C0, na, G.nt, tm,
                            b_p0, b_dp);
                commit_elect(smem_u32(&empty[slot]));
                if (q == nblocks - 1) commit_elect(smem_u32(&done));
            }
        }
        qg += unsigned(nblocks);
        mbar_sleep(smem_u32(&done), it & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

        // Epilogue (all operand shared memory is free now).
        // E1: per 16 columns, warp w's lanes hold byte 32w + lane of each output chunk; a
        // per-warp transpose through shared memory gives each thread all 8 byte columns of
        // one limb: V = sum_u S[u] 2^(8u) = lo + hi 2^64 (hi < 2^25), kept as LO / HI.
        const int xend = 2 * na - C0 < G.nt ? 2 * na - C0 : G.nt;  // columns inside the product
        const int xe16 = (xend + 15) & ~15;                         // + zero columns up to 16
        const int nl = 16 * xe16;                                   // limbs resolved (multiple of 256)
        // padded layouts keep the transpose and the limb stores free of bank conflicts:
        // Tw rows of 36 words; limb L of LO at L + 2 (L >> 4), of HI at L + 4 (L >> 4)
        uint64_t* LO = reinterpret_cast<uint64_t*>(sm);
        uint32_t* HI = reinterpret_cast<uint32_t*>(sm + kEpiLoBytes * G.nt);
        uint32_t* Tw = reinterpret_cast<uint32_t*>(sm + (kEpiLoBytes + kEpiHiBytes) * G.nt) + warp * (16 * 36);
        auto lx = [](int L) { return L + 2 * (L >> 4); };
        auto hx = [](int L) { return L + 4 * (L >> 4); };
        for (int c0 = 0; c0 < (warp < 4 ? xe16 : 0); c0 += 16) {
            uint32_t v[16];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                : "r"(tm + (uint32_t(warp * 32) << 16) + uint32_t(c0)));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 16; ++j) Tw[j * 36 + lane] = v[j];
            __syncwarp();
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = (lane & 7) + 8 * h, u = lane >> 3;  // round h: columns 8h..8h+7 x 4 limbs
                {
                    const uint4 q0 = *reinterpret_cast<const uint4*>(Tw + c * 36 + 8 * u);
                    const uint4 q1 = *reinterpret_cast<const uint4*>(Tw + c * 36 + 8 * u + 4);
                    const uint64_t x = uint64_t(q0.x) + (uint64_t(q0.y) << 8) + (uint64_t(q0.z) << 16) + (uint64_t(q0.w) << 24);
                    const uint64_t y = uint64_t(q1.x) + (uint64_t(q1.y) << 8) + (uint64_t(q1.z) << 16) + (uint64_t(q1.w) << 24);
                    const uint64_t lo = x + (y << 32);
                    const int L = 16 * (c0 + c) + 4 * warp + u;
                    LO[lx(L)] = lo;
                    HI[hx(L)] = uint32_t(y >> 32) + (lo < x ? 1u : 0u);
                }
            }
            __syncwarp();
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        if (G.splits > 1) {
            // partial limbs of this s-range: a second kernel adds the splits and the carries
            const size_t base = (pair * size_t(G.splits) + size_t(split)) * size_t(2 * m) + size_t(16 * C0);
            for (int e = tid; e < 16 * xend; e += kThreads) {
                part_lo[base + e] = LO[lx(e)];
                part_hi[base + e] = HI[hx(e)];
            }
        } else {
            // E2: the tile's limbs = LO + HI shifted one limb, carries resolved in the CTA with the
            // add kernel's generate / propagate algebra. Warp w owns limbs [w nl/4, (w+1) nl/4) in
            // rounds of 32 consecutive limbs (lane = limb, conflict-free): pass 1 folds the rounds
            // into the warp's (carry-out, all-propagate), pass 2 applies the carries.
            {
                const int per_warp = nl / 4, rounds = per_warp / 32;  // nl = 16 * xe16 -> rounds >= 2
                const int base = warp * per_warp;
                __shared__ uint32_t wagg[4][2];
                if (warp < 4) {
                    uint32_t Gw = 0, Pw = 1;
                    for (int r = 0; r < rounds; ++r) {
                        const int L = base + 32 * r + lane;
                        const uint64_t lo = LO[lx(L)];
                        const uint64_t sv = lo + (L > 0 ? uint64_t(HI[hx(L - 1)]) : 0ull);
                        const uint32_t g = __ballot_sync(0xffffffffu, sv < lo), pp = __ballot_sync(0xffffffffu, sv == ~0ull);
                        const uint32_t go = uint32_t(((uint64_t(g) << 1) + pp) >> 32);  // round carry-out, carry-in 0
                        Gw = go | ((pp == 0xffffffffu) & Gw);
                        Pw &= pp == 0xffffffffu;
                    }
                    if (lane == 0) {
                        wagg[warp][0] = Gw;
                        wagg[warp][1] = Pw;
                    }
                }
                __syncthreads();
                if (warp < 4) {
                    uint32_t c = 0;
                    for (int w = 0; w < warp; ++w) c = wagg[w][0] | (wagg[w][1] & c);
                    for (int r = 0; r < rounds; ++r) {
                        const int L = base + 32 * r + lane;
                        const uint64_t lo = LO[lx(L)];
                        const uint64_t sv = lo + (L > 0 ? uint64_t(HI[hx(L - 1)]) : 0ull);
                        const uint32_t g = __ballot_sync(0xffffffffu, sv < lo), pp = __ballot_sync(0xffffffffu, sv == ~0ull);
                        const uint64_t y = ((uint64_t(g) << 1) | c) + pp;
                        LO[lx(L)] = sv + (uint32_t((y ^ pp) >> lane) & 1u);
                        c = uint32_t(y >> 32);
                    }
                    if (warp == 3 && lane == 31 && G.tiles > 1)  // carry word into the next tile
                        carry_words[pair * size_t(G.tiles) + size_t(C0 / G.nt)] = uint64_t(HI[hx(nl - 1)]) + c;
                }
            }
            __syncthreads();
            {
                uint64_t* orow = out + pair * size_t(2 * m) + size_t(16 * C0);
                for (int e = tid; e < 8 * xend; e += kThreads)
                    reinterpret_cast<uint4*>(orow)[e] = *reinterpret_cast<const uint4*>(LO + lx(2 * e));
            }
        }
        if (tid == 0) item_sh = next_item != nullptr ? gridDim.x + atomicAdd(next_item, 1u) : items;
        __syncthreads();  // epilogue done with shared memory and TMEM before the next item stages
        item = item_sh;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(G.cols) : "memory");
}

// Tiles after the first were resolved with carry-in 0: add each tile's carry word at the
// next tile's first limb, propagating (one thread per pair; the additions commute).
__global__ void k_umma_tile_carries(uint64_t* __restrict__ out, const uint64_t* __restrict__ cw, size_t m,
                                    size_t batch, int tiles, int tile_limbs) {
    const size_t pair = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (pair >= batch) return;
    uint64_t* row = out + pair * 2 * m;
    for (int t = 1; t < tiles; ++t) {
        uint64_t add = cw[pair * tiles + t - 1];
        for (size_t L = size_t(t) * tile_limbs; add != 0 && L < 2 * m; ++L) {
            const uint64_t s = row[L] + add;
            add = s < add ? 1u : 0u;
            row[L] = s;
        }
    }
}

// Split items: out[L] = sum of the splits' low words, next[L + 1] = their high words plus
// the low-word carries (then one batched add resolves out + next).
__global__ void k_umma_reduce(uint64_t* __restrict__ out, uint64_t* __restrict__ next,
                              const uint64_t* __restrict__ part_lo, const uint32_t* __restrict__ part_hi, size_t m,
                              size_t batch, int splits) {
    const size_t idx = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= batch * 2 * m) return;
    const size_t pair = idx / (2 * m), L = idx % (2 * m);
    uint64_t lo = 0, hi = 0;
    for (int sp = 0; sp < splits; ++sp) {
        const size_t k = (pair * size_t(splits) + size_t(sp)) * 2 * m + L;
        const uint64_t v = part_lo[k];
        lo += v;
        hi += (lo < v ? 1u : 0u) + uint64_t(part_hi[k]);
    }
    out[idx] = lo;
    if (L + 1 < 2 * m) next[idx + 1] = hi;
    if (L == 0) next[idx] = 0;
}

uint32_t umma_max_smem() {
    uint32_t mx = 0;
    for (int m = 256; m <= kUmmaMaxM; m += 16) {
        const UmmaPlan G = umma_plan(m);
        const int per_sm = 512 / G.cols < 8 ? 512 / G.cols : 8;
        const uint32_t floor_smem = uint32_t(228 * 1024 / (per_sm + 1)) + 16;
        const uint32_t smem = G.smem > floor_smem ? G.smem : floor_smem;
        if (smem > mx) mx = smem;
    }
    return mx;
}

}  // namespace

bool mul_umma_supported(size_t m) {
    static const int enabled = [] {
        const char* e = std::getenv("DOTG_MUL_UMMA");
        return e ? std::atoi(e) : 1;
    }();
    return enabled != 0 && m >= 256 && m <= size_t(kUmmaMaxM) && m % 16 == 0;
}

size_t mul_umma_direct_max() {
    static const size_t v = [] {
        const char* e = std::getenv("DOTG_UMMA_DIRECT");
        const long x = e ? std::atol(e) : kUmmaMaxM;
        return size_t(x >= 256 && x <= kUmmaMaxM ? x : kUmmaMaxM);
    }();
    return v;
}

size_t mul_umma_leaf(size_t m, size_t batch) {
    // Karatsuba level passes are latency-bound for a handful of huge numbers, so few levels
    // over big leaves win when the batch holds little work; with more limbs in flight the
    // 25% of products saved per level win (tools/umma_timing.py,
    // profiles/r02_umma_wide_variants.txt).
    static const long env = [] {
        const char* e = std::getenv("DOTG_UMMA_LEAF");
        return e ? std::atol(e) : 0L;
    }();
    if (env >= 256 && env <= kUmmaMaxM && (env & (env - 1)) == 0) return size_t(env);
    const double limbs = double(m) * double(batch);
    return limbs <= double(1 << 17) ? size_t(65536) : (limbs <= double(1 << 18) ? size_t(16384) : size_t(4096));
}

cudaError_t launch_mul_umma(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                            cudaStream_t st) {
    if (batch == 0) return cudaSuccess;
    if (!(m >= 256 && m <= size_t(kUmmaMaxM) && m % 16 == 0)) return cudaErrorInvalidValue;
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
            sms = 148;
    }
    // DOTG_UMMA_FILL=1: a batch with fewer (pair, tile) items than CTA slots gets its s-range
    // split so every SM holds MMA streams. Measured slower in most shapes (the split items'
    // partial limbs, reduce and batched add cost more than the idle SMs:
    // profiles/r02_umma_wide_variants.txt), so off by default.
    static const int fill = std::getenv("DOTG_UMMA_FILL") ? std::atoi(std::getenv("DOTG_UMMA_FILL")) : 0;
    UmmaPlan G = umma_plan(int(m));
    {
        const int per_sm0 = 512 / G.cols < 8 ? 512 / G.cols : 8;
        const size_t slots = size_t(sms) * size_t(per_sm0);
        const size_t base = batch * size_t(G.tiles);
        if (fill && G.splits == 1 && base < slots) G = umma_plan(int(m), int((slots + base - 1) / base));
    }
    if (G.splits > 1) {  // partial limbs: 12 B per limb per split; keep them under 1 GiB per launch
        const size_t per_pair = size_t(G.splits) * 2 * m * 12 + 2 * m * 8;
        const size_t chunk = (size_t(1) << 30) / per_pair > 0 ? (size_t(1) << 30) / per_pair : 1;
        if (batch > chunk) {
            for (size_t p0 = 0; p0 < batch; p0 += chunk) {
                const size_t nb = batch - p0 < chunk ? batch - p0 : chunk;
                const cudaError_t e = launch_mul_umma(out + p0 * 2 * m, a + p0 * m, b + p0 * m, m, nb, st);
                if (e != cudaSuccess) return e;
            }
            return cudaSuccess;
        }
    }
    cudaError_t e = cudaSuccess;
    const size_t items = batch * size_t(G.tiles) * size_t(G.splits);
    if (items > size_t(0x7fffffff)) return cudaErrorInvalidConfiguration;
    retain_stream_pool();
    uint64_t *cw = nullptr, *plo = nullptr, *nxt = nullptr;
    uint32_t* phi = nullptr;
    if (G.splits > 1) {
        e = cudaMallocAsync(&plo, batch * size_t(G.splits) * 2 * m * 8, st);
        if (e == cudaSuccess) e = cudaMallocAsync(&phi, batch * size_t(G.splits) * 2 * m * 4, st);
        if (e == cudaSuccess) e = cudaMallocAsync(&nxt, batch * 2 * m * 8, st);
    } else if (G.tiles > 1) {
        e = cudaMallocAsync(&cw, batch * size_t(G.tiles) * 8, st);
    }
    // occupancy: TMEM holds 512 columns per SM, so ask for enough shared memory that no
    // more CTAs than that fit (a CTA waiting in tcgen05.alloc would hold its SM slot)
    const int per_sm = 512 / G.cols < 8 ? 512 / G.cols : 8;
    const uint32_t floor_smem = uint32_t(228 * 1024 / (per_sm + 1)) + 16;
    const uint32_t smem = G.smem > floor_smem ? G.smem : floor_smem;
    // the largest dynamic shared memory any size needs, set once per process (not a stream
    // operation, so launches stay capturable into CUDA graphs)
    static const cudaError_t attr = [] {
        cudaError_t r = cudaFuncSetAttribute(k_mul_umma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(umma_max_smem()));
        if (r == cudaSuccess)
            r = cudaFuncSetAttribute(k_mul_umma, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     int(cudaSharedmemCarveoutMaxShared));
        return r;
    }();
    if (e == cudaSuccess) e = attr;
    // persistent: as many CTAs as fit (TMEM and shared memory), each looping over items
    // CTAs per SM: TMEM columns and shared memory (228 KB per SM, 1 KB reserved per CTA plus
    // the static barriers); cudaOccupancyMaxActiveBlocksPerMultiprocessor reports 1 here (it
    // assumes the carveout of the largest dynamic size set on the function).
    int occ = int((228 * 1024) / (smem + 2048));
    if (occ > per_sm) occ = per_sm;
    if (occ < 1) occ = 1;
    // DOTG_UMMA_PERSIST=P > 0: P CTAs per SM slot, items taken from a global counter (same
    // speed as one CTA per item, measured: profiles/r02_umma_wide_variants.txt); default 0
    static const int persist = std::getenv("DOTG_UMMA_PERSIST") ? std::atoi(std::getenv("DOTG_UMMA_PERSIST")) : 0;
    const size_t cap = persist > 0 ? size_t(sms) * size_t(occ) * size_t(persist) : items;
    const size_t grid = items < cap ? items : cap;
    unsigned* ctr = nullptr;
    if (e == cudaSuccess && grid < items) {
        e = cudaMallocAsync(&ctr, sizeof(unsigned), st);
        if (e == cudaSuccess) e = cudaMemsetAsync(ctr, 0, sizeof(unsigned), st);
    }
    if (e == cudaSuccess) {
        k_mul_umma<<<unsigned(grid), kThreads, smem, st>>>(out, cw, plo, phi, a, b, G, unsigned(items), ctr);
        count_launch();
        e = cudaGetLastError();
    }
    if (ctr != nullptr) cudaFreeAsync(ctr, st);
    if (e == cudaSuccess && G.splits > 1) {
        k_umma_reduce<<<unsigned((batch * 2 * m + 255) / 256), 256, 0, st>>>(out, nxt, plo, phi, m, batch, G.splits);
        count_launch();
        e = cudaGetLastError();
        if (e == cudaSuccess) e = launch_addsub_batch(false, out, out, nxt, nullptr, 2 * m, batch, 0, st);
    }
    if (e == cudaSuccess && G.splits == 1 && G.tiles > 1) {
        k_umma_tile_carries<<<unsigned((batch + 127) / 128), 128, 0, st>>>(out, cw, m, batch, G.tiles, 16 * G.nt);
        count_launch();
        e = cudaGetLastError();
    }
    for (void* q : {static_cast<void*>(plo), static_cast<void*>(phi), static_cast<void*>(nxt)})
        if (q != nullptr) cudaFreeAsync(q, st);
    if (cw != nullptr) cudaFreeAsync(cw, st);
    return e;
}

}  // namespace dotg
