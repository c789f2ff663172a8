// addsub_long.cu - one long number (up to 2^30+ limbs), tiled over the whole GPU and
// shardable by limb range across GPUs (config 5).
//
// Replaces the reference's span-form dot_add_words / dot_sub_words on long operands
// (include/dot/addsub.hpp:98-103, src/addsub.cpp:136-170), where a long number is a
// serial chain of w-limb chunks whose carry-out is the next chunk's carry-in
// (addsub.cpp:147-164). Here the chain is replaced by a (G, P) scan at three levels:
//
//   pass 1  k_long_local   one CTA per tile of 4096 limbs: phases 1-2 per limb,
//                          ballot masks per warp row, one mask addition per 32-bit
//                          word + one per tile (two-level lookahead in shared memory),
//                          phase-4 carry application, store. The tile's carry-in is
//                          unknown in this pass and treated as 0, EXCEPT that the
//                          tile's leading propagate run [0, pt) - the only limbs whose
//                          value depends on that carry-in, besides limb pt itself - is
//                          not written (deferred). State per tile: pt, tile G, tile P.
//   pass 2  k_long_scan_chunks + k_long_shard_agg: one CTA per 1024 tiles scans the tile
//                          (G, P) symbolically in the unknown carry-in X with warp
//                          ballots (cin_t = g_ex | (p_ex & X) relative to the chunk),
//                          one warp composes the chunk aggregates into the shard
//                          aggregate {G, P} (8 bytes) for the cross-GPU exchange.
//   pass 3  k_long_finish  X from the gathered shard aggregates, the chunk carry-in from
//                          a ballot scan of the chunk aggregates; per tile: write the
//                          deferred prefix as the propagate value for cin_t and bump
//                          limb pt by cin_t. This is the reference's rare Phase 4
//                          (addsub.cpp:61-79) lifted to tiles: on random data it is one
//                          8-byte read-modify-write per tile with cin_t = 1.
//
// Traffic is the algorithmic 24 B/limb plus ~8 B per tile; a long all-propagate run is
// written exactly once (by pass 3), never rewritten. No CTA waits on another CTA.
#include <cuda_runtime.h>

#include <cstdint>

#include "device.cuh"
#include "internal.h"

namespace dotg {

namespace {

constexpr int kThreads = 256;            // threads per tile CTA
constexpr int kRows = 4;                 // vectors per thread
constexpr int kV = 4;                    // limbs per vector (256-bit)
constexpr int kTile = kThreads * kRows * kV;  // 4096 limbs
constexpr int kWords = kTile / kV / 32;  // 32 ballot words per tile

// State word per tile: bits [0,16) pt, 16 tile G, 17 tile P, 18 g_ex, 19 p_ex.
constexpr uint32_t kBitG = 1u << 16, kBitP = 1u << 17, kBitGex = 1u << 18, kBitPex = 1u << 19;

size_t num_tiles(size_t m) { return (m + kTile - 1) / kTile; }

template <bool SUB, bool VEC>
__global__ void __launch_bounds__(kThreads) k_long_local(uint64_t* out, const uint64_t* a,
                                                         const uint64_t* b, size_t m,
                                                         uint32_t* state, size_t sw) {
    __shared__ uint32_t sG[kWords], sP[kWords], sC[kWords];
    __shared__ uint32_t s_pt;
    // grid.y = independent numbers of m limbs each (batch of long numbers), state regions
    // of sw words apiece; grid.y = 1 for the single number / shard
    out += size_t(blockIdx.y) * m;
    a += size_t(blockIdx.y) * m;
    b += size_t(blockIdx.y) * m;
    state += size_t(blockIdx.y) * sw;
    const size_t tile = blockIdx.x;
    const size_t L0 = tile * size_t(kTile);
    const size_t len = (m - L0) < size_t(kTile) ? (m - L0) : size_t(kTile);
    const bool full = len == size_t(kTile);
    const unsigned tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;

    uint64_t s[kRows][kV], y[kRows][kV];
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
        const size_t o = size_t(r * kThreads + tid) * kV;  // limb offset within tile
        if (VEC && full) {
            ld_stream<kV>(a + L0 + o, s[r]);
            ld_stream<kV>(b + L0 + o, y[r]);
        } else {
#pragma unroll
            for (int k = 0; k < kV; ++k) {
                const bool in = o + k < len;
                s[r][k] = in ? a[L0 + o + k] : (SUB ? 0ull : ~0ull);  // fake limbs propagate
                y[r][k] = in ? b[L0 + o + k] : 0ull;
            }
        }
    }
    uint32_t g[kRows][kV], p[kRows][kV];
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
#pragma unroll
        for (int k = 0; k < kV; ++k) s[r][k] = lane_op<SUB>(s[r][k], y[r][k], g[r][k], p[r][k]);
        uint32_t G, P;
        fold_gp<kV>(g[r], p[r], G, P);
        const uint32_t gw = __ballot_sync(0xffffffffu, G);
        const uint32_t pw = __ballot_sync(0xffffffffu, P);
        if (lane == 0) {
            sG[r * (kThreads / 32) + warp] = gw;
            sP[r * (kThreads / 32) + warp] = pw;
        }
    }
    if (tid == 0) s_pt = 0xffffffffu;
    __syncthreads();

    uint32_t tileG = 0, tileP = 0;
    if (warp == 0) {
        // Word level: lane i owns ballot word i (super-lanes 32i .. 32i+31).
        const uint32_t G = sG[lane], P = sP[lane];
        const uint64_t y0 = (uint64_t(G) << 1) + uint64_t(P);
        const uint32_t wg = uint32_t(y0 >> 32) & 1u;
        const uint32_t wp = P == 0xffffffffu;
        // Tile level: one more mask addition over the 32 words (tile carry-in = 0).
        const uint32_t GW = __ballot_sync(0xffffffffu, wg);
        const uint32_t PW = __ballot_sync(0xffffffffu, wp);
        const uint64_t yw = (uint64_t(GW) << 1) + uint64_t(PW);
        const uint32_t cin = uint32_t((yw ^ uint64_t(PW)) >> lane) & 1u;
        sC[lane] = uint32_t(((uint64_t(G) << 1 | cin) + uint64_t(P)) ^ uint64_t(P));
        tileG = uint32_t(yw >> 32) & 1u;
        tileP = PW == 0xffffffffu;
    }
    __syncthreads();

    // Locate the first non-propagate super-lane from shared memory (cheap, uniform).
    unsigned js = kWords * 32;
#pragma unroll 1
    for (int w = 0; w < kWords; ++w) {
        const uint32_t pw = sP[w];
        if (pw != 0xffffffffu) {
            js = unsigned(w) * 32u + unsigned(__ffs(~pw) - 1);
            break;
        }
    }

#pragma unroll
    for (int r = 0; r < kRows; ++r) {
        const unsigned j = unsigned(r * kThreads) + tid;
        const uint32_t c = (sC[j >> 5] >> (j & 31u)) & 1u;
        apply_superlane<SUB, kV>(s[r], g[r], p[r], c);
        const size_t o = size_t(j) * kV;
        if (j > js) {
            if (VEC && full) {
                st_stream<kV>(out + L0 + o, s[r]);
            } else {
#pragma unroll
                for (int k = 0; k < kV; ++k)
                    if (o + k < len) out[L0 + o + k] = s[r][k];
            }
        } else if (j == js) {
            // Owner of the first non-propagate super-lane: limbs before its first
            // non-propagate limb belong to the deferred prefix.
            int k0 = kV;
#pragma unroll
            for (int k = kV - 1; k >= 0; --k)
                if (!p[r][k]) k0 = k;
#pragma unroll
            for (int k = 0; k < kV; ++k)
                if (k >= k0 && o + k < len) out[L0 + o + k] = s[r][k];
            const size_t pt = o + size_t(k0);
            s_pt = uint32_t(pt < len ? pt : len);
        }
    }
    __syncthreads();
    if (tid == 0) {
        const uint32_t pt = s_pt == 0xffffffffu ? uint32_t(len) : s_pt;
        state[tile] = pt | (tileG ? kBitG : 0u) | (tileP ? kBitP : 0u);
    }
}

// Compose (g1,p1) then (g2,p2): carry out of the concatenation (lower part first).
__device__ __forceinline__ void compose(uint32_t& g, uint32_t& p, uint32_t g2, uint32_t p2) {
    g = g2 | (p2 & g);
    p = p & p2;
}

// Compose 32 lanes' (g, p) (lane 0 lowest) with two mask additions: returns each lane's
// exclusive prefix (eg, ep) and the aggregate of all 32 (ag, ap). cin = eg | (ep & X).
__device__ __forceinline__ void warp_scan_gp(uint32_t g, uint32_t p, unsigned lane, uint32_t& eg, uint32_t& ep,
                                             uint32_t& ag, uint32_t& ap) {
    const uint32_t GW = __ballot_sync(0xffffffffu, g);
    const uint32_t PW = __ballot_sync(0xffffffffu, p);
    const uint64_t y0 = (uint64_t(GW) << 1) + PW;          // carry-in X = 0
    const uint64_t y1 = ((uint64_t(GW) << 1) | 1u) + PW;   // carry-in X = 1
    const uint32_t c0 = uint32_t(y0 ^ PW), c1 = uint32_t(y1 ^ PW);
    eg = (c0 >> lane) & 1u;
    ep = ((c1 ^ c0) >> lane) & 1u;
    ag = uint32_t(y0 >> 32) & 1u;
    ap = PW == 0xffffffffu;
}

constexpr int kChunk = 1024;  // tiles per scan chunk (one CTA of pass 2)

// Pass 2a: one CTA per chunk of 1024 tiles. Each tile gets its exclusive (g, p) relative
// to the chunk start; each chunk its aggregate (bit 0 G, bit 1 P).
__global__ void __launch_bounds__(kChunk) k_long_scan_chunks(uint32_t* state, size_t n, uint32_t* chunk_agg,
                                                              size_t sw) {
    __shared__ uint32_t swg[32], swp[32];
    state += size_t(blockIdx.y) * sw;
    chunk_agg += size_t(blockIdx.y) * sw;
    const unsigned tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const size_t t = size_t(blockIdx.x) * kChunk + tid;
    const uint32_t st = t < n ? state[t] : kBitP;  // identity (G = 0, P = 1) past the end
    uint32_t lg, lp, wg, wp;
    warp_scan_gp((st & kBitG) ? 1u : 0u, (st & kBitP) ? 1u : 0u, lane, lg, lp, wg, wp);
    if (lane == 0) {
        swg[warp] = wg;
        swp[warp] = wp;
    }
    __syncthreads();
    if (warp == 0) {
        uint32_t eg, ep, cg, cp;
        warp_scan_gp(swg[lane], swp[lane], lane, eg, ep, cg, cp);
        __syncwarp();
        swg[lane] = eg;
        swp[lane] = ep;
        if (lane == 0) chunk_agg[blockIdx.x] = cg | (cp << 1);
    }
    __syncthreads();
    uint32_t eg = swg[warp], ep = swp[warp];
    compose(eg, ep, lg, lp);
    if (t < n) state[t] = (st & (0xffffu | kBitG | kBitP)) | (eg ? kBitGex : 0u) | (ep ? kBitPex : 0u);
}

// Exclusive (g, p) over chunk aggregates [0, c) (whole warp, result in every lane).
__device__ __forceinline__ void chunk_prefix(const uint32_t* chunk_agg, size_t c, unsigned lane, uint32_t& g,
                                             uint32_t& p) {
    g = 0;
    p = 1;
    for (size_t base = 0; base < c; base += 32) {
        const size_t k = base + lane;
        const uint32_t v = k < c ? chunk_agg[k] : 2u;  // identity past c
        uint32_t eg, ep, ag, ap;
        warp_scan_gp(v & 1u, (v >> 1) & 1u, lane, eg, ep, ag, ap);
        compose(g, p, ag, ap);
    }
}

// Pass 2b: shard aggregate {G, P} = composition of all chunk aggregates.
__global__ void __launch_bounds__(32) k_long_shard_agg(const uint32_t* chunk_agg, size_t nchunks, uint32_t* agg,
                                                       size_t sw) {
    chunk_agg += size_t(blockIdx.y) * sw;
    agg += 2 * size_t(blockIdx.y);
    uint32_t g, p;
    chunk_prefix(chunk_agg, nchunks, threadIdx.x, g, p);
    if (threadIdx.x == 0) {
        agg[0] = g;
        agg[1] = p;
    }
}

// Pass 3: resolve the shard carry-in X from the gathered aggregates, then fix up each
// tile whose carry-in is 1 or whose leading propagate run was deferred.
template <bool SUB>
__global__ void __launch_bounds__(256) k_long_finish(uint64_t* out, size_t m, const uint32_t* state,
                                                     const uint32_t* chunk_agg, size_t n,
                                                     const uint32_t* all_aggs, int rank, int world,
                                                     uint32_t* carry_out, size_t sw) {
    // grid.y > 1: a batch of independent numbers (world = 1, own aggregate, own carry)
    out += size_t(blockIdx.y) * m;
    state += size_t(blockIdx.y) * sw;
    chunk_agg += size_t(blockIdx.y) * sw;
    all_aggs += 2 * size_t(blockIdx.y);
    if (carry_out != nullptr) carry_out += blockIdx.y;
    uint32_t x = 0;  // carry into this shard
    uint32_t total = 0;
    for (int q = 0; q < world; ++q) {
        const uint32_t G = all_aggs[2 * q], P = all_aggs[2 * q + 1];
        if (q == rank) x = total;
        total = G | (P & total);
    }
    if (carry_out != nullptr && blockIdx.x == 0 && threadIdx.x == 0) *carry_out = total;

    const unsigned lane = threadIdx.x & 31u;
    const size_t warp = (size_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const size_t t = warp * 32 + lane;
    // carry into this warp's chunk (all 32 tiles of a warp share one chunk)
    uint32_t cg, cp;
    chunk_prefix(chunk_agg, (warp * 32) / kChunk, lane, cg, cp);
    const uint32_t xc = cg | (cp & x);
    uint32_t cin = 0, pt = 0;
    size_t len = 0;
    if (t < n) {
        const uint32_t st = state[t];
        cin = ((st & kBitGex) ? 1u : 0u) | (((st & kBitPex) ? 1u : 0u) & xc);
        pt = st & 0xffffu;
        const size_t L0 = t * size_t(kTile);
        len = (m - L0) < size_t(kTile) ? (m - L0) : size_t(kTile);
        if (cin && pt < len) {
            uint64_t* q = out + L0 + pt;
            *q = apply_carry<SUB>(*q, 1u);
        }
    }
    // Deferred prefixes: the whole warp writes each one, coalesced.
    uint32_t need = __ballot_sync(0xffffffffu, t < n && pt > 0);
    while (need) {
        const int src = __ffs(need) - 1;
        need &= need - 1;
        const uint32_t c = __shfl_sync(0xffffffffu, cin, src);
        const uint32_t n_pre = __shfl_sync(0xffffffffu, pt, src);
        const size_t L0 = (warp * 32 + size_t(src)) * size_t(kTile);
        const uint64_t v = prop_value<SUB>(c);
        uint64_t* o = out + L0;
        uint32_t i0 = 0;
        if ((reinterpret_cast<uintptr_t>(o) & 31u) == 0) {  // 256-bit stores for the bulk
            const uint64_t vv[4] = {v, v, v, v};
            const uint32_t n4 = n_pre & ~3u;
            for (uint32_t i = 4 * lane; i < n4; i += 128) st_stream<4>(o + i, vv);
            i0 = n4;
        }
        for (uint32_t i = i0 + lane; i < n_pre; i += 32) o[i] = v;
    }
}

}  // namespace

// State scratch: one word per tile, then one word per chunk of kChunk tiles.
size_t state_words(size_t n) { return (n + 63) / 64 * 64; }
size_t num_chunks(size_t n) { return (n + kChunk - 1) / kChunk; }

size_t long_state_bytes(size_t m) {
    const size_t n = num_tiles(m);
    return (state_words(n) + num_chunks(n) + 64) * sizeof(uint32_t);
}

cudaError_t launch_long_local(bool sub, uint64_t* out, const uint64_t* a, const uint64_t* b,
                              size_t m, void* state, uint32_t* agg, cudaStream_t stream) {
    const size_t n = num_tiles(m);
    uint32_t* st = static_cast<uint32_t*>(state);
    if (n == 0) {
        // Empty shard: identity aggregate {G = 0, P = 1}.
        static const uint32_t ident[2] = {0u, 1u};
        return cudaMemcpyAsync(agg, ident, sizeof(ident), cudaMemcpyHostToDevice, stream);
    }
    const bool vec = (reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(a) |
                      reinterpret_cast<uintptr_t>(b)) % 32 == 0;
    if (n > 0xffffffffull) return cudaErrorInvalidValue;
    const unsigned grid = unsigned(n);
    if (sub) {
        if (vec) k_long_local<true, true><<<grid, kThreads, 0, stream>>>(out, a, b, m, st, 0);
        else k_long_local<true, false><<<grid, kThreads, 0, stream>>>(out, a, b, m, st, 0);
    } else {
        if (vec) k_long_local<false, true><<<grid, kThreads, 0, stream>>>(out, a, b, m, st, 0);
        else k_long_local<false, false><<<grid, kThreads, 0, stream>>>(out, a, b, m, st, 0);
    }
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    uint32_t* chunk_agg = st + state_words(n);
    const size_t nch = num_chunks(n);
    k_long_scan_chunks<<<unsigned(nch), kChunk, 0, stream>>>(st, n, chunk_agg, 0);
    count_launch();
    k_long_shard_agg<<<1, 32, 0, stream>>>(chunk_agg, nch, agg, 0);
    count_launch();
    return cudaGetLastError();
}

// An empty shard (m = 0) still takes part in the exchange: it is all-propagate with no
// generate, {G, P} = {0, 1} - the identity of the (G, P) composition.
__global__ void k_shard_identity(uint32_t* agg) {
    agg[0] = 0u;
    agg[1] = 1u;
}

// Whole-number carry from the gathered shard aggregates (what k_long_finish writes for a
// non-empty shard): total = G_{w-1} | (P_{w-1} & total_{w-2}) ...
__global__ void k_compose_aggs(const uint32_t* all_aggs, int world, uint32_t* carry_out) {
    uint32_t total = 0;
    for (int q = 0; q < world; ++q) total = all_aggs[2 * q] | (all_aggs[2 * q + 1] & total);
    *carry_out = total;
}

cudaError_t launch_shard_identity(uint32_t* agg, cudaStream_t stream) {
    k_shard_identity<<<1, 1, 0, stream>>>(agg);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_compose_aggs(const uint32_t* all_aggs, int world, uint32_t* carry_out, cudaStream_t stream) {
    k_compose_aggs<<<1, 1, 0, stream>>>(all_aggs, world, carry_out);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_long_finish(bool sub, uint64_t* out, size_t m, void* state,
                               const uint32_t* all_aggs, int rank, int world, uint32_t* carry_out,
                               cudaStream_t stream) {
    const size_t n = num_tiles(m);
    const size_t warps = (n + 31) / 32;
    const size_t blocks = n == 0 ? 1 : (warps * 32 + 255) / 256;
    const uint32_t* st = static_cast<const uint32_t*>(state);
    const uint32_t* chunk_agg = st + state_words(n);
    if (sub)
        k_long_finish<true><<<unsigned(blocks), 256, 0, stream>>>(out, m, st, chunk_agg, n, all_aggs, rank,
                                                                  world, carry_out, 0);
    else
        k_long_finish<false><<<unsigned(blocks), 256, 0, stream>>>(out, m, st, chunk_agg, n, all_aggs, rank,
                                                                   world, carry_out, 0);
    count_launch();
    return cudaGetLastError();
}

// A batch of long numbers (row-major [batch][m]): the three passes once for all of them,
// grid.y = number; each number is its own single "shard" (world 1), its carry its flag.
cudaError_t launch_long_batch(bool sub, uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags,
                              size_t m, size_t batch, cudaStream_t stream) {
    if (batch == 0 || m == 0) return cudaErrorInvalidValue;
    if (batch > 65535) return cudaErrorInvalidConfiguration;
    const size_t n = num_tiles(m);
    const size_t sw = long_state_bytes(m) / sizeof(uint32_t);  // words per number (64-aligned pad inside)
    retain_stream_pool();
    uint32_t* st = nullptr;
    cudaError_t e = cudaMallocAsync(&st, (batch * sw + 2 * batch) * sizeof(uint32_t), stream);
    if (e != cudaSuccess) return e;
    uint32_t* aggs = st + batch * sw;
    const bool vec = (m % 4 == 0) && (reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(a) |
                                      reinterpret_cast<uintptr_t>(b)) % 32 == 0;
    const dim3 g1{unsigned(n), unsigned(batch), 1u};
    if (sub) {
        if (vec) k_long_local<true, true><<<g1, kThreads, 0, stream>>>(out, a, b, m, st, sw);
        else k_long_local<true, false><<<g1, kThreads, 0, stream>>>(out, a, b, m, st, sw);
    } else {
        if (vec) k_long_local<false, true><<<g1, kThreads, 0, stream>>>(out, a, b, m, st, sw);
        else k_long_local<false, false><<<g1, kThreads, 0, stream>>>(out, a, b, m, st, sw);
    }
    const size_t nch = num_chunks(n);
    uint32_t* chunk_agg = st + state_words(n);
    k_long_scan_chunks<<<dim3(unsigned(nch), unsigned(batch)), kChunk, 0, stream>>>(st, n, chunk_agg, sw);
    k_long_shard_agg<<<dim3(1, unsigned(batch)), 32, 0, stream>>>(chunk_agg, nch, aggs, sw);
    const size_t warps = (n + 31) / 32;
    const dim3 g3{unsigned((warps * 32 + 255) / 256), unsigned(batch), 1u};
    if (sub)
        k_long_finish<true><<<g3, 256, 0, stream>>>(out, m, st, chunk_agg, n, aggs, 0, 1, flags, sw);
    else
        k_long_finish<false><<<g3, 256, 0, stream>>>(out, m, st, chunk_agg, n, aggs, 0, 1, flags, sw);
    count_launch(4);
    e = cudaGetLastError();
    cudaFreeAsync(st, stream);
    return e;
}

}  // namespace dotg
