// addsub_batch.cu - batched multi-limb add/sub of independent pairs on sm_100a.
//
// Replaces the reference's per-pair span call dot_add_words / dot_sub_words
// (include/dot/addsub.hpp:98-103 -> src/addsub.cpp:136-170), whose only loop-carried
// dependency is the carry between w-limb chunks (addsub.cpp:152-157). Here the four DoT
// phases (addsub.hpp:1-11) run across lanes instead of across chunks:
//   1. lane-independent limb sums      (addsub.cpp:35-37)   -> lane_op
//   2. generate/propagate extraction    (addsub.cpp:39-46)   -> g, p per limb, folded per
//                                                              super-lane of V limbs
//   3. carry resolve: one warp ballot of G and P, then ONE integer mask addition
//      C = ((G<<1) + P) ^ P per number (the reference's Phase-4 formula,
//      addsub.cpp:61-79, applied to every lane at once instead of only on cascades)
//   4. carry application inside the super-lane (p-chains of <= V limbs).
// There is no serial chunk chain and no data-dependent branch: the "rare" cascade of the
// reference costs the same as the common case here.
//
// Row-major layout [batch][m] (the reference's Limbs back to back): a team of T lanes
// owns one number; lane t of the team holds R vectors of V limbs at limb offsets
// r*V*T + t*V, so each vector load of a warp covers 32/T whole numbers contiguously
// (coalesced 256-bit LDG/STG). Interleaved layout [m][batch] and non-power-of-two m use
// a thread-per-pair strided kernel with the same carry semantics.
#include <cuda_runtime.h>

#include <cstdint>

#include "device.cuh"
#include "internal.h"

namespace dotg {

template <int M, int V>
struct TeamCfg {
    static constexpr int SL = M / V;             // super-lanes per number
    static constexpr int T = SL < 32 ? SL : 32;  // lanes per number
    static constexpr int R = SL / T;             // vectors per lane per number
    static constexpr int NPW = 32 / T;           // numbers per warp row-group
    static constexpr int W = (SL + 63) / 64;     // 64-bit mask words per number
    static_assert(M % V == 0 && SL % T == 0, "M must be a power of two multiple of V");
};

template <bool SUB, int M, int V, int U>
__global__ void __launch_bounds__(256) k_addsub_team(uint64_t* out, const uint64_t* a,
                                                     const uint64_t* b, uint32_t* flags,
                                                     size_t batch) {
    using C = TeamCfg<M, V>;
    const unsigned lane = threadIdx.x & 31u;
    const unsigned team = lane / C::T;
    const unsigned t = lane % C::T;
    const size_t warp = (size_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const size_t base_num = warp * size_t(C::NPW * U);

    uint64_t s[U][C::R][V];
    uint64_t bv[U][C::R][V];
    // Issue every load of the warp's U row-groups before any arithmetic (MLP).
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const size_t num = base_num + size_t(u * C::NPW) + team;
        const bool ok = num < batch;
#pragma unroll
        for (int r = 0; r < C::R; ++r) {
            const size_t off = num * M + size_t(r * V * C::T + t * V);
            if (ok) {
                ld_stream<V>(a + off, s[u][r]);
                ld_stream<V>(b + off, bv[u][r]);
            } else {
#pragma unroll
                for (int k = 0; k < V; ++k) s[u][r][k] = bv[u][r][k] = 0;
            }
        }
    }

#pragma unroll
    for (int u = 0; u < U; ++u) {
        const size_t num = base_num + size_t(u * C::NPW) + team;
        const bool ok = num < batch;
        uint32_t g[C::R][V], p[C::R][V];
        uint64_t Gm[C::W], Pm[C::W];
#pragma unroll
        for (int w = 0; w < C::W; ++w) Gm[w] = Pm[w] = 0;
#pragma unroll
        for (int r = 0; r < C::R; ++r) {
            // Phase 1 + 2.
#pragma unroll
            for (int k = 0; k < V; ++k) s[u][r][k] = lane_op<SUB>(s[u][r][k], bv[u][r][k], g[r][k], p[r][k]);
            uint32_t G, P;
            fold_gp<V>(g[r], p[r], G, P);
            const uint32_t gw = __ballot_sync(0xffffffffu, G);
            const uint32_t pw = __ballot_sync(0xffffffffu, P);
            if constexpr (C::T == 32) {
                Gm[r / 2] |= uint64_t(gw) << (32 * (r % 2));
                Pm[r / 2] |= uint64_t(pw) << (32 * (r % 2));
            } else {
                const uint32_t tm = (1u << C::T) - 1u;
                Gm[0] = (gw >> (team * C::T)) & tm;
                Pm[0] = (pw >> (team * C::T)) & tm;
            }
        }
        // Phase 3: mask-add lookahead over the number's SL super-lanes (cin = 0).
        uint64_t Cm[C::W];
        uint32_t k = 0;
#pragma unroll
        for (int w = 0; w < C::W; ++w) {
            const uint32_t gin = w == 0 ? 0u : uint32_t(Gm[w - 1] >> 63);
            Cm[w] = lookahead64(Gm[w], Pm[w], k, gin, k);
        }
        uint32_t flag;
        if constexpr (C::SL % 64 == 0) flag = uint32_t(Gm[C::W - 1] >> 63) | k;
        else flag = uint32_t(Cm[C::W - 1] >> (C::SL % 64)) & 1u;

        // Phase 4: apply carries inside each super-lane, store.
#pragma unroll
        for (int r = 0; r < C::R; ++r) {
            const unsigned j = unsigned(r * C::T) + t;
            const uint32_t c = uint32_t(Cm[j / 64] >> (j % 64)) & 1u;
            apply_superlane<SUB, V>(s[u][r], g[r], p[r], c);
            if (ok) st_stream<V>(out + num * M + size_t(r * V * C::T + t * V), s[u][r]);
        }
        if (flags != nullptr && ok && t == 0) flags[num] = flag;
    }
}

// Thread per pair, any m and any strides: pair p, limb i at p*sp + i*si. Interleaved
// layout (sp = 1, si = batch) is coalesced; row-major (sp = m, si = 1) is the fallback
// for m that is not a power of two or misaligned pointers. Same carry semantics as the
// limb-serial oracle (src/oracle.cpp:16-48).
template <bool SUB>
__global__ void __launch_bounds__(256) k_addsub_strided(uint64_t* out, const uint64_t* a,
                                                        const uint64_t* b, uint32_t* flags,
                                                        size_t m, size_t batch, size_t sp,
                                                        size_t si) {
    const size_t pidx = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (pidx >= batch) return;
    const uint64_t* pa = a + pidx * sp;
    const uint64_t* pb = b + pidx * sp;
    uint64_t* po = out + pidx * sp;
    uint32_t c = 0;
    size_t i = 0;
    constexpr int UN = 8;
    for (; i + UN <= m; i += UN) {
        uint64_t x[UN], y[UN];
#pragma unroll
        for (int k = 0; k < UN; ++k) {
            x[k] = pa[(i + k) * si];
            y[k] = pb[(i + k) * si];
        }
#pragma unroll
        for (int k = 0; k < UN; ++k) {
            uint32_t g, p;
            const uint64_t sv = lane_op<SUB>(x[k], y[k], g, p);
            x[k] = apply_carry<SUB>(sv, c);
            c = g | (p & c);
        }
#pragma unroll
        for (int k = 0; k < UN; ++k) po[(i + k) * si] = x[k];
    }
    for (; i < m; ++i) {
        uint32_t g, p;
        const uint64_t sv = lane_op<SUB>(pa[i * si], pb[i * si], g, p);
        po[i * si] = apply_carry<SUB>(sv, c);
        c = g | (p & c);
    }
    if (flags != nullptr) flags[pidx] = c;
}

namespace {

template <bool SUB, int M, int V, int U>
cudaError_t run_team(uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags,
                     size_t batch, cudaStream_t st) {
    using C = TeamCfg<M, V>;
    const size_t per_warp = size_t(C::NPW) * U;
    const size_t warps = (batch + per_warp - 1) / per_warp;
    const size_t blocks = (warps * 32 + 255) / 256;
    k_addsub_team<SUB, M, V, U><<<unsigned(blocks), 256, 0, st>>>(out, a, b, flags, batch);
    count_launch();
    return cudaGetLastError();
}

template <bool SUB>
cudaError_t run_strided(uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags,
                        size_t m, size_t batch, size_t sp, size_t si, cudaStream_t st) {
    const size_t blocks = (batch + 255) / 256;
    k_addsub_strided<SUB><<<unsigned(blocks), 256, 0, st>>>(out, a, b, flags, m, batch, sp, si);
    count_launch();
    return cudaGetLastError();
}

bool aligned(const void* p, size_t bytes) { return (reinterpret_cast<uintptr_t>(p) % bytes) == 0; }

template <bool SUB>
cudaError_t dispatch(uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags, size_t m,
                     size_t batch, int layout, cudaStream_t st) {
    if (layout == 1) return run_strided<SUB>(out, a, b, flags, m, batch, 1, batch, st);
    const bool a32 = aligned(out, 32) && aligned(a, 32) && aligned(b, 32);
    const bool a16 = aligned(out, 16) && aligned(a, 16) && aligned(b, 16);
    switch (m) {
        case 1: return run_team<SUB, 1, 1, 2>(out, a, b, flags, batch, st);
        case 2:
            if (a16) return run_team<SUB, 2, 2, 2>(out, a, b, flags, batch, st);
            break;
        case 4:
            if (a32) return run_team<SUB, 4, 4, 2>(out, a, b, flags, batch, st);
            break;
        case 8:
            if (a32) return run_team<SUB, 8, 4, 2>(out, a, b, flags, batch, st);
            break;
        case 16:
            if (a32) return run_team<SUB, 16, 4, 2>(out, a, b, flags, batch, st);
            break;
        case 32:
            if (a32) return run_team<SUB, 32, 4, 2>(out, a, b, flags, batch, st);
            break;
        case 64:
            if (a32) return run_team<SUB, 64, 4, 2>(out, a, b, flags, batch, st);
            break;
        case 128:
            if (a32) return run_team<SUB, 128, 4, 2>(out, a, b, flags, batch, st);
            break;
        case 256:
            if (a32) return run_team<SUB, 256, 4, 1>(out, a, b, flags, batch, st);
            break;
        case 512:
            if (a32) return run_team<SUB, 512, 4, 1>(out, a, b, flags, batch, st);
            break;
        default:
            break;
    }
    return run_strided<SUB>(out, a, b, flags, m, batch, m, 1, st);
}

}  // namespace

cudaError_t launch_addsub_batch(bool sub, uint64_t* out, const uint64_t* a, const uint64_t* b,
                                uint32_t* flags, size_t m, size_t batch, int layout,
                                cudaStream_t stream) {
    if (batch == 0) return cudaSuccess;
    if (m == 0) {
        if (flags == nullptr) return cudaSuccess;
        return cudaMemsetAsync(flags, 0, batch * sizeof(uint32_t), stream);
    }
    return sub ? dispatch<true>(out, a, b, flags, m, batch, layout, stream)
               : dispatch<false>(out, a, b, flags, m, batch, layout, stream);
}

}  // namespace dotg
