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
// r*V*T + t*V, so each 256-bit vector load of a warp covers 32/T whole numbers
// contiguously. Every warp task is 256 limbs per operand whatever m is, so tasks of
// different sizes cost the same.
//
// Launch shape: ONE persistent kernel per call, grid = SMs x resident CTAs, warps
// striding over the concatenated task lists of up to kMaxGroup independent problems
// (dotg_addsub_grouped). A whole multi-size sweep is one launch: no inter-kernel gaps,
// no wave-quantisation tail per size.
//
// Interleaved layout [m][batch] and non-power-of-two m use a thread-per-pair strided
// kernel with the same carry semantics.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cmath>
#include <cstdlib>
#include <type_traits>

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

// (V, U) per power-of-two m: 256 limbs per operand per warp task for every m >= 4.
__host__ __device__ constexpr int team_v(uint32_t m) { return m >= 4 ? 4 : int(m); }
__host__ __device__ constexpr int team_u(uint32_t m) { return m >= 256 ? 1 : 2; }
__host__ __device__ constexpr uint64_t numbers_per_task(uint32_t m) {
    // NPW * U with T = min(m / V, 32)
    return uint64_t(32 / ((m / team_v(m)) < 32 ? (m / team_v(m)) : 32)) * uint64_t(team_u(m));
}

// Phase ticks of the timed instantiation (the GPU counterpart of the reference's
// AddSubStats::collect_ticks laps, PhaseTimer in kernels.hpp:20-37): SM clock cycles per
// warp, lane 0 accumulating. Buckets in AddSubStats order: load, add, carry_gen,
// carry_add, store, overflow. "overflow" (the reference's Phase-4 cascade) stays 0: the
// mask addition of carry_gen resolves cascades with the same instructions as the common
// case. A lap reads %clock64 only after a value depending on the previous phase's
// results, so outstanding loads are charged to the phase that waits for them.
enum TickBucket { kTickLoad = 0, kTickAdd, kTickCarryGen, kTickCarryAdd, kTickStore, kTickOverflow, kTicks };
template <bool TIMED>
struct WarpTimer {
    uint64_t t0 = 0;
    uint64_t acc[kTicks] = {};
    __device__ __forceinline__ void start() {
        if constexpr (TIMED) asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0)::"memory");
    }
    // dep: any value produced by the phase (forces its completion before the clock read)
    __device__ __forceinline__ void lap(int bucket, uint64_t dep) {
        if constexpr (TIMED) {
            uint64_t t1;
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1) : "l"(dep) : "memory");
            acc[bucket] += t1 - t0;
            t0 = t1;
        }
    }
};

template <bool SUB, int M, int V, int U, bool TIMED = false>
__device__ __forceinline__ void team_task(const AddSubProblem& P, uint64_t task, WarpTimer<TIMED>& tm) {
    using C = TeamCfg<M, V>;
    const unsigned lane = threadIdx.x & 31u;
    const unsigned team = lane / C::T;
    const unsigned t = lane % C::T;
    const uint64_t base_num = task * uint64_t(C::NPW * U);
    const uint64_t batch = P.batch;
    const uint64_t* __restrict__ a = P.a;
    const uint64_t* __restrict__ b = P.b;

    uint64_t s[U][C::R][V];
    uint64_t bv[U][C::R][V];
    tm.start();
    // Issue every load of the task before any arithmetic (MLP).
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const uint64_t num = base_num + uint64_t(u * C::NPW) + team;
        const bool ok = num < batch;
#pragma unroll
        for (int r = 0; r < C::R; ++r) {
            const uint64_t off = num * M + uint64_t(r * V * C::T + t * V);
            if (ok) {
                ld_stream<V>(a + off, s[u][r]);
                ld_stream<V>(b + off, bv[u][r]);
            } else {
#pragma unroll
                for (int k = 0; k < V; ++k) s[u][r][k] = bv[u][r][k] = 0;
            }
        }
    }

    if constexpr (TIMED) {
        uint64_t dep = 0;
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int r = 0; r < C::R; ++r)
#pragma unroll
                for (int k = 0; k < V; ++k) dep ^= s[u][r][k] ^ bv[u][r][k];
        tm.lap(kTickLoad, dep);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const uint64_t num = base_num + uint64_t(u * C::NPW) + team;
        const bool ok = num < batch;
        uint32_t g[C::R][V], p[C::R][V];
        uint64_t Gm[C::W], Pm[C::W];
#pragma unroll
        for (int w = 0; w < C::W; ++w) Gm[w] = Pm[w] = 0;
#pragma unroll
        if constexpr (TIMED) {  // phase 1 (lane sums) timed on its own, as in chunk_generic
#pragma unroll
            for (int r = 0; r < C::R; ++r)
#pragma unroll
                for (int k = 0; k < V; ++k) s[u][r][k] = lane_op<SUB>(s[u][r][k], bv[u][r][k], g[r][k], p[r][k]);
            uint64_t dep = 0;
#pragma unroll
            for (int r = 0; r < C::R; ++r)
#pragma unroll
                for (int k = 0; k < V; ++k) dep += s[u][r][k] + g[r][k] + p[r][k];
            tm.lap(kTickAdd, dep);
        }
#pragma unroll
        for (int r = 0; r < C::R; ++r) {
            // Phase 1 + 2.
            if constexpr (!TIMED) {
#pragma unroll
                for (int k = 0; k < V; ++k) s[u][r][k] = lane_op<SUB>(s[u][r][k], bv[u][r][k], g[r][k], p[r][k]);
            }
            uint32_t G, P2;
            fold_gp<V>(g[r], p[r], G, P2);
            const uint32_t gw = __ballot_sync(0xffffffffu, G);
            const uint32_t pw = __ballot_sync(0xffffffffu, P2);
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
        tm.lap(kTickCarryGen, Cm[0] + flag);

        // Phase 4: apply carries inside each super-lane, store.
        if constexpr (TIMED) {
            uint64_t dep = 0;
#pragma unroll
            for (int r = 0; r < C::R; ++r) {
                const unsigned j = unsigned(r * C::T) + t;
                const uint32_t c = uint32_t(Cm[j / 64] >> (j % 64)) & 1u;
                apply_superlane<SUB, V>(s[u][r], g[r], p[r], c);
#pragma unroll
                for (int k = 0; k < V; ++k) dep += s[u][r][k];
            }
            tm.lap(kTickCarryAdd, dep);
        }
#pragma unroll
        for (int r = 0; r < C::R; ++r) {
            if constexpr (!TIMED) {
                const unsigned j = unsigned(r * C::T) + t;
                const uint32_t c = uint32_t(Cm[j / 64] >> (j % 64)) & 1u;
                apply_superlane<SUB, V>(s[u][r], g[r], p[r], c);
            }
            if (ok) st_stream<V>(P.out + num * M + uint64_t(r * V * C::T + t * V), s[u][r]);
        }
        if (P.flags != nullptr && ok && t == 0) P.flags[num] = flag;
        tm.lap(kTickStore, 0);
    }
}

template <bool SUB, bool TIMED = false>
__device__ __forceinline__ void dispatch_small(const AddSubProblem& P, uint64_t task, WarpTimer<TIMED>& tm) {
    switch (P.m) {
        case 1: team_task<SUB, 1, 1, 2, TIMED>(P, task, tm); break;
        case 2: team_task<SUB, 2, 2, 2, TIMED>(P, task, tm); break;
        case 4: team_task<SUB, 4, 4, 2, TIMED>(P, task, tm); break;
        case 8: team_task<SUB, 8, 4, 2, TIMED>(P, task, tm); break;
        case 16: team_task<SUB, 16, 4, 2, TIMED>(P, task, tm); break;
        case 32: team_task<SUB, 32, 4, 2, TIMED>(P, task, tm); break;
        case 64: team_task<SUB, 64, 4, 2, TIMED>(P, task, tm); break;
        case 128: team_task<SUB, 128, 4, 2, TIMED>(P, task, tm); break;
        case 256: team_task<SUB, 256, 4, 1, TIMED>(P, task, tm); break;
        default: break;
    }
}

// BIG = false: m in {1, ..., 256}; BIG = true: m == 512 (kept apart so its register
// footprint does not cap the occupancy of the common sizes).
template <bool BIG>
__global__ void __launch_bounds__(256) k_addsub_grouped(const __grid_constant__ AddSubGroup grp) {
    const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    WarpTimer<false> tm;
    int pi = 0;
    for (uint64_t t = warp; t < grp.total_tasks; t += nw) {
        while (pi + 1 < grp.n && grp.p[pi + 1].task_begin <= t) ++pi;
        const AddSubProblem& P = grp.p[pi];
        const uint64_t task = t - P.task_begin;
        if constexpr (BIG) {
            if (P.sub) team_task<true, 512, 4, 1>(P, task, tm);
            else team_task<false, 512, 4, 1>(P, task, tm);
        } else {
            if (P.sub) dispatch_small<true>(P, task, tm);
            else dispatch_small<false>(P, task, tm);
        }
    }
}

// The same persistent task loop with the phase laps compiled in (one problem, m a power of
// two <= 256, row-major): results identical to k_addsub_grouped; ticks = device uint64[6]
// accumulated (AddSubStats bucket order), summed over warps.
__global__ void __launch_bounds__(256) k_addsub_timed(const AddSubProblem P, uint64_t ntasks, uint64_t* ticks) {
    const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    WarpTimer<true> tm;
    for (uint64_t t = warp; t < ntasks; t += nw) {
        if (P.sub) dispatch_small<true, true>(P, t, tm);
        else dispatch_small<false, true>(P, t, tm);
    }
    if ((threadIdx.x & 31u) == 0)
        for (int i = 0; i < kTicks; ++i)
            if (tm.acc[i]) atomicAdd(reinterpret_cast<unsigned long long*>(ticks + i), (unsigned long long)tm.acc[i]);
}

cudaError_t launch_addsub_timed(bool sub, uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags,
                                size_t m, size_t batch, uint64_t* ticks, cudaStream_t st) {
    if (m == 0 || m > 256 || (m & (m - 1)) != 0) return cudaErrorNotSupported;
    AddSubProblem P{};
    P.out = out;
    P.a = a;
    P.b = b;
    P.flags = flags;
    P.batch = batch;
    P.m = uint32_t(m);
    P.sub = sub ? 1u : 0u;
    const uint64_t ntasks = (batch + numbers_per_task(uint32_t(m)) - 1) / numbers_per_task(uint32_t(m));
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_addsub_timed, 256, 0);
    const uint64_t cap = uint64_t(sms) * uint64_t(per > 0 ? per : 1);
    const uint64_t need = (ntasks + 7) / 8;
    k_addsub_timed<<<unsigned(need < cap ? (need ? need : 1) : cap), 256, 0, st>>>(P, ntasks, ticks);
    count_launch();
    return cudaGetLastError();
}

// Thread per pair, any m and any strides: pair p, limb i at p*sp + i*si. Interleaved
// layout (sp = 1, si = batch) is coalesced; row-major (sp = m, si = 1) is the fallback
// for m that is not a power of two or misaligned pointers. Same carry semantics as the
// limb-serial oracle (src/oracle.cpp:16-48). Rows go UN at a time with all their loads
// in flight - the last, partial group too (predicated), so m < UN and ragged tails keep
// their loads batched (r02: a one-row-at-a-time tail held m = 1 ... 7 at 0.69-0.77 of HBM).
// VP = 2 (interleaved, even batch, 16-byte aligned rows): a thread owns two adjacent
// pairs and moves 16 bytes per row and operand.
#ifndef DOTG_TPP_UN
#define DOTG_TPP_UN 8
#endif
template <bool SUB, int VP>
__global__ void __launch_bounds__(256, VP == 1 ? 6 : 3) k_addsub_strided(uint64_t* out, const uint64_t* a,
                                                        const uint64_t* b, uint32_t* flags,
                                                        size_t m, size_t batch, size_t sp,
                                                        size_t si) {
    constexpr int UN = DOTG_TPP_UN;
    const size_t pidx = (size_t(blockIdx.x) * blockDim.x + threadIdx.x) * VP;
    if (pidx >= batch) return;
    const uint64_t* pa = a + pidx * sp;
    const uint64_t* pb = b + pidx * sp;
    uint64_t* po = out + pidx * sp;
    uint32_t c[VP];
#pragma unroll
    for (int v = 0; v < VP; ++v) c[v] = 0;
    // rows i .. i + n - 1 (n <= N), every load of the group first
    auto chunk = [&](auto NN, size_t i, int n) {
        constexpr int N = decltype(NN)::value;
        uint64_t x[N][VP], y[N][VP];
#pragma unroll
        for (int k = 0; k < N; ++k)
            if (k < n) {
                if constexpr (VP == 2) {
                    const ulonglong2 u = *reinterpret_cast<const ulonglong2*>(pa + (i + k) * si);
                    const ulonglong2 w = *reinterpret_cast<const ulonglong2*>(pb + (i + k) * si);
                    x[k][0] = u.x, x[k][1] = u.y, y[k][0] = w.x, y[k][1] = w.y;
                } else {
                    x[k][0] = pa[(i + k) * si];
                    y[k][0] = pb[(i + k) * si];
                }
            }
#pragma unroll
        for (int k = 0; k < N; ++k)
            if (k < n) {
#pragma unroll
                for (int v = 0; v < VP; ++v) {
                    uint32_t g, p;
                    const uint64_t sv = lane_op<SUB>(x[k][v], y[k][v], g, p);
                    x[k][v] = apply_carry<SUB>(sv, c[v]);
                    c[v] = g | (p & c[v]);
                }
                if constexpr (VP == 2)
                    *reinterpret_cast<ulonglong2*>(po + (i + k) * si) = make_ulonglong2(x[k][0], x[k][1]);
                else
                    po[(i + k) * si] = x[k][0];
            }
    };
    size_t i = 0;
    for (; i + UN <= m; i += UN) chunk(std::integral_constant<int, UN>{}, i, UN);
    for (; i < m; i += 4) chunk(std::integral_constant<int, 4>{}, i, m - i < 4 ? int(m - i) : 4);  // tail, 4 rows at a time
    if (flags != nullptr) {
#pragma unroll
        for (int v = 0; v < VP; ++v) flags[pidx + v] = c[v];
    }
}

// Interleaved numbers of M <= 3 limbs: a thread owns 4 adjacent pairs, every row one
// 32-byte load per operand and one 32-byte store (all M rows in flight), the 4 flags one
// 16-byte store - a carry-chained streaming add. (The per-pair kernel above keeps only
// 2-6 loads of 8 bytes per thread in flight at these sizes: 0.38-0.77 of HBM.)
template <bool SUB, int M>
__global__ void __launch_bounds__(256) k_addsub_il_tiny(uint64_t* __restrict__ out, const uint64_t* __restrict__ a,
                                                        const uint64_t* __restrict__ b, uint32_t* __restrict__ flags,
                                                        size_t batch) {
    const size_t p = (size_t(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
    if (p >= batch) return;
    uint64_t x[M][4], y[M][4];
#pragma unroll
    for (int r = 0; r < M; ++r) {
        ld_stream<4>(a + size_t(r) * batch + p, x[r]);
        ld_stream<4>(b + size_t(r) * batch + p, y[r]);
    }
    uint32_t c[4] = {0, 0, 0, 0};
#pragma unroll
    for (int r = 0; r < M; ++r) {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            uint32_t g, pr;
            const uint64_t sv = lane_op<SUB>(x[r][v], y[r][v], g, pr);
            x[r][v] = apply_carry<SUB>(sv, c[v]);
            c[v] = g | (pr & c[v]);
        }
        st_stream<4>(out + size_t(r) * batch + p, x[r]);
    }
    if (flags != nullptr) *reinterpret_cast<uint4*>(flags + p) = make_uint4(c[0], c[1], c[2], c[3]);
}

// Row-major numbers of 3 <= m <= 7 limbs (not a power of two): a CTA stages its P
// pairs' rows (P * m contiguous limbs per operand, 16-byte loads, UN of them in flight per
// thread) into shared memory, each thread then walks its own pair's limbs with one carry
// (the limb-serial oracle's loop, oracle.cpp:16-48) writing the sums over the staged a,
// and the CTA stores the P * m result limbs contiguously. Loads and stores stay fully
// coalesced whatever m is; the serial walks read shared memory with stride m limbs
// (2-way bank conflicts for odd m, the minimum for 8-byte lanes). Measured (tools/il_graph.py
// rows, B x m = 2^22): m = 3 / 5 / 6 / 7 at 0.77 / 0.87 / 0.84 / 0.89 of HBM against 0.69 /
// 0.67 / 0.67 / 0.71 on k_addsub_rows_any; from m = 9 up the per-thread walks (and, for even
// m, bank conflicts: m = 24 0.36) lose to k_addsub_rows_any, which keeps them.
template <bool SUB>
__global__ void __launch_bounds__(128) k_addsub_rows_staged(uint64_t* __restrict__ out, const uint64_t* __restrict__ a,
                                                            const uint64_t* __restrict__ b, uint32_t* __restrict__ flags,
                                                            uint32_t m, size_t batch, uint32_t P) {
    extern __shared__ __align__(16) uint64_t st[];  // [P * m] a (then the sums) | [P * m] b
    const size_t p0 = size_t(blockIdx.x) * P;
    const uint32_t np = uint32_t(batch - p0 < size_t(P) ? batch - p0 : size_t(P));
    const uint32_t n = np * m;  // limbs per operand in this CTA (even: P is a multiple of 32)
    const ulonglong2* ga = reinterpret_cast<const ulonglong2*>(a + p0 * m);
    const ulonglong2* gb = reinterpret_cast<const ulonglong2*>(b + p0 * m);
    ulonglong2* sa = reinterpret_cast<ulonglong2*>(st);
    ulonglong2* sb = reinterpret_cast<ulonglong2*>(st + size_t(P) * m);
    const uint32_t n2 = n / 2, T = blockDim.x;
    constexpr int UN = 4;
    for (uint32_t e0 = threadIdx.x; e0 < n2; e0 += UN * T) {
        ulonglong2 x[UN], y[UN];
#pragma unroll
        for (int u = 0; u < UN; ++u)
            if (e0 + u * T < n2) x[u] = __ldcs(ga + e0 + u * T), y[u] = __ldcs(gb + e0 + u * T);
#pragma unroll
        for (int u = 0; u < UN; ++u)
            if (e0 + u * T < n2) sa[e0 + u * T] = x[u], sb[e0 + u * T] = y[u];
    }
    if ((n & 1u) && threadIdx.x == 0) st[n - 1] = a[p0 * m + n - 1], st[size_t(P) * m + n - 1] = b[p0 * m + n - 1];
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < np; t += T) {
        uint64_t* ra = st + size_t(t) * m;
        const uint64_t* rb = st + size_t(P) * m + size_t(t) * m;
        uint32_t c = 0;
        uint32_t i = 0;
        for (; i + 4 <= m; i += 4) {
            uint64_t x[4], y[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) x[k] = ra[i + k], y[k] = rb[i + k];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                uint32_t g, pr;
                const uint64_t sv = lane_op<SUB>(x[k], y[k], g, pr);
                ra[i + k] = apply_carry<SUB>(sv, c);
                c = g | (pr & c);
            }
        }
        for (; i < m; ++i) {
            uint32_t g, pr;
            const uint64_t sv = lane_op<SUB>(ra[i], rb[i], g, pr);
            ra[i] = apply_carry<SUB>(sv, c);
            c = g | (pr & c);
        }
        if (flags != nullptr) flags[p0 + t] = c;
    }
    __syncthreads();
    ulonglong2* go = reinterpret_cast<ulonglong2*>(out + p0 * m);
    for (uint32_t e = threadIdx.x; e < n2; e += T) __stcs(go + e, sa[e]);
    if ((n & 1u) && threadIdx.x == 0) out[p0 * m + n - 1] = st[n - 1];
}

// Row-pitched thread per pair: operand rows at their own pitches (views of wider arrays).
template <bool SUB>
__global__ void __launch_bounds__(256) k_addsub_pitched(uint64_t* out, size_t ldo, const uint64_t* a, size_t lda,
                                                        const uint64_t* b, size_t ldb, uint32_t* flags, size_t m,
                                                        size_t batch) {
    const size_t pidx = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (pidx >= batch) return;
    const uint64_t* pa = a + pidx * lda;
    const uint64_t* pb = b + pidx * ldb;
    uint64_t* po = out + pidx * ldo;
    uint32_t c = 0;
    for (size_t i = 0; i < m; ++i) {
        uint32_t g, p;
        const uint64_t sv = lane_op<SUB>(pa[i], pb[i], g, p);
        po[i] = apply_carry<SUB>(sv, c);
        c = g | (p & c);
    }
    if (flags != nullptr) flags[pidx] = c;
}

// Interleaved layout, one launch, nothing held across the barrier: a CTA of W warps owns
// a strip of 32 (or 64: two per lane) pairs; warp w owns limb rows [w*L, (w+1)*L), L = m / W.
//   phase 1: stream the warp's rows in chunks of 8 (16 loads in flight), fold every
//            chunk's generate / propagate bits into the segment's (G, P) - nothing stored,
//            no operand kept in registers;
//   fold:    (G, P) per pair as two ballot masks per warp, ONE barrier, each warp folds
//            the lower segments bit-parallel over its 32 pairs;
//   phase 2: stream the rows again (the strip was just read: L2 hits), add with the known
//            carry-in, store.
// DRAM sees the operands once; registers stay small, so 8-warp CTAs fit 8 per SM and
// the whole B x m = 2^22 batch is resident in ONE wave (the register-holding kernel above
// needs 1.73 waves at m = 256).
// W warps (segments) per CTA, chosen per call so that ceil(batch / 32) CTAs at <= 64
// registers (1024 threads per SM) fit in one wave: W <= 148 * 1024 / batch.
#ifndef DOTG_IL2_OCC
#define DOTG_IL2_OCC 1024  // resident threads per SM the register budget is sized for
#endif
template <bool SUB, int kIL2W, int PPL>
__global__ void __launch_bounds__(kIL2W * 32, DOTG_IL2_OCC / 32 / kIL2W) k_addsub_il2(uint64_t* __restrict__ out, const uint64_t* __restrict__ a,
                                                           const uint64_t* __restrict__ b, uint32_t* flags, size_t m,
                                                           size_t batch) {
    // PPL pairs per lane (2: one 16-byte load per limb row covers two adjacent pairs)
    __shared__ uint32_t sG[kIL2W][PPL], sP[kIL2W][PPL];
    const int w = int(threadIdx.x >> 5), lane = int(threadIdx.x & 31u);
    const size_t p = (size_t(blockIdx.x) * 32 + size_t(lane)) * PPL;
    const bool ok = p < batch;  // PPL = 2: batch is even, a lane has both pairs or none
    const size_t L = (m + kIL2W - 1) / kIL2W;  // rows per warp
    const size_t r0 = size_t(w) * L;
    const size_t r1 = r0 + L < m ? r0 + L : m;
#ifndef DOTG_IL2_CH
#define DOTG_IL2_CH 4
#endif
    constexpr int CH = DOTG_IL2_CH;
    auto load = [&](const uint64_t* base, size_t row, uint64_t (&v)[PPL], bool stream) {
        if constexpr (PPL == 2) {
            const ulonglong2* q = reinterpret_cast<const ulonglong2*>(base + row * batch + p);
            const ulonglong2 t = stream ? __ldcs(q) : __ldcg(q);
            v[0] = t.x;
            v[1] = t.y;
        } else {
            v[0] = stream ? __ldcs(base + row * batch + p) : __ldcg(base + row * batch + p);
        }
    };
    // phase 1: segment (G, P) with carry-in 0, chunk by chunk
    uint32_t G[PPL], P[PPL];
#pragma unroll
    for (int q = 0; q < PPL; ++q) G[q] = 0, P[q] = 1;
    for (size_t c0 = r0; c0 < r1; c0 += CH) {
        uint64_t x[CH][PPL], y[CH][PPL];
#pragma unroll
        for (int k = 0; k < CH; ++k) {
#pragma unroll
            for (int q = 0; q < PPL; ++q) x[k][q] = y[k][q] = 0;
            if (ok && c0 + k < r1) {
                load(a, c0 + k, x[k], false);
                load(b, c0 + k, y[k], false);
            }
        }
#pragma unroll
        for (int k = 0; k < CH; ++k)
            if (c0 + k < r1)
#pragma unroll
                for (int q = 0; q < PPL; ++q) {
                    uint32_t g, pr;
                    lane_op<SUB>(x[k][q], y[k][q], g, pr);
                    G[q] = g | (pr & G[q]);
                    P[q] &= pr;
                }
    }
#pragma unroll
    for (int q = 0; q < PPL; ++q) {
        const uint32_t Gm = __ballot_sync(0xffffffffu, ok && r0 < r1 ? G[q] : 0u);
        const uint32_t Pm = __ballot_sync(0xffffffffu, !ok || r0 >= r1 || P[q]);
        if (lane == 0) {
            sG[w][q] = Gm;
            sP[w][q] = Pm;
        }
    }
    __syncthreads();
    uint32_t c[PPL];
#pragma unroll
    for (int q = 0; q < PPL; ++q) {
        uint32_t cm = 0;  // carries into segment w, one bit per lane
#pragma unroll
        for (int j = 0; j < kIL2W; ++j)
            if (j < w) cm = sG[j][q] | (sP[j][q] & cm);
        c[q] = (cm >> lane) & 1u;
    }
    // phase 2: the same rows again, with the carry
    for (size_t c0 = r0; c0 < r1; c0 += CH) {
        uint64_t x[CH][PPL], y[CH][PPL];
#pragma unroll
        for (int k = 0; k < CH; ++k) {
#pragma unroll
            for (int q = 0; q < PPL; ++q) x[k][q] = y[k][q] = 0;
            if (ok && c0 + k < r1) {
                load(a, c0 + k, x[k], true);
                load(b, c0 + k, y[k], true);
            }
        }
#pragma unroll
        for (int k = 0; k < CH; ++k)
            if (ok && c0 + k < r1) {
                uint64_t r[PPL];
#pragma unroll
                for (int q = 0; q < PPL; ++q) {
                    uint32_t g, pr;
                    const uint64_t v = lane_op<SUB>(x[k][q], y[k][q], g, pr);
                    r[q] = apply_carry<SUB>(v, c[q]);
                    c[q] = g | (pr & c[q]);
                }
                if constexpr (PPL == 2)
                    __stcs(reinterpret_cast<ulonglong2*>(out + (c0 + k) * batch + p), make_ulonglong2(r[0], r[1]));
                else
                    __stcs(out + (c0 + k) * batch + p, r[0]);
            }
    }
    if (ok && flags != nullptr && r1 == m && r0 < r1)
#pragma unroll
        for (int q = 0; q < PPL; ++q) flags[p + q] = c[q];
}

template <bool SUB>
cudaError_t run_interleaved_il2(uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags, size_t m,
                                size_t batch, cudaStream_t st) {
    static thread_local struct { int dev = -1, sms = 148; } di;
    int dev = 0;
    cudaGetDevice(&dev);
    if (di.dev != dev) {
        cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, dev);
        di.dev = dev;
    }
    static const int ppl_knob = [] {
        const char* e = std::getenv("DOTG_IL2_PPL");  // A/B knob: pairs per lane (1 or 2)
        return e ? std::atoi(e) : 2;
    }();
    // two pairs per lane (16-byte row loads) while that still leaves a strip per SM
    // (tools/il2_ab.sh: m = 16 ... 256 +1-9%, m = 1024 at B = 4096 -27% with half the CTAs)
    const bool two = ppl_knob == 2 && batch % 2 == 0 && (batch + 63) / 64 >= size_t(di.sms) &&
                     ((reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(a) |
                       reinterpret_cast<uintptr_t>(b)) & 15u) == 0;
    const size_t ctas = (batch + (two ? 63 : 31)) / (two ? 64 : 32);
    static const int wdiv = [] {
        const char* e = std::getenv("DOTG_IL2_WDIV");  // A/B knob: fewer, longer segments
        return e ? std::atoi(e) : 1;
    }();
    int W = 32;
    while (W > 2 && (size_t(W) * ctas > size_t(di.sms) * (DOTG_IL2_OCC / 32) || size_t(W) * 8 > m)) W /= 2;
    for (int d = wdiv; d > 1 && W > 2; d /= 2) W /= 2;
    const unsigned grid = unsigned(ctas);
#define DOTG_IL2_LAUNCH(WW)                                                                                   \
    (two ? (k_addsub_il2<SUB, WW, 2><<<grid, WW * 32, 0, st>>>(out, a, b, flags, m, batch), 0)              \
         : (k_addsub_il2<SUB, WW, 1><<<grid, WW * 32, 0, st>>>(out, a, b, flags, m, batch), 0))
    switch (W) {
        case 32: DOTG_IL2_LAUNCH(32); break;
        case 16: DOTG_IL2_LAUNCH(16); break;
        case 8: DOTG_IL2_LAUNCH(8); break;
        case 4: DOTG_IL2_LAUNCH(4); break;
        default: DOTG_IL2_LAUNCH(2); break;
    }
#undef DOTG_IL2_LAUNCH
    count_launch();
    return cudaGetLastError();
}

// Interleaved layout, one streaming pass with an in-CTA fix-up (nothing re-read, nothing
// held): a CTA of W warps owns a strip of 32 * PPL pairs, warp w the limb rows
// [w*L, (w+1)*L). Each warp streams its rows UN at a time (2 * UN * PPL loads in flight
// per lane, like the thread-per-pair kernel) and stores them resolved with carry-in 0 -
// except its first row, which it keeps in a register - while recording, per pair, the
// first row whose provisional limb is not the propagating value (~0 for add, 0 for sub)
// and that limb. After ONE barrier (the warps' (G, P) as ballot masks, folded bit-parallel
// as in k_addsub_il2), a carry-in of 1 changes exactly the rows up to that first
// non-propagating one: rows before it become the opposite propagating value (stored
// without reading), that row becomes limb + 1 (- 1 for sub) from the register. With
// random limbs that is the held first row alone. (G, P) of a segment: G = its provisional
// carry out, P = every provisional limb propagating - exclusive, since all-~0 limbs with a
// carry out would exceed a + b.
template <bool SUB, int UN, int PPL, bool DB>
__global__ void __launch_bounds__(512) k_addsub_ilf(uint64_t* __restrict__ out, const uint64_t* __restrict__ a,
                                                    const uint64_t* __restrict__ b, uint32_t* flags, size_t m,
                                                    size_t batch, uint32_t L, uint32_t G) {
    // G lanes per segment (32, 16 or 8): a warp holds 32 / G segments of the strip's G * PPL
    // pairs (narrower strips: more CTAs when the batch is small)
    __shared__ uint32_t sG[64][PPL], sP[64][PPL];
    const int w = int(threadIdx.x >> 5), lane = int(threadIdx.x & 31u);
    const uint32_t spw = 32u / G, ls = uint32_t(lane) % G;     // segments per warp, lane in segment
    const uint32_t seg = uint32_t(w) * spw + uint32_t(lane) / G;  // segment index in the CTA
    const size_t p = (size_t(blockIdx.x) * G + ls) * PPL;
    const bool ok = p < batch;  // PPL > 1: batch % PPL == 0, a lane has all its pairs or none
    const size_t r0 = size_t(seg) * L < m ? size_t(seg) * L : m;
    const size_t r1 = r0 + L < m ? r0 + L : m;
    constexpr uint64_t kProp = SUB ? 0ull : ~0ull;
    uint64_t first[PPL], qv[PPL];
    uint32_t c[PPL], allp[PPL], q[PPL];
#pragma unroll
    for (int j = 0; j < PPL; ++j) first[j] = qv[j] = 0, c[j] = 0, allp[j] = 1, q[j] = 0;
    using Chunk = uint64_t[UN][PPL];
    auto ld = [&](Chunk& x, Chunk& y, size_t c0) {
#pragma unroll
        for (int k = 0; k < UN; ++k)
            if (c0 + k < r1) {
                if constexpr (PPL == 4) {  // one 32-byte load per row and operand
                    const uint64_t* pa = a + (c0 + k) * batch + p;
                    const uint64_t* pb = b + (c0 + k) * batch + p;
                    asm("ld.global.L1::no_allocate.L2::evict_first.v4.u64 {%0,%1,%2,%3}, [%4];"
                        : "=l"(x[k][0]), "=l"(x[k][1]), "=l"(x[k][2]), "=l"(x[k][3])
                        : "l"(pa));
                    asm("ld.global.L1::no_allocate.L2::evict_first.v4.u64 {%0,%1,%2,%3}, [%4];"
                        : "=l"(y[k][0]), "=l"(y[k][1]), "=l"(y[k][2]), "=l"(y[k][3])
                        : "l"(pb));
                } else if constexpr (PPL == 2) {
                    const ulonglong2 u = __ldcs(reinterpret_cast<const ulonglong2*>(a + (c0 + k) * batch + p));
                    const ulonglong2 v = __ldcs(reinterpret_cast<const ulonglong2*>(b + (c0 + k) * batch + p));
                    x[k][0] = u.x, x[k][1] = u.y, y[k][0] = v.x, y[k][1] = v.y;
                } else {
                    x[k][0] = __ldcs(a + (c0 + k) * batch + p);
                    y[k][0] = __ldcs(b + (c0 + k) * batch + p);
                }
            }
    };
    auto proc = [&](Chunk& x, Chunk& y, size_t c0) {
#pragma unroll
        for (int k = 0; k < UN; ++k)
            if (c0 + k < r1) {
                const uint32_t rel = uint32_t(c0 + k - r0);
#pragma unroll
                for (int j = 0; j < PPL; ++j) {
                    uint32_t g, pr;
                    const uint64_t v = apply_carry<SUB>(lane_op<SUB>(x[k][j], y[k][j], g, pr), c[j]);
                    c[j] = g | (pr & c[j]);
                    const uint32_t isp = v == kProp;
                    if (allp[j] && !isp) q[j] = rel, qv[j] = v;
                    allp[j] &= isp;
                    x[k][j] = v;
                }
                if (rel == 0) {
#pragma unroll
                    for (int j = 0; j < PPL; ++j) first[j] = x[k][j];
                } else if constexpr (PPL == 4) {
                    st_stream<4>(out + (c0 + k) * batch + p, x[k]);
                } else if constexpr (PPL == 2) {
                    __stcs(reinterpret_cast<ulonglong2*>(out + (c0 + k) * batch + p), make_ulonglong2(x[k][0], x[k][1]));
                } else {
                    __stcs(out + (c0 + k) * batch + p, x[k][0]);
                }
            }
    };
    if (ok && r0 < r1) {
        Chunk x0, y0;
        if constexpr (DB) {
            // two chunks in flight: the next chunk's loads are issued before this one is resolved
            Chunk x1, y1;
            size_t c0 = r0;
            ld(x0, y0, c0);
            while (true) {
                if (c0 + UN < r1) ld(x1, y1, c0 + UN);
                proc(x0, y0, c0);
                c0 += UN;
                if (c0 >= r1) break;
                if (c0 + UN < r1) ld(x0, y0, c0 + UN);
                proc(x1, y1, c0);
                c0 += UN;
                if (c0 >= r1) break;
            }
        } else {
            for (size_t c0 = r0; c0 < r1; c0 += UN) {
                ld(x0, y0, c0);
                proc(x0, y0, c0);
            }
        }
    }
    const bool has = ok && r0 < r1;
    const uint32_t gmask = G == 32 ? 0xffffffffu : (1u << G) - 1u;
#pragma unroll
    for (int j = 0; j < PPL; ++j) {
        const uint32_t Gm = __ballot_sync(0xffffffffu, has && c[j]);
        const uint32_t Pm = __ballot_sync(0xffffffffu, !has || allp[j]);
        if (uint32_t(lane) < spw) {  // lane k stores the warp's k-th segment's masks
            const uint32_t sh = uint32_t(lane) * G;
            sG[uint32_t(w) * spw + uint32_t(lane)][j] = (Gm >> sh) & gmask;
            sP[uint32_t(w) * spw + uint32_t(lane)][j] = (Pm >> sh) & gmask;
        }
    }
    __syncthreads();
    if (!has) return;
#pragma unroll
    for (int j = 0; j < PPL; ++j) {
        uint32_t cm = 0;  // carries into this segment, one bit per pair lane
        for (uint32_t i = 0; i < seg; ++i) cm = sG[i][j] | (sP[i][j] & cm);
        const uint32_t cin = (cm >> ls) & 1u;
        uint64_t* po = out + r0 * batch + p + j;
        if (!cin) {
            po[0] = first[j];
        } else if (!allp[j] && q[j] == 0) {
            po[0] = apply_carry<SUB>(first[j], 1u);
        } else {
            // rows [0, q) were all propagating (held row 0 among them): they flip; row q
            // (if any) takes the carry
            const uint32_t n = allp[j] ? uint32_t(r1 - r0) : q[j];
            for (uint32_t i = 0; i < n; ++i) po[size_t(i) * batch] = prop_value<SUB>(1u);
            if (!allp[j]) po[size_t(n) * batch] = apply_carry<SUB>(qv[j], 1u);
        }
        if (flags != nullptr && r1 == m) flags[p + j] = c[j] | (allp[j] & cin);
    }
}

// Rows per warp and warps per CTA for k_addsub_ilf: enough warps to cover the GPU in ONE
// wave (warps stream their rows; a second wave would start late and end the launch with a
// tail), rows per warp at least one unrolled chunk.
template <bool SUB>
cudaError_t run_interleaved_ilf(uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags, size_t m,
                                size_t batch, cudaStream_t st) {
    static thread_local struct { int dev = -1, sms = 148; } di;
    int dev = 0;
    cudaGetDevice(&dev);
    if (di.dev != dev) {
        cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, dev);
        di.dev = dev;
    }
    static const int ppl_knob = [] {
        const char* e = std::getenv("DOTG_ILF_PPL");  // A/B knob: pairs per lane (1 or 2; 0 = auto)
        return e ? std::atoi(e) : 0;
    }();
    static const int un_knob = [] {
        const char* e = std::getenv("DOTG_ILF_UN");  // A/B knob: rows per chunk (8 or 16, single-buffered)
        return e ? std::atoi(e) : 0;
    }();
    static const int db_knob = [] {
        const char* e = std::getenv("DOTG_ILF_DB");  // A/B knob: 1 = two chunks in flight
        return e ? std::atoi(e) : 1;
    }();
    static const int wdiv = [] {
        const char* e = std::getenv("DOTG_ILF_WDIV");  // A/B knob: fewer, longer segments
        return e ? std::atoi(e) : 1;
    }();
    // variants (chunk rows x pairs per lane, double-buffered?): 32 operand words in
    // registers each (16 x 1 double-buffered would spill)
    using KFn = void (*)(uint64_t*, const uint64_t*, const uint64_t*, uint32_t*, size_t, size_t, uint32_t, uint32_t);
    static constexpr int kNV = 7;
    static const KFn kfn[kNV] = {k_addsub_ilf<SUB, 16, 1, false>, k_addsub_ilf<SUB, 8, 1, false>,
                                 k_addsub_ilf<SUB, 8, 2, false>,  k_addsub_ilf<SUB, 8, 1, true>,
                                 k_addsub_ilf<SUB, 4, 2, true>,   k_addsub_ilf<SUB, 4, 4, false>,
                                 k_addsub_ilf<SUB, 2, 4, true>};
    static constexpr int kUN[kNV] = {16, 8, 8, 8, 4, 4, 2};
    // resident CTAs per SM for each (variant, W = 1 ... 16)
    static thread_local struct { int dev = -1; int per[kNV][5]; } oc;
    if (oc.dev != dev) {
        for (int v = 0; v < kNV; ++v)
            for (int i = 0; i < 5; ++i) {
                int n = 0;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, reinterpret_cast<const void*>(kfn[v]), 32 << i, 0);
                oc.per[v][i] = n > 0 ? n : 1;
            }
        oc.dev = dev;
    }
    static const int g_knob = [] {
        const char* e = std::getenv("DOTG_ILF_G");  // A/B knob: lanes per segment (32, 16, 8; 0 = auto)
        return e ? std::atoi(e) : 0;
    }();
    // Shape: lanes per segment G, W = 2^wi warps per CTA, strips of G * PPL pairs, S = W * 32
    // / G segments per strip. Every segment streams at least one chunk and the grid is ONE
    // wave (warps stream their rows; a second wave would start late and end the launch
    // with a tail); among those, the most warps weighted by the share of SMs given a CTA
    // (ncu: with fewer strips than SMs the rest idle). Ties keep G = 32 (whole 128-byte
    // lines per warp row) and 16-byte rows.
    struct Shape { int kv = 0, wi = 0; uint32_t G = 32; size_t strips = 0; double score = -1.0; };
    auto consider = [&](Shape& best, int kv, int ppl) {
        for (uint32_t G = 32; G >= 8; G /= 2) {
            if (g_knob != 0 && uint32_t(g_knob) != G) continue;
            const size_t strips = (batch + size_t(G) * ppl - 1) / (size_t(G) * ppl);
            int wi = 4;
            while (wi > 0 && (strips > size_t(oc.per[kv][wi]) * size_t(di.sms) ||
                              ((size_t(kUN[kv]) << wi) * (32 / G)) > m))
                --wi;
            for (int d = wdiv; d > 1 && wi > 0; d /= 2) --wi;
            // resident warps x share of SMs with a CTA x whole-wave efficiency (a grid that
            // does not fit one wave even at W = 1 ends with a partial wave)
            const double cap = double(oc.per[kv][wi]) * double(di.sms);
            const double waves = double(strips) / cap;
            const double sc = std::min(double(strips), cap) * double(1 << wi) *
                              std::min(1.0, double(strips) / double(di.sms)) *
                              (waves <= 1.0 ? 1.0 : waves / std::ceil(waves));
            if (sc > best.score * 1.0001) best = Shape{kv, wi, G, strips, sc};
        }
    };
    const uintptr_t al = reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(a) |
                         reinterpret_cast<uintptr_t>(b);
    const bool can2 = batch % 2 == 0 && (al & 15u) == 0;
    const bool can4 = batch % 4 == 0 && (al & 31u) == 0;
    const int v1 = db_knob ? 3 : (un_knob == 8 ? 1 : 0), v2 = db_knob ? 4 : 2, v4 = db_knob ? 6 : 5;
    Shape sh;
    if (ppl_knob == 4 && can4) {
        consider(sh, v4, 4);
    } else if (ppl_knob == 2 && can2) {
        consider(sh, v2, 2);
    } else if (ppl_knob == 1 || !can2) {
        consider(sh, v1, 1);
    } else {  // 16-byte rows unless 8-byte rows give more warps on more SMs
        consider(sh, v2, 2);
        consider(sh, v1, 1);
    }
    const int W = 1 << sh.wi;
    const uint32_t S = uint32_t(W) * (32u / sh.G);
    const uint32_t L = uint32_t((m + S - 1) / S);
    kfn[sh.kv]<<<unsigned(sh.strips), W * 32, 0, st>>>(out, a, b, flags, m, batch, L, sh.G);
    count_launch();
    return cudaGetLastError();
}

// Interleaved layout, thread per pair fed by a TMA ring (k_addsub_ilt): a one-warp CTA
// owns a strip of P pairs (P * 8 contiguous bytes of every limb row) and walks all m rows
// of its strip serially, one carry per thread, like the limb-serial oracle
// (oracle.cpp:16-48) - no segments, no fix-up. Its operands arrive through an S-stage ring
// of [R rows][P pairs] boxes, one 2-D tensor copy (cp.async.bulk.tensor, the TMA engine)
// per operand and stage, so S * R rows per CTA are in flight without holding them in
// registers (the register-held loads of the thread-per-pair kernel cap it at 16 rows per
// lane: 0.52 of HBM at m = 128). Out-of-range pairs and rows of a box are zero-filled by
// the TMA unit. Every CTA has the same work and the grid fits the GPU at once, so the
// strips progress at the rate HBM serves them and end together (k_addsub_ilf's
// strip-per-CTA grid loses ~25% of the SM time to strips spread 1-2 per SM). Rows are
// stored straight from registers (coalesced P * 8 bytes per warp). Measured first with one
// 1-D bulk copy per row: a CTA then completed ~16 row copies per microsecond whatever the
// ring depth, so the time grew with m (m = 128: 0.88 of HBM, m = 256: 0.54, m = 1024:
// 0.15); a box per stage removes that per-copy cost.
// Needs batch even and 16-byte aligned operands (the tensor map's row stride and base).
template <bool SUB, int P, int R, int S>
__global__ void __launch_bounds__(P) k_addsub_ilt(const __grid_constant__ CUtensorMap ta,
                                                  const __grid_constant__ CUtensorMap tb,
                                                  uint64_t* __restrict__ out, uint32_t* __restrict__ flags, size_t m,
                                                  size_t batch) {
    static_assert(P <= 32 && P % 2 == 0, "one warp per strip, 16-byte rows");
    constexpr unsigned kMask = P == 32 ? 0xffffffffu : (1u << P) - 1u;  // the CTA's lanes
    constexpr uint32_t kBox = R * P * 8;                                 // bytes per operand box
    extern __shared__ __align__(128) uint64_t ring[];  // [S][2][R][P]
    __shared__ uint64_t bar[S];
    const int t = int(threadIdx.x);
    const size_t p0 = size_t(blockIdx.x) * P;
    const size_t nst = (m + R - 1) / R;
    auto issue = [&](size_t k) {  // lane 0: stage k into slot k % S
        const int s = int(k % S);
        uint64_t* dst = ring + size_t(s) * 2 * R * P;
        bulk::expect_tx(&bar[s], 2u * kBox);
        const int x = int(p0), y = int(k * R);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
            "[%4];" ::"r"(bulk::saddr(dst)),
            "l"(&ta), "r"(x), "r"(y), "r"(bulk::saddr(&bar[s]))
            : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
            "[%4];" ::"r"(bulk::saddr(dst + R * P)),
            "l"(&tb), "r"(x), "r"(y), "r"(bulk::saddr(&bar[s]))
            : "memory");
    };
    if (t == 0) {
        for (int s = 0; s < S; ++s) bulk::init(&bar[s]);
        bulk::init_fence();
        for (size_t k = 0; k < size_t(S) && k < nst; ++k) issue(k);
    }
    __syncwarp(kMask);
    const bool act = p0 + size_t(t) < batch;
    uint32_t c = 0;
    for (size_t k = 0; k < nst; ++k) {
        const int s = int(k % S);
        bulk::wait(&bar[s], uint32_t(k / S) & 1u);
        const uint64_t* sa = ring + size_t(s) * 2 * R * P + t;
        const uint64_t* sb = sa + R * P;
        const size_t r0 = k * R;
        uint64_t x[R], y[R];
#pragma unroll
        for (int r = 0; r < R; ++r) x[r] = sa[r * P], y[r] = sb[r * P];
        if (act) {
            uint64_t* po = out + r0 * batch + p0 + t;
            if (r0 + R <= m) {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    uint32_t g, p;
                    const uint64_t v = apply_carry<SUB>(lane_op<SUB>(x[r], y[r], g, p), c);
                    c = g | (p & c);
                    __stcs(po + size_t(r) * batch, v);
                }
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r)
                    if (r0 + r < m) {
                        uint32_t g, p;
                        const uint64_t v = apply_carry<SUB>(lane_op<SUB>(x[r], y[r], g, p), c);
                        c = g | (p & c);
                        __stcs(po + size_t(r) * batch, v);
                    }
            }
        }
        // slot s is consumed (its values were used above): refill it with stage k + S
        __syncwarp(kMask);
        if (t == 0 && k + S < nst) issue(k + S);
    }
    if (act && flags != nullptr) flags[p0 + t] = c;
}

// Tensor map of one [m][batch] u64 operand with [R][P] boxes (cuTensorMapEncodeTiled
// through the runtime's driver entry point: no link against libcuda).
bool encode_rows_map(CUtensorMap* map, const uint64_t* base, size_t m, size_t batch, uint32_t P, uint32_t R) {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }();
    if (fn == nullptr) return false;
    const cuuint64_t dims[2] = {cuuint64_t(batch), cuuint64_t(m)};
    const cuuint64_t strides[1] = {cuuint64_t(batch) * 8u};
    const cuuint32_t box[2] = {P, R};
    const cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<uint64_t*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Shape for k_addsub_ilt: 32-pair strips (256-byte box rows) when that gives at least two
// strips per SM, else 16-pair strips; 8-row stages, as many of them in flight per strip
// (4, 8 or 16) as keep every strip of the grid resident at once. Returns
// cudaErrorNotSupported for shapes it does not take (odd batch, unaligned operands, no
// tensor-map entry point, 2^31 or more pairs or rows).
template <bool SUB>
cudaError_t run_interleaved_ilt(uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags, size_t m,
                                size_t batch, cudaStream_t st) {
    if (batch % 2 != 0 || (reinterpret_cast<uintptr_t>(a) & 15u) != 0 || (reinterpret_cast<uintptr_t>(b) & 15u) != 0 ||
        batch >= (size_t(1) << 31) || m >= (size_t(1) << 31))  // TMA box coordinates are signed 32-bit
        return cudaErrorNotSupported;
    static thread_local struct { int dev = -1, sms = 148, smem_sm = 233472, smem_cta = 232448; } di;
    int dev = 0;
    cudaGetDevice(&dev);
    if (di.dev != dev) {
        cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&di.smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        cudaDeviceGetAttribute(&di.smem_cta, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        di.dev = dev;
    }
    static const int s_knob = [] {
        const char* e = std::getenv("DOTG_ILT_STAGES");  // A/B knob: 4, 8 or 16 stages (0 = auto)
        return e ? std::atoi(e) : 0;
    }();
    static const int p_knob = [] {
        const char* e = std::getenv("DOTG_ILT_P");  // A/B knob: 16 or 32 pairs per strip (0 = auto)
        return e ? std::atoi(e) : 0;
    }();
    static const int r_knob = [] {
        const char* e = std::getenv("DOTG_ILT_R");  // A/B knob: rows per stage (8 or 32; 0 = auto)
        return e ? std::atoi(e) : 0;
    }();
    const bool wide = p_knob ? p_knob == 32 : (batch + 31) / 32 >= 2 * size_t(di.sms);
    const int PP = wide ? 32 : 16;
    const size_t strips = (batch + PP - 1) / PP;
    if (strips > size_t(0x7fffffff)) return cudaErrorNotSupported;
    CUtensorMap ta, tb;
    // (rows per stage R, stages S): the most rows in flight per strip with every strip of
    // the grid resident at once (each CTA also takes ~1 KB of reserved and static shared
    // memory), ties to the bigger box - a CTA's TMA boxes complete at a rate set by their
    // count more than their bytes (m = 512: R = 32 x 4 stages 0.86 of HBM, R = 8 x 16 0.67).
    // When no shape fits one wave, the smallest. (64- and 128-row boxes measured slower:
    // m = 1024 at B = 4096 0.41 with 64 x 4 against 0.59 with 32 x 8.)
    const size_t per_sm = (strips + di.sms - 1) / di.sms;
    static constexpr int kRS[6][2] = {{32, 16}, {32, 8}, {32, 4}, {8, 16}, {8, 8}, {8, 4}};
    int pick = 5;
    for (int i = 0; i < 6; ++i) {
        const size_t bytes = size_t(kRS[i][0]) * kRS[i][1] * 2 * PP * 8 + 2048;
        const bool fits = per_sm * bytes <= size_t(di.smem_sm) && bytes - 2048 <= size_t(di.smem_cta);
        const int rows = kRS[i][0] * kRS[i][1], best = kRS[pick][0] * kRS[pick][1];
        const bool pick_fits = per_sm * (size_t(kRS[pick][0]) * kRS[pick][1] * 2 * PP * 8 + 2048) <= size_t(di.smem_sm);
        if (fits && (!pick_fits || rows > best)) pick = i;
    }
    for (int i = 0; i < 6; ++i)  // A/B knobs
        if ((r_knob == 0 || r_knob == kRS[i][0]) && (s_knob == 0 || s_knob == kRS[i][1]) && (r_knob || s_knob) &&
            size_t(kRS[i][0]) * kRS[i][1] * 2 * PP * 8 <= size_t(di.smem_cta)) {
            pick = i;
            break;
        }
    const int R = kRS[pick][0];
    if (!encode_rows_map(&ta, a, m, batch, uint32_t(PP), uint32_t(R)) ||
        !encode_rows_map(&tb, b, m, batch, uint32_t(PP), uint32_t(R)))
        return cudaErrorNotSupported;
#define DOTG_ILT_LAUNCH(P_, R_, S_)                                                                      \
    do {                                                                                                 \
        const size_t smem = size_t(S_) * 2 * (R_) * (P_) * sizeof(uint64_t);                              \
        static thread_local int attr_dev = -1;                                                           \
        if (attr_dev != dev) {                                                                           \
            cudaError_t e = cudaFuncSetAttribute(k_addsub_ilt<SUB, P_, R_, S_>,                           \
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)); \
            if (e != cudaSuccess) return e;                                                              \
            attr_dev = dev;                                                                              \
        }                                                                                                \
        k_addsub_ilt<SUB, P_, R_, S_><<<unsigned(strips), P_, smem, st>>>(ta, tb, out, flags, m, batch); \
    } while (0)
#define DOTG_ILT_SHAPES(P_)                              \
    switch (pick) {                                      \
        case 0: DOTG_ILT_LAUNCH(P_, 32, 16); break;      \
        case 1: DOTG_ILT_LAUNCH(P_, 32, 8); break;       \
        case 2: DOTG_ILT_LAUNCH(P_, 32, 4); break;       \
        case 3: DOTG_ILT_LAUNCH(P_, 8, 16); break;       \
        case 4: DOTG_ILT_LAUNCH(P_, 8, 8); break;        \
        default: DOTG_ILT_LAUNCH(P_, 8, 4); break;       \
    }
    if (PP == 32) {
        DOTG_ILT_SHAPES(32)
    } else {
        DOTG_ILT_SHAPES(16)
    }
#undef DOTG_ILT_SHAPES
#undef DOTG_ILT_LAUNCH
    count_launch();
    return cudaGetLastError();
}

// Interleaved layout, two streaming passes (no barrier, no register holding): the
// long-number scheme of addsub_long.cu applied to segments of kSL limbs x 32 pairs.
//   pass 1 (k_il_local): warp = (strip of 32 pairs, segment of kSL limb rows); every
//     load of the segment in flight, then the segment resolved with carry-in 0 and
//     stored at once; per (segment, pair) one state byte: G (carry out for carry-in 0),
//     P (every limb propagates), pt (first non-propagating limb, kSL if none). Only
//     limbs [0, pt] of a segment depend on its carry-in.
//   pass 2 (k_il_finish): thread per pair walks its S state bytes (coalesced across the
//     pairs), c_{j+1} = G_j | (P_j & c_j), and where c_j = 1 rewrites limbs [0, pt] of
//     segment j (propagate value below pt, +-1 at pt): on random data one 8-byte RMW per
//     segment with carry-in 1, mostly in the same limb row across a warp.
// Warps are numbered strip-fastest so concurrently running warps stream contiguous
// stretches of each limb row.
constexpr int kSL = 8;  // limbs per segment
// A batch of numbers of <= kSL limbs is one segment per pair: the flag is final in pass 1
// and the finish pass is skipped. (Measured r02, tools/il_modes.py, B x m = 2^22: pass 1
// with 4 pairs per lane and 256-bit row loads ran 2.6-3.9 TB/s, below 1 pair per lane.)
template <bool SUB>
__global__ void __launch_bounds__(256) k_il_local(uint64_t* __restrict__ out, const uint64_t* __restrict__ a,
                                                  const uint64_t* __restrict__ b, uint8_t* __restrict__ state,
                                                  uint32_t* __restrict__ flags, size_t m, size_t batch,
                                                  size_t nstrips, size_t nwarps) {
    const size_t gw = (size_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (gw >= nwarps) return;
    const size_t strip = gw % nstrips, seg = gw / nstrips;
    constexpr int PPL = 1;
    const size_t p = strip * 32 + (threadIdx.x & 31u);
    if (p >= batch) return;
    const size_t i0 = seg * kSL;
    const int L = int(m - i0 < size_t(kSL) ? m - i0 : size_t(kSL));
    uint64_t s[kSL][PPL], y[kSL][PPL];
#pragma unroll
    for (int k = 0; k < kSL; ++k) {
#pragma unroll
        for (int q = 0; q < PPL; ++q) s[k][q] = y[k][q] = 0;
        if (k < L) {
            const size_t off = (i0 + size_t(k)) * batch + p;
            s[k][0] = __ldcs(a + off);
            y[k][0] = __ldcs(b + off);
        }
    }
    uint32_t word = 0;
#pragma unroll
    for (int q = 0; q < PPL; ++q) {
        uint32_t c = 0, all = 1, pt = kSL;
#pragma unroll
        for (int k = 0; k < kSL; ++k)
            if (k < L) {
                uint32_t g, pr;
                const uint64_t v = lane_op<SUB>(s[k][q], y[k][q], g, pr);
                s[k][q] = apply_carry<SUB>(v, c);
                if (!pr && pt == kSL) pt = uint32_t(k);
                c = g | (pr & c);
                all &= pr;
            }
        if (pt > uint32_t(L)) pt = uint32_t(L);
        word |= (c | (all << 1) | (pt << 2)) << (8 * q);
        if (m <= size_t(kSL) && flags != nullptr) flags[p + q] = c;
    }
#pragma unroll
    for (int k = 0; k < kSL; ++k)
        if (k < L) {
            const size_t off = (i0 + size_t(k)) * batch + p;
            __stcs(out + off, s[k][0]);
        }
    if (m > size_t(kSL)) state[seg * batch + p] = uint8_t(word);
}

template <bool SUB>
__global__ void __launch_bounds__(256) k_il_finish(uint64_t* __restrict__ out, const uint8_t* __restrict__ state,
                                                   uint32_t* flags, size_t m, size_t batch, size_t nseg) {
    const size_t p = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= batch) return;
    constexpr int CH = 16;  // segments per round: their state loads, then their fix-up loads, in flight together
    uint32_t c = 0;
    for (size_t j0 = 0; j0 < nseg; j0 += CH) {
        uint32_t st[CH];
#pragma unroll
        for (int k = 0; k < CH; ++k)  // past the last segment: the identity {G, P} = {0, 1}
            st[k] = j0 + k < nseg ? uint32_t(__ldcs(state + (j0 + k) * batch + p)) : 2u;
        uint32_t cin = 0;  // bit k: carry into segment j0 + k
#pragma unroll
        for (int k = 0; k < CH; ++k) {
            cin |= c << k;
            c = (st[k] & 1u) | ((st[k] >> 1) & 1u & c);
        }
        if (j0 + CH > nseg) cin &= (1u << (nseg - j0)) - 1u;  // no fix-ups past the last segment
        if (cin == 0) continue;
        uint64_t v[CH];
#pragma unroll
        for (int k = 0; k < CH; ++k) {
            v[k] = 0;
            const size_t i0 = (j0 + k) * kSL;
            const uint32_t pt = st[k] >> 2;
            if (((cin >> k) & 1u) && i0 + pt < m && pt < uint32_t(kSL)) v[k] = out[(i0 + pt) * batch + p];
        }
#pragma unroll
        for (int k = 0; k < CH; ++k) {
            if (!((cin >> k) & 1u)) continue;
            const size_t i0 = (j0 + k) * kSL;
            const uint32_t pt = st[k] >> 2;
            for (uint32_t q = 0; q < pt; ++q) out[(i0 + q) * batch + p] = prop_value<SUB>(1u);
            if (i0 + pt < m && pt < uint32_t(kSL)) out[(i0 + pt) * batch + p] = apply_carry<SUB>(v[k], 1u);
        }
    }
    if (flags != nullptr) flags[p] = c;
}

// Row-major, any m (no power-of-two team shape): the batch is one flat limb array, so a
// warp walks a task of whole pairs as 128-limb chunks (lane = 4 consecutive limbs, one
// 256-bit load per operand when aligned) and resolves carries with the ballot mask
// addition of the team kernels made *segmented*: a limb that starts a pair resets the
// carry, so in the lane fold it clears both G and P (nothing crosses a pair boundary),
// and the flag of a pair is the carry out of its last limb. Pair positions advance by
// the precomputed 128 / m and 128 % m per chunk - no division in the loop.
template <bool SUB, int U>
__global__ void __launch_bounds__(256) k_addsub_rows_any(uint64_t* __restrict__ out, const uint64_t* __restrict__ a,
                                                         const uint64_t* __restrict__ b, uint32_t* flags, size_t m,
                                                         size_t batch, size_t ppt, size_t ntasks, bool vec) {
    const int lane = threadIdx.x & 31;
    const size_t nwarps = size_t(gridDim.x) * (blockDim.x >> 5);
    const uint32_t mm = uint32_t(m);  // m < 2^32 (checked by the launcher)
    const uint32_t q128 = 128u / mm, r128 = 128u % mm;
    const uint32_t l4 = 4u * uint32_t(lane);
    const uint32_t q_l = l4 / mm, r_l = l4 % mm;
    for (size_t task = size_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); task < ntasks; task += nwarps) {
        const size_t p0 = task * ppt;
        const size_t p1 = p0 + ppt < batch ? p0 + ppt : batch;
        const size_t end = p1 * m;
        size_t pidx = p0 + q_l;  // pair of this lane's first limb in the current chunk
        uint32_t pos = r_l;      // its position inside that pair
        uint32_t cin = 0;        // carry into the chunk
        // U chunks of 128 limbs per step: every load of the step in flight before the
        // first chunk's carries resolve (r02: one chunk at a time held odd m at 0.70-0.79
        // of HBM and m = 4096 rows at 0.45)
        for (size_t cb0 = p0 * m; cb0 < end; cb0 += 128 * U) {
            uint64_t x[U][4], y[U][4];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const size_t f = cb0 + 128 * u + l4;
#pragma unroll
                for (int k = 0; k < 4; ++k) x[u][k] = y[u][k] = 0;
                if (vec && f + 3 < end) {
                    ld_stream<4>(a + f, x[u]);
                    ld_stream<4>(b + f, y[u]);
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (f + k < end) {
                            x[u][k] = a[f + k];
                            y[u][k] = b[f + k];
                        }
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const size_t cb = cb0 + 128 * u;
                if (cb >= end) break;
                const size_t f = cb + l4;
                uint64_t sv[4];
                uint32_t g[4], pr[4], start = 0, last = 0;
                uint32_t G = 0, P = 1;
                {
                    uint32_t ps = pos;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const bool ok = f + k < end;
                        sv[k] = lane_op<SUB>(x[u][k], y[u][k], g[k], pr[k]);
                        if (!ok) g[k] = pr[k] = 0;
                        if (ok && ps == 0) start |= 1u << k;
                        if (ok && ps + 1 == mm) last |= 1u << k;
                        if ((start >> k) & 1u) G = P = 0;  // a pair starts: nothing enters from below
                        G = g[k] | (pr[k] & G);
                        P &= pr[k];
                        ps = ps + 1 == mm ? 0 : ps + 1;
                    }
                }
                const uint32_t Gm = __ballot_sync(0xffffffffu, G), Pm = __ballot_sync(0xffffffffu, P);
                const uint64_t yv = ((uint64_t(Gm) << 1) | cin) + uint64_t(Pm);
                uint32_t c = ((uint32_t(yv) ^ Pm) >> lane) & 1u;
                cin = uint32_t(yv >> 32);
                size_t pq = pidx;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if ((start >> k) & 1u) c = 0;
                    const uint64_t o = apply_carry<SUB>(sv[k], c);
                    c = g[k] | (pr[k] & c);
                    sv[k] = o;
                    if ((last >> k) & 1u) {
                        if (flags != nullptr) flags[pq] = c;
                        ++pq;
                    }
                }
                if (vec && f + 3 < end) {
                    st_stream<4>(out + f, sv);
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (f + k < end) out[f + k] = sv[k];
                }
                pidx += q128;
                pos += r128;
                if (pos >= mm) {
                    pos -= mm;
                    ++pidx;
                }
            }
        }
    }
}

namespace {

// segment state fits a modest scratch, and the grid fits 32-bit block counts
bool nseg_fits(size_t m, size_t batch) {
    const size_t nseg = (m + kSL - 1) / kSL;
    return nseg * batch <= (size_t(1) << 32) && (nseg * ((batch + 31) / 32) + 7) / 8 < (size_t(1) << 31);
}

template <bool SUB>
cudaError_t run_interleaved_2pass(uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags, size_t m,
                                  size_t batch, cudaStream_t st) {
    const size_t nseg = (m + kSL - 1) / kSL, nstrips = (batch + 31) / 32;
    const size_t nwarps = nseg * nstrips;
    uint8_t* state = nullptr;
    cudaError_t e = cudaSuccess;
    if (nseg > 1) {
        retain_stream_pool();
        e = cudaMallocAsync(reinterpret_cast<void**>(&state), nseg * batch, st);
        if (e != cudaSuccess) return e;
    }
    k_il_local<SUB><<<unsigned((nwarps + 7) / 8), 256, 0, st>>>(out, a, b, state, flags, m, batch, nstrips, nwarps);
    count_launch();
    e = cudaGetLastError();
    if (nseg == 1) return e;
    if (e == cudaSuccess) {
        k_il_finish<SUB><<<unsigned((batch + 255) / 256), 256, 0, st>>>(out, state, flags, m, batch, nseg);
        count_launch();
        e = cudaGetLastError();
    }
    cudaError_t e2 = cudaFreeAsync(state, st);
    return e != cudaSuccess ? e : e2;
}

// Interleaved routes, per-launch fraction of HBM when launches run back to back (CUDA
// graph over 3 rotating input copies, tools/il_graph.py; B200, B x m = 2^22 limbs) at
// m = 4 / 16 / 32 / 64 / 128 / 256 / 512 / 1024 (profiles/r02_il_graph*.jsonl):
//   thread per pair (r01 tail)   0.77 / 0.86 / 0.90 / 0.75 / 0.52 / 0.30 / 0.17 / 0.09
//   re-read CTAs (il2)           0.77 / 0.73 / 0.74 / 0.74 / 0.71 / 0.69 / 0.67 / 0.64
//   two passes                   0.82 / 0.56 / 0.64 / 0.71 / 0.69 / 0.60 / 0.48 / 0.35
//   streaming + fix-up (ilf)        - / 0.84 / 0.83 / 0.82 / 0.80 / 0.80 / 0.77 / 0.72
//   TMA box ring (ilt)           0.57 / 0.88 / 0.87 / 0.85 / 0.88 / 0.86 / 0.86 / 0.59
// Auto (profiles/r02_il_graph_auto_final.jsonl: 0.80-0.91 for m = 1 ... 512, 0.76 at
// m = 1024 with 4096 pairs): k_addsub_il_tiny for m <= 3 (4 pairs per thread, 32-byte
// rows; 0.89-0.91, where ilf ran 0.09-0.23), thread per pair below 48 limbs (two pairs per
// thread under 8 limbs; 0.85-0.91), k_addsub_ilt from 48 limbs for even batches of >= 8192
// pairs, k_addsub_ilf otherwise, except a few very long numbers (m > 2048 and fewer than
// 4096 pairs), which take the two-pass route (its warps are (strip, segment) pairs, so they
// still fill the GPU). DOTG_IL_MODE (A/B knob) forces 2 (thread per pair), 3 (il2), 4 (two
// passes), 5 (ilf), 6 (ilt) or 7 (il_tiny) where they apply.
int il_mode() {
    static const int v = [] {
        const char* e = std::getenv("DOTG_IL_MODE");
        return e ? std::atoi(e) : 0;
    }();
    return v;
}
int il_route(size_t m, size_t batch) {
    const int mode = il_mode();
    if (mode == 2) return 0;
    if (mode == 3) return m >= 16 ? 3 : 0;
    if (mode == 4) return nseg_fits(m, batch) ? 4 : 0;
    if (mode == 5) return m >= 2 && (batch + 7) / 8 <= size_t(0x7fffffff) ? 5 : 0;
    if (mode == 6) return 6;  // k_addsub_ilt where it applies (else thread per pair)
    if (mode == 7) return m <= 3 ? 7 : 0;  // k_addsub_il_tiny where it applies
    if (m <= 3) return 7;                                      // 4 pairs per thread, 32-byte rows
    if ((batch + 7) / 8 > size_t(0x7fffffff)) return 0;        // ilf's grid has a CTA per strip
    if (m < 48) return 0;                                      // thread per pair
    if (batch >= 8192 && batch % 2 == 0) return 6;             // thread per pair on a TMA ring
    if (m <= 2048 || batch >= 4096) return 5;                  // streaming pass + in-CTA fix-up
    return nseg_fits(m, batch) ? 4 : 5;  // a few very long numbers: (strip, segment) warps fill the GPU
}

template <bool SUB>
cudaError_t run_strided(uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags,
                        size_t m, size_t batch, size_t sp, size_t si, cudaStream_t st) {
    static const unsigned bs = [] {
        const char* e = std::getenv("DOTG_TPP_BLOCK");  // A/B knob: threads per CTA (32 ... 256)
        const int v = e ? std::atoi(e) : 256;
        return unsigned(v >= 32 && v <= 256 ? v : 256);
    }();
    static const int vp_knob = [] {
        const char* e = std::getenv("DOTG_TPP_VP");  // A/B knob: pairs per thread (1 or 2; 0 = auto)
        return e ? std::atoi(e) : 0;
    }();
    // two pairs per thread: interleaved rows, even batch, 16-byte aligned rows, and a
    // grid that still has >= 8 threads per SM lane slot (small m, big batch)
    const bool can2 = sp == 1 && batch % 2 == 0 && si % 2 == 0 &&
                      ((reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(a) |
                        reinterpret_cast<uintptr_t>(b)) & 15u) == 0;
    const bool two = can2 && (vp_knob ? vp_knob == 2 : (m < 8 && batch >= (size_t(1) << 20)));
    const size_t threads = two ? batch / 2 : batch;
    const size_t blocks = (threads + bs - 1) / bs;
    if (two) k_addsub_strided<SUB, 2><<<unsigned(blocks), bs, 0, st>>>(out, a, b, flags, m, batch, sp, si);
    else k_addsub_strided<SUB, 1><<<unsigned(blocks), bs, 0, st>>>(out, a, b, flags, m, batch, sp, si);
    count_launch();
    return cudaGetLastError();
}

bool aligned(const void* p, size_t bytes) { return (reinterpret_cast<uintptr_t>(p) % bytes) == 0; }

// k_addsub_il_tiny for 1 <= m <= 3: batch % 4 == 0, rows 32-byte aligned (operands and
// output), flags 16-byte aligned; cudaErrorNotSupported otherwise.
template <bool SUB>
cudaError_t run_il_tiny(uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags, size_t m, size_t batch,
                        cudaStream_t st) {
    if (m < 1 || m > 3 || batch % 4 != 0 || !aligned(out, 32) || !aligned(a, 32) || !aligned(b, 32) ||
        (flags != nullptr && !aligned(flags, 16)))
        return cudaErrorNotSupported;
    const size_t blocks = (batch / 4 + 255) / 256;
    if (blocks > size_t(0x7fffffff)) return cudaErrorNotSupported;
    if (m == 1) k_addsub_il_tiny<SUB, 1><<<unsigned(blocks), 256, 0, st>>>(out, a, b, flags, batch);
    else if (m == 2) k_addsub_il_tiny<SUB, 2><<<unsigned(blocks), 256, 0, st>>>(out, a, b, flags, batch);
    else k_addsub_il_tiny<SUB, 3><<<unsigned(blocks), 256, 0, st>>>(out, a, b, flags, batch);
    count_launch();
    return cudaGetLastError();
}

// k_addsub_rows_staged: P pairs per CTA (a multiple of 32, at most 128) so that a CTA's
// two operand stages fit ~48 KB (4 CTAs per SM); 16-byte aligned operands and output.
template <bool SUB>
cudaError_t run_rows_staged(uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags, size_t m,
                            size_t batch, cudaStream_t st) {
    if (m < 3 || m >= 64 || !aligned(out, 16) || !aligned(a, 16) || !aligned(b, 16)) return cudaErrorNotSupported;
    uint32_t P = uint32_t((48 * 1024) / (16 * m)) & ~31u;
    if (P > 128) P = 128;
    if (P < 32) P = 32;
    const size_t smem = size_t(2) * P * m * 8;
    const size_t blocks = (batch + P - 1) / P;
    if (blocks > size_t(0x7fffffff)) return cudaErrorNotSupported;
    static thread_local int attr_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (attr_dev != dev) {  // up to 63 KB at m = 63 (P = 32)
        cudaError_t e = cudaFuncSetAttribute(k_addsub_rows_staged<SUB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             64 * 1024);
        if (e != cudaSuccess) return e;
        attr_dev = dev;
    }
    k_addsub_rows_staged<SUB><<<unsigned(blocks), P, smem, st>>>(out, a, b, flags, uint32_t(m), batch, P);
    count_launch();
    return cudaGetLastError();
}

constexpr int kRowsU = 4;  // chunks of 128 limbs in flight per warp
template <bool SUB>
cudaError_t run_rows_any(uint64_t* out, const uint64_t* a, const uint64_t* b, uint32_t* flags, size_t m,
                         size_t batch, cudaStream_t st) {
    // tasks of whole pairs, ~512 limbs each, with a limb count that keeps every task start
    // 4-limb (32-byte) aligned so the 256-bit path applies throughout
    static const int rows_u = [] {
        const char* e = std::getenv("DOTG_ROWS_U");  // A/B knob: chunks in flight per warp (1, 2, 4)
        const int v = e ? std::atoi(e) : kRowsU;
        return v == 1 || v == 2 ? v : kRowsU;
    }();
    size_t ppt = m >= 512 ? 1 : 512 / m;
    const size_t g4 = (m % 4 == 0) ? 1 : (m % 2 == 0 ? 2 : 4);  // pairs per 4-limb alignment
    ppt = (ppt + g4 - 1) / g4 * g4;
    const bool vec = (ppt * m) % 4 == 0 && aligned(out, 32) && aligned(a, 32) && aligned(b, 32);
    const size_t ntasks = (batch + ppt - 1) / ppt;
    static thread_local struct { int dev = -1, cap = 0; } di;
    int dev = 0;
    cudaGetDevice(&dev);
    if (di.dev != dev) {
        int sms = 0, per = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_addsub_rows_any<SUB, kRowsU>, 256, 0);
        di.cap = sms * (per > 0 ? per : 1);
        di.dev = dev;
    }
    const size_t need = (ntasks + 7) / 8;
    const unsigned grid = unsigned(need < size_t(di.cap) ? need : size_t(di.cap));
    if (rows_u == 1) k_addsub_rows_any<SUB, 1><<<grid, 256, 0, st>>>(out, a, b, flags, m, batch, ppt, ntasks, vec);
    else if (rows_u == 2) k_addsub_rows_any<SUB, 2><<<grid, 256, 0, st>>>(out, a, b, flags, m, batch, ppt, ntasks, vec);
    else k_addsub_rows_any<SUB, kRowsU><<<grid, 256, 0, st>>>(out, a, b, flags, m, batch, ppt, ntasks, vec);
    count_launch();
    return cudaGetLastError();
}
bool pow2(size_t m) { return m != 0 && (m & (m - 1)) == 0; }
// DOTG_ROWS_STAGED=0 (A/B): row-major 3 <= m <= 7 off the powers of two on k_addsub_rows_any
bool rows_staged_on() {
    static const int v = [] {
        const char* e = std::getenv("DOTG_ROWS_STAGED");
        return e ? std::atoi(e) : 1;
    }();
    return v != 0;
}

// 0: team-small kernel, 1: team-big (m = 512), 2: strided kernel
int route(const AddSubProblem& P, int layout) {
    if (layout == 1 || !pow2(P.m) || P.m > 512) return 2;
    const size_t need = P.m >= 4 ? 32 : P.m * 8;
    if (!aligned(P.out, need) || !aligned(P.a, need) || !aligned(P.b, need)) return 2;
    return P.m == 512 ? 1 : 0;
}

struct DevInfo {
    int dev = -1, sms = 148, blocks_small = 8, blocks_big = 4;
};

const DevInfo& dev_info() {
    static thread_local DevInfo info;
    int dev = 0;
    cudaGetDevice(&dev);
    if (info.dev != dev) {
        info.dev = dev;
        cudaDeviceGetAttribute(&info.sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&info.blocks_small, k_addsub_grouped<false>, 256, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&info.blocks_big, k_addsub_grouped<true>, 256, 0);
        if (info.blocks_small < 1) info.blocks_small = 1;
        if (info.blocks_big < 1) info.blocks_big = 1;
    }
    return info;
}

cudaError_t launch_group(bool big, AddSubGroup& g, cudaStream_t st) {
    if (g.n == 0 || g.total_tasks == 0) return cudaSuccess;
    const DevInfo& di = dev_info();
    const uint64_t need_blocks = (g.total_tasks + 7) / 8;  // 8 warps per CTA
    const uint64_t cap = uint64_t(di.sms) * uint64_t(big ? di.blocks_big : di.blocks_small);
    const unsigned blocks = unsigned(need_blocks < cap ? need_blocks : cap);
    if (big) k_addsub_grouped<true><<<blocks, 256, 0, st>>>(g);
    else k_addsub_grouped<false><<<blocks, 256, 0, st>>>(g);
    count_launch();
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_addsub_group(const AddSubProblem* probs, const int* layouts, int n, cudaStream_t stream) {
    AddSubGroup small{}, big{};
    for (int i = 0; i < n; ++i) {
        AddSubProblem P = probs[i];
        if (P.batch == 0) continue;
        if (P.m == 0) {
            if (P.flags != nullptr) {
                cudaError_t e = cudaMemsetAsync(P.flags, 0, P.batch * sizeof(uint32_t), stream);
                if (e != cudaSuccess) return e;
            }
            continue;
        }
        // one limb per number: [batch][1] and [1][batch] are the same array, so m = 1 takes
        // the interleaved routes (k_addsub_il_tiny: 0.90 of HBM vs 0.72 on the team kernel)
        const int lay = P.m == 1 ? 1 : layouts[i];
        const int r = route(P, lay);
        if (r == 2 && lay == 1) {
            const int ir = il_route(P.m, P.batch);
            if (ir != 0) {
                cudaError_t e;
                if (ir == 3)
                    e = P.sub ? run_interleaved_il2<true>(P.out, P.a, P.b, P.flags, P.m, P.batch, stream)
                              : run_interleaved_il2<false>(P.out, P.a, P.b, P.flags, P.m, P.batch, stream);
                else if (ir == 5)
                    e = P.sub ? run_interleaved_ilf<true>(P.out, P.a, P.b, P.flags, P.m, P.batch, stream)
                              : run_interleaved_ilf<false>(P.out, P.a, P.b, P.flags, P.m, P.batch, stream);
                else if (ir == 7) {
                    e = P.sub ? run_il_tiny<true>(P.out, P.a, P.b, P.flags, P.m, P.batch, stream)
                              : run_il_tiny<false>(P.out, P.a, P.b, P.flags, P.m, P.batch, stream);
                    if (e == cudaErrorNotSupported)  // batch % 4 or alignment
                        e = P.sub ? run_strided<true>(P.out, P.a, P.b, P.flags, P.m, P.batch, 1, P.batch, stream)
                                  : run_strided<false>(P.out, P.a, P.b, P.flags, P.m, P.batch, 1, P.batch, stream);
                } else if (ir == 6) {
                    e = P.sub ? run_interleaved_ilt<true>(P.out, P.a, P.b, P.flags, P.m, P.batch, stream)
                              : run_interleaved_ilt<false>(P.out, P.a, P.b, P.flags, P.m, P.batch, stream);
                    if (e == cudaErrorNotSupported && P.m >= 2)  // odd batch or unaligned rows
                        e = P.sub ? run_interleaved_ilf<true>(P.out, P.a, P.b, P.flags, P.m, P.batch, stream)
                                  : run_interleaved_ilf<false>(P.out, P.a, P.b, P.flags, P.m, P.batch, stream);
                    else if (e == cudaErrorNotSupported)
                        e = P.sub ? run_strided<true>(P.out, P.a, P.b, P.flags, P.m, P.batch, 1, P.batch, stream)
                                  : run_strided<false>(P.out, P.a, P.b, P.flags, P.m, P.batch, 1, P.batch, stream);
                }
                else
                    e = P.sub ? run_interleaved_2pass<true>(P.out, P.a, P.b, P.flags, P.m, P.batch, stream)
                              : run_interleaved_2pass<false>(P.out, P.a, P.b, P.flags, P.m, P.batch, stream);
                if (e != cudaSuccess) return e;
                continue;
            }
        }
        // long numbers: two tiles (8192 limbs) or more each -> the tiled long-number passes
        // for the whole batch (a warp walking a pair's chunks serially would leave the GPU
        // idle for batches of a few numbers: tools/long_batch_timing.py)
        if (layouts[i] == 0 && P.m >= 8192 && P.batch <= 65535) {
            cudaError_t e = launch_long_batch(P.sub != 0, P.out, P.a, P.b, P.flags, P.m, P.batch, stream);
            if (e != cudaSuccess) return e;
            continue;
        }
        if (r == 2 && layouts[i] == 0 && P.m >= 3 && P.m <= 7 && rows_staged_on()) {
            cudaError_t e = P.sub ? run_rows_staged<true>(P.out, P.a, P.b, P.flags, P.m, P.batch, stream)
                                  : run_rows_staged<false>(P.out, P.a, P.b, P.flags, P.m, P.batch, stream);
            if (e != cudaErrorNotSupported) {
                if (e != cudaSuccess) return e;
                continue;
            }
        }
        if (r == 2 && layouts[i] == 0 && P.m >= 3 && P.m < (size_t(1) << 31) &&
            aligned(P.out, 8) && aligned(P.a, 8) && aligned(P.b, 8)) {
            cudaError_t e = P.sub ? run_rows_any<true>(P.out, P.a, P.b, P.flags, P.m, P.batch, stream)
                                  : run_rows_any<false>(P.out, P.a, P.b, P.flags, P.m, P.batch, stream);
            if (e != cudaSuccess) return e;
            continue;
        }
        if (r == 2) {
            const bool inter = layouts[i] == 1;
            cudaError_t e = P.sub ? run_strided<true>(P.out, P.a, P.b, P.flags, P.m, P.batch, inter ? 1 : P.m,
                                                      inter ? P.batch : 1, stream)
                                  : run_strided<false>(P.out, P.a, P.b, P.flags, P.m, P.batch, inter ? 1 : P.m,
                                                       inter ? P.batch : 1, stream);
            if (e != cudaSuccess) return e;
            continue;
        }
        AddSubGroup& g = r == 1 ? big : small;
        if (g.n == kMaxGroup) {
            cudaError_t e = launch_group(r == 1, g, stream);
            if (e != cudaSuccess) return e;
            g = AddSubGroup{};
        }
        P.task_begin = g.total_tasks;
        g.total_tasks += (P.batch + numbers_per_task(P.m) - 1) / numbers_per_task(P.m);
        g.p[g.n++] = P;
    }
    cudaError_t e = launch_group(false, small, stream);
    if (e != cudaSuccess) return e;
    return launch_group(true, big, stream);
}

cudaError_t launch_addsub_pitched(bool sub, uint64_t* out, size_t ldo, const uint64_t* a, size_t lda,
                                  const uint64_t* b, size_t ldb, uint32_t* flags, size_t m, size_t batch,
                                  cudaStream_t stream) {
    if (batch == 0) return cudaSuccess;
    if (ldo == m && lda == m && ldb == m) return launch_addsub_batch(sub, out, a, b, flags, m, batch, 0, stream);
    const unsigned blocks = unsigned((batch + 255) / 256);
    if (sub) k_addsub_pitched<true><<<blocks, 256, 0, stream>>>(out, ldo, a, lda, b, ldb, flags, m, batch);
    else k_addsub_pitched<false><<<blocks, 256, 0, stream>>>(out, ldo, a, lda, b, ldb, flags, m, batch);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_addsub_batch(bool sub, uint64_t* out, const uint64_t* a, const uint64_t* b,
                                uint32_t* flags, size_t m, size_t batch, int layout,
                                cudaStream_t stream) {
    AddSubProblem P{};
    P.out = out;
    P.a = a;
    P.b = b;
    P.flags = flags;
    P.batch = batch;
    P.m = uint32_t(m);
    P.sub = sub ? 1u : 0u;
    if (m > 0xffffffffull) {
        // absurdly long rows: only the strided kernel takes a 64-bit m
        return sub ? run_strided<true>(out, a, b, flags, m, batch, layout == 1 ? 1 : m, layout == 1 ? batch : 1, stream)
                   : run_strided<false>(out, a, b, flags, m, batch, layout == 1 ? 1 : m, layout == 1 ? batch : 1, stream);
    }
    return launch_addsub_group(&P, &layout, 1, stream);
}

}  // namespace dotg
