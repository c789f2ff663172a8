// stats.cu - instrumentation parity with the reference's AddSubStats counters
// (include/dot/addsub.hpp:53-72): chunks_processed and phase4_triggers.
//
// The reference runs each number as a serial chain of w-limb chunks (addsub.cpp:136-170;
// w = lane_count(Width): 8 for scalar/w8, 2, 4) and counts the chunks whose Phase 4 fired
// (addsub.cpp:48-79): Phase 3 adds the shifted lane carries c_i (c_i = g_{i-1} inside the
// chunk, the chunk's carry-in for its first lane) and Phase 4 fires iff some lane wraps,
// i.e. iff some lane has c_i = 1 and propagates (s_i == ~0 for add, s_i == 0 for sub).
//
// The device path never runs those phases (it resolves every carry with one mask add), so
// the counters are derived after the fact from a, b and the result: the true carry into
// limb i is out_i - (a_i + b_i) for add, (a_i - b_i) - out_i for sub. Off the hot path:
// called only when a caller asks for stats.
#include <cuda_runtime.h>

#include <cstdint>

#include "device.cuh"
#include "internal.h"

namespace dotg {

namespace {

template <bool SUB>
__global__ void __launch_bounds__(256) k_addsub_stats(const uint64_t* out, const uint64_t* a, const uint64_t* b,
                                                      size_t m, size_t batch, size_t sp, size_t si, unsigned w,
                                                      unsigned long long* counters) {
    const size_t chunks_per = (m + w - 1) / w;
    const size_t total = chunks_per * batch;
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    unsigned long long fires = 0, chunks = 0;
    for (size_t idx = size_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total; idx += stride) {
        const size_t p = idx / chunks_per, k = idx % chunks_per;
        const size_t i0 = k * w, i1 = (i0 + w < m) ? i0 + w : m;
        uint32_t prev_g = 0, fired = 0;
        for (size_t i = i0; i < i1; ++i) {
            const size_t off = p * sp + i * si;
            uint32_t g, pr;
            const uint64_t s = lane_op<SUB>(a[off], b[off], g, pr);
            // phase-2 carry: the chunk's true carry-in for its first lane, else g_{i-1}
            const uint32_t c2 = i == i0 ? uint32_t(SUB ? (s - out[off]) : (out[off] - s)) & 1u : prev_g;
            fired |= c2 & pr;
            prev_g = g;
        }
        fires += fired;
        ++chunks;
    }
    // one atomic pair per warp
    for (int o = 16; o > 0; o >>= 1) {
        fires += __shfl_down_sync(0xffffffffu, fires, o);
        chunks += __shfl_down_sync(0xffffffffu, chunks, o);
    }
    if ((threadIdx.x & 31u) == 0) {
        if (chunks) atomicAdd(counters, chunks);
        if (fires) atomicAdd(counters + 1, fires);
    }
}

// carry_census(k) (src/oracle.cpp:65-78): over all (x, y) in [0, 2^k)^2, pairs whose sum is
// exactly 2^k - 1 (propagate) and pairs whose sum carries out (>= 2^k). The same
// exhaustive 2^2k enumeration as the reference (the point is to check the closed forms),
// as a grid-stride over pair indices t = x * 2^k + y.
__global__ void __launch_bounds__(256) k_carry_census(unsigned k, unsigned long long* counts) {
    const uint64_t n = uint64_t(1) << k, total = n * n, max = n - 1;
    unsigned long long ms = 0, cs = 0;
    for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
         t += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t s = (t >> k) + (t & max);
        ms += s == max;
        cs += s >= n;
    }
    for (int o = 16; o > 0; o >>= 1) {
        ms += __shfl_down_sync(0xffffffffu, ms, o);
        cs += __shfl_down_sync(0xffffffffu, cs, o);
    }
    if ((threadIdx.x & 31u) == 0) {
        atomicAdd(counts, ms);
        atomicAdd(counts + 1, cs);
    }
}

// Monte-Carlo carry frequency of random 64-bit limb additions (run_stats,
// src/bench.cpp:278-287): sample n = (x_n, y_n) from the counter-based splitmix64 stream
// (the device's workload generator) instead of mt19937_64; the check is statistical.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__global__ void __launch_bounds__(256) k_mc_carry(uint64_t samples, uint64_t seed, unsigned long long* carries) {
    unsigned long long c = 0;
    for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < samples;
         t += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t x = mix64(seed + (2 * t + 1) * 0x9e3779b97f4a7c15ull);
        const uint64_t y = mix64(seed + (2 * t + 2) * 0x9e3779b97f4a7c15ull);
        c += (x + y) < x;
    }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31u) == 0) atomicAdd(carries, c);
}

}  // namespace

cudaError_t launch_carry_census(unsigned k, uint64_t* counts, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(counts, 0, 2 * sizeof(uint64_t), st);
    if (e != cudaSuccess) return e;
    k_carry_census<<<148 * 8, 256, 0, st>>>(k, reinterpret_cast<unsigned long long*>(counts));
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_mc_carry(uint64_t samples, uint64_t seed, uint64_t* carries, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(carries, 0, sizeof(uint64_t), st);
    if (e != cudaSuccess) return e;
    k_mc_carry<<<148 * 8, 256, 0, st>>>(samples, seed, reinterpret_cast<unsigned long long*>(carries));
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_addsub_stats(bool sub, const uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m,
                                size_t batch, int layout, unsigned lanes, uint64_t* counters, cudaStream_t st) {
    if (m == 0 || batch == 0) return cudaSuccess;
    const size_t total = (m + lanes - 1) / lanes * batch;
    size_t blocks = (total + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    const size_t sp = layout == 1 ? 1 : m, si = layout == 1 ? batch : 1;
    unsigned long long* c = reinterpret_cast<unsigned long long*>(counters);
    if (sub) k_addsub_stats<true><<<unsigned(blocks), 256, 0, st>>>(out, a, b, m, batch, sp, si, lanes, c);
    else k_addsub_stats<false><<<unsigned(blocks), 256, 0, st>>>(out, a, b, m, batch, sp, si, lanes, c);
    count_launch();
    return cudaGetLastError();
}

}  // namespace dotg
