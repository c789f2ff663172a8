// compare.cu - batched unsigned comparison, the reference's compare (include/dot/limbs.hpp:84,
// src/limbs.cpp:46-53: -1 / 0 / +1, high zero limbs ignored) for equal-length pairs, as the
// config generators use it for the sub a >= b swap. With equal lengths the significant-limb
// rule reduces to the first difference from the top.
//
// Row-major: a team of T = min(32, 2^ceil(log2 m)) lanes per pair, lanes strided over the
// pair's limbs (coalesced), each lane's highest differing limb, a shuffle max over the team,
// the sign from that limb. Interleaved: one thread per pair scanning from the top (the
// threads of a warp read consecutive pairs of each limb row).
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"

namespace dotg {

namespace {

template <int T>
__global__ void __launch_bounds__(256) k_compare_rows(int32_t* out, const uint64_t* __restrict__ a,
                                                      const uint64_t* __restrict__ b, size_t m, size_t batch) {
    const size_t gt = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t p = gt / T;
    const unsigned r = unsigned(threadIdx.x) % T;
    const bool ok = p < batch;
    const uint64_t* pa = a + (ok ? p : 0) * m;
    const uint64_t* pb = b + (ok ? p : 0) * m;
    unsigned top = 0;  // 1 + highest differing limb seen by this lane
    if (ok)
        for (size_t i = r; i < m; i += T)
            if (__ldg(pa + i) != __ldg(pb + i)) top = unsigned(i) + 1;
#pragma unroll
    for (int s = T / 2; s > 0; s >>= 1) {
        const unsigned o = __shfl_xor_sync(0xffffffffu, top, s);
        top = o > top ? o : top;
    }
    if (ok && r == 0) {
        int v = 0;
        if (top != 0) v = __ldg(pa + top - 1) < __ldg(pb + top - 1) ? -1 : 1;
        out[p] = v;
    }
}

__global__ void __launch_bounds__(256) k_compare_interleaved(int32_t* out, const uint64_t* __restrict__ a,
                                                             const uint64_t* __restrict__ b, size_t m,
                                                             size_t batch) {
    const size_t p = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= batch) return;
    int v = 0;
    for (size_t i = m; i-- > 0;) {
        const uint64_t x = __ldg(a + i * batch + p), y = __ldg(b + i * batch + p);
        if (x != y) {
            v = x < y ? -1 : 1;
            break;
        }
    }
    out[p] = v;
}

template <int T>
cudaError_t run_rows(int32_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch, cudaStream_t st) {
    const size_t threads = batch * T;
    k_compare_rows<T><<<unsigned((threads + 255) / 256), 256, 0, st>>>(out, a, b, m, batch);
    count_launch();
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_compare_batch(int32_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                                 int layout, cudaStream_t st) {
    if (batch == 0) return cudaSuccess;
    if (m == 0) return cudaMemsetAsync(out, 0, batch * sizeof(int32_t), st);
    if (layout == 1) {
        k_compare_interleaved<<<unsigned((batch + 255) / 256), 256, 0, st>>>(out, a, b, m, batch);
        count_launch();
        return cudaGetLastError();
    }
    if (m <= 1) return run_rows<1>(out, a, b, m, batch, st);
    if (m <= 2) return run_rows<2>(out, a, b, m, batch, st);
    if (m <= 4) return run_rows<4>(out, a, b, m, batch, st);
    if (m <= 8) return run_rows<8>(out, a, b, m, batch, st);
    if (m <= 16) return run_rows<16>(out, a, b, m, batch, st);
    return run_rows<32>(out, a, b, m, batch, st);
}

}  // namespace dotg
