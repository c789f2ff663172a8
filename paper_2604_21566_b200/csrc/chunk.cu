// chunk.cu - the reference's chunk-level operations add_w_limbs / sub_w_limbs
// (include/dot/addsub.hpp:78-89, src/addsub.cpp:172-190), batched: chunk p is w limbs
// (1 <= w <= 8) at a + p*w, b + p*w with its own carry-in, and yields w sums, the chunk's
// carry-out and whether Phase 4 fired (addsub.cpp:55-79: some lane wrapped when its Phase-3
// carry was added, i.e. it received c_i = 1 and propagates).
//
// One thread per chunk: the w lanes' generate / propagate bits form two w-bit masks and one
// integer add (((G << 1) | cin) + P) ^ P settles every carry of the chunk - the reference's
// own Phase-4 formula applied to all lanes at once; bit w of the sum is the carry-out.
// A test/API surface (the reference's tests drive it); the hot path is addsub_batch.cu.
#include <cuda_runtime.h>

#include <cstdint>

#include "device.cuh"
#include "internal.h"

namespace dotg {

namespace {

template <bool SUB>
__global__ void __launch_bounds__(256) k_chunk_batch(uint64_t* sums, uint32_t* carry_out, uint32_t* fired,
                                                     const uint64_t* a, const uint64_t* b,
                                                     const uint32_t* carry_in, unsigned w, size_t batch) {
    const size_t p = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= batch) return;
    const uint32_t cin = carry_in != nullptr ? carry_in[p] : 0u;
    if (cin > 1u) {  // the reference throws (addsub.cpp:177); the batch form flags the chunk
        carry_out[p] = 0xffffffffu;
        if (fired != nullptr) fired[p] = 0;
        return;
    }
    uint64_t s[8];
    uint32_t G = 0, P = 0;
#pragma unroll
    for (unsigned i = 0; i < 8; ++i) {
        if (i < w) {
            uint32_t g, pr;
            s[i] = lane_op<SUB>(a[p * w + i], b[p * w + i], g, pr);
            G |= g << i;
            P |= pr << i;
        }
    }
    const uint32_t c2 = (G << 1) | cin;  // Phase-2 carries, aligned to the lanes they feed
    const uint32_t settled = c2 + P;
    const uint32_t c = (settled ^ P) & ((1u << w) - 1u);
#pragma unroll
    for (unsigned i = 0; i < 8; ++i)
        if (i < w) sums[p * w + i] = SUB ? s[i] - ((c >> i) & 1u) : s[i] + ((c >> i) & 1u);
    carry_out[p] = (settled >> w) & 1u;
    if (fired != nullptr) fired[p] = (c2 & P & ((1u << w) - 1u)) != 0u;
}

}  // namespace

cudaError_t launch_chunk_batch(bool sub, uint64_t* sums, uint32_t* carry_out, uint32_t* fired, const uint64_t* a,
                               const uint64_t* b, const uint32_t* carry_in, unsigned w, size_t batch,
                               cudaStream_t st) {
    if (batch == 0) return cudaSuccess;
    const unsigned blocks = unsigned((batch + 255) / 256);
    if (sub) k_chunk_batch<true><<<blocks, 256, 0, st>>>(sums, carry_out, fired, a, b, carry_in, w, batch);
    else k_chunk_batch<false><<<blocks, 256, 0, st>>>(sums, carry_out, fired, a, b, carry_in, w, batch);
    count_launch();
    return cudaGetLastError();
}

}  // namespace dotg
