// util.cu - reproducible input generation on the device (workload setup, not the hot
// path): out[i] = splitmix64 output for counter offset + i + 1, identical to the host
// generator oracle/dot_oracle.c:dotor_fill_splitmix64 so multi-GiB config-5 inputs can be
// made in HBM and re-derived on the host for the oracle.
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"

namespace dotg {

__device__ __forceinline__ uint64_t splitmix64_at(uint64_t seed, uint64_t k) {
    uint64_t z = seed + k * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void k_fill_splitmix64(uint64_t* out, size_t n, uint64_t seed, uint64_t offset) {
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = splitmix64_at(seed, offset + i + 1);
}

cudaError_t launch_fill_splitmix64(uint64_t* out, size_t n, uint64_t seed, uint64_t offset, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    size_t blocks = (n + 255) / 256;
    const size_t cap = size_t(sms) * 16;
    if (blocks > cap) blocks = cap;
    k_fill_splitmix64<<<unsigned(blocks), 256, 0, st>>>(out, n, seed, offset);
    return cudaGetLastError();
}

}  // namespace dotg
