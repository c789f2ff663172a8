// imma_peak.cu - legacy warp-level integer tensor-core (mma.sync IMMA) rate on sm_100a.
//
// Question: can an 8-bit limb-split column multiplication on the tensor pipe beat the
// IMAD.WIDE pipe (32 u32 products/clk/SM)? One u32 x u32 product = 16 u8 x u8 products,
// so mma.sync must sustain > 512 u8 MACs/clk/SM just to break even.
//
// Variants (each warp runs kChains independent accumulator chains):
//   u8   mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32
//   f16  mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 (for scale)
// Output: one JSON object, MACs per SM-clock and per second.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    std::fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

template <int kChains>
__global__ void k_u8(uint32_t* out, long long* cyc, uint32_t seed, int iters) {
    uint32_t a[4], b[2];
    for (int j = 0; j < 4; ++j) a[j] = seed * (threadIdx.x + 3 * j + 1);
    for (int j = 0; j < 2; ++j) b[j] = seed ^ (threadIdx.x * 7 + j);
    int d[kChains][4] = {};
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < kChains; ++j)
            asm volatile(
                "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};"
                : "+r"(d[j][0]), "+r"(d[j][1]), "+r"(d[j][2]), "+r"(d[j][3])
                : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    long long t1 = clock64();
    uint32_t acc = 0;
    for (int j = 0; j < kChains; ++j) acc ^= d[j][0] ^ d[j][1] ^ d[j][2] ^ d[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int kChains>
__global__ void k_f16(uint32_t* out, long long* cyc, uint32_t seed, int iters) {
    uint32_t a[4], b[2];
    for (int j = 0; j < 4; ++j) a[j] = 0x3c003c00u;
    for (int j = 0; j < 2; ++j) b[j] = 0x3c003c00u;
    float d[kChains][4] = {};
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < kChains; ++j)
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};"
                : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
                : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    long long t1 = clock64();
    float acc = 0;
    for (int j = 0; j < kChains; ++j) acc += d[j][0] + d[j][1] + d[j][2] + d[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = __float_as_uint(acc) ^ seed;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <typename K>
int run(const char* name, K kern, double macs_per_mma, int chains, int warps, int sms, uint32_t* out,
        long long* cyc, bool last) {
    const int iters = 4096;
    const int blocks = sms;
    kern<<<blocks, warps * 32>>>(out, cyc, 1u, 16);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<blocks, warps * 32>>>(out, cyc, 1u, iters);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<long long> c(blocks);
    CK(cudaMemcpy(c.data(), cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost));
    const long long cmax = *std::max_element(c.begin(), c.end());
    const double macs_sm = double(warps) * chains * iters * macs_per_mma;
    std::printf("  {\"variant\": \"%s\", \"warps_per_sm\": %d, \"chains\": %d, \"macs_per_clk_sm\": %.1f, "
                "\"tops\": %.1f}%s\n",
                name, warps, chains, macs_sm / double(cmax), 2.0 * macs_sm * blocks / (ms * 1e-3) / 1e12,
                last ? "" : ",");
    return 0;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    uint32_t* out;
    long long* cyc;
    CK(cudaMalloc(&out, size_t(sms) * 1024 * 4));
    CK(cudaMalloc(&cyc, size_t(sms) * 8));
    std::printf("{\"sms\": %d, \"results\": [\n", sms);
    for (int w : {4, 8, 16}) {
        run("u8_m16n8k32", k_u8<4>, 16 * 8 * 32, 4, w, sms, out, cyc, false);
        run("u8_m16n8k32", k_u8<8>, 16 * 8 * 32, 8, w, sms, out, cyc, false);
    }
    for (int w : {4, 8, 16}) run("f16_m16n8k16", k_f16<8>, 16 * 8 * 16, 8, w, sms, out, cyc, w == 16);
    std::printf("]}\n");
    return 0;
}
