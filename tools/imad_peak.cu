// imad_peak.cu - integer-multiply issue-rate microbenchmark for the mul roofline.
//
// BASELINE.md §2 asks for the IMAD roofline denominator to be measured on the box:
// roofline = SMs x IMAD issues/clk/SM x measured SM clock. This tool runs one
// single-wave grid (every CTA resident at once) of independent instruction chains
// per variant and reports, per variant, lane-ops per SM-clock (from clock64 inside
// the kernel) and lane-ops per second (from CUDA events).
//
// Variants (PTX -> SASS checked with cuobjdump):
//   imad      mad.lo.u32                    -> IMAD
//   imad_wide mad.wide.u32                  -> IMAD.WIDE.U32
//   imad_hi   mad.hi.u32                    -> IMAD.HI.U32
//   cc_chain  mad.lo.cc / madc.hi.cc / addc  (one 32x32->64 product into a 96-bit
//             column accumulator; counted as 1 product = 3 instructions)
//   dfma      fma.rn.f64                    -> DFMA
//   ffma      fma.rn.f32                    -> FFMA (sanity reference)
//
// Output: one JSON object on stdout.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    std::fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

constexpr int kChains = 8;

__global__ void k_imad(uint32_t* out, long long* cyc, uint32_t seed, int iters) {
    uint32_t x[kChains];
    const uint32_t y = seed ^ threadIdx.x, z = seed * 3u + 1u;
    for (int j = 0; j < kChains; ++j) x[j] = seed + threadIdx.x * 7u + j;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int j = 0; j < kChains; ++j)
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[j]) : "r"(y), "r"(z));
    }
    long long t1 = clock64();
    uint32_t acc = 0;
    for (int j = 0; j < kChains; ++j) acc ^= x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_imad_wide(uint32_t* out, long long* cyc, uint32_t seed, int iters) {
    uint64_t x[kChains];
    const uint32_t y = seed ^ threadIdx.x;
    for (int j = 0; j < kChains; ++j) x[j] = seed + threadIdx.x * 7u + j;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int j = 0; j < kChains; ++j)
                asm volatile("{\n\t.reg .u32 t;\n\tcvt.u32.u64 t, %0;\n\tmad.wide.u32 %0, t, %1, %0;\n\t}"
                             : "+l"(x[j]) : "r"(y | 1u));
    }
    long long t1 = clock64();
    uint64_t acc = 0;
    for (int j = 0; j < kChains; ++j) acc ^= x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = uint32_t(acc ^ (acc >> 32));
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_imad_hi(uint32_t* out, long long* cyc, uint32_t seed, int iters) {
    uint32_t x[kChains];
    const uint32_t y = seed ^ threadIdx.x, z = seed * 3u + 1u;
    for (int j = 0; j < kChains; ++j) x[j] = seed + threadIdx.x * 7u + j;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int j = 0; j < kChains; ++j)
                asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(x[j]) : "r"(y), "r"(z));
    }
    long long t1 = clock64();
    uint32_t acc = 0;
    for (int j = 0; j < kChains; ++j) acc ^= x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// One product a*b (32x32->64) accumulated into a 96-bit column (lo, mid, hi).
__global__ void k_cc_chain(uint32_t* out, long long* cyc, uint32_t seed, int iters) {
    constexpr int C = 4;  // independent columns
    uint32_t lo[C], mid[C], hi[C];
    uint32_t a = seed ^ threadIdx.x, b = seed * 3u + 1u;
    for (int j = 0; j < C; ++j) { lo[j] = j; mid[j] = 0; hi[j] = 0; }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 32; ++u)
#pragma unroll
            for (int j = 0; j < C; ++j)
                asm volatile(
                    "mad.lo.cc.u32 %0, %3, %4, %0;\n\t"
                    "madc.hi.cc.u32 %1, %3, %4, %1;\n\t"
                    "addc.u32 %2, %2, 0;"
                    : "+r"(lo[j]), "+r"(mid[j]), "+r"(hi[j]) : "r"(a + j), "r"(b));
    }
    long long t1 = clock64();
    uint32_t acc = 0;
    for (int j = 0; j < C; ++j) acc ^= lo[j] ^ mid[j] ^ hi[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_dfma(uint32_t* out, long long* cyc, uint32_t seed, int iters) {
    double x[kChains];
    const double y = 1.0000001 + seed * 1e-12, z = 1e-9;
    for (int j = 0; j < kChains; ++j) x[j] = 1.0 + threadIdx.x * 1e-6 + j;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int j = 0; j < kChains; ++j)
                asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x[j]) : "d"(y), "d"(z));
    }
    long long t1 = clock64();
    double acc = 0;
    for (int j = 0; j < kChains; ++j) acc += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = uint32_t(acc);
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ffma(uint32_t* out, long long* cyc, uint32_t seed, int iters) {
    float x[kChains];
    const float y = 1.0001f + seed * 1e-9f, z = 1e-7f;
    for (int j = 0; j < kChains; ++j) x[j] = 1.0f + threadIdx.x * 1e-6f + j;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int j = 0; j < kChains; ++j)
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[j]) : "f"(y), "f"(z));
    }
    long long t1 = clock64();
    float acc = 0;
    for (int j = 0; j < kChains; ++j) acc += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = uint32_t(acc);
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

using kfn = void (*)(uint32_t*, long long*, uint32_t, int);

int main() {
    int dev = 0, sms = 0, clk_khz = 0;
    CK(cudaSetDevice(dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
    const int threads = 512, blocks_per_sm = 4, blocks = sms * blocks_per_sm;
    const int iters = 4096;
    uint32_t* out; long long* cyc;
    CK(cudaMalloc(&out, sizeof(uint32_t) * blocks * threads));
    CK(cudaMalloc(&cyc, sizeof(long long) * blocks));
    struct V { const char* name; kfn f; double ops_per_inner; };
    // ops_per_inner: lane-ops of the named kind per (it) iteration per thread.
    V vs[] = {
        {"imad", k_imad, 16.0 * kChains},
        {"imad_wide", k_imad_wide, 16.0 * kChains},
        {"imad_hi", k_imad_hi, 16.0 * kChains},
        {"cc_chain_products", k_cc_chain, 32.0 * 4},
        {"dfma", k_dfma, 16.0 * kChains},
        {"ffma", k_ffma, 16.0 * kChains},
    };
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    std::printf("{\"sms\": %d, \"clock_rate_khz\": %d, \"threads_per_sm\": %d, \"variants\": {", sms,
                clk_khz, threads * blocks_per_sm);
    bool first = true;
    for (const V& v : vs) {
        v.f<<<blocks, threads>>>(out, cyc, 1u, 64);  // warm-up
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        float best_ms = 1e30f; double best_cyc = 0;
        for (int rep = 0; rep < 3; ++rep) {
            CK(cudaEventRecord(e0));
            v.f<<<blocks, threads>>>(out, cyc, 1u + rep, iters);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms = 0; CK(cudaEventElapsedTime(&ms, e0, e1));
            std::vector<long long> h(blocks);
            CK(cudaMemcpy(h.data(), cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost));
            const double maxc = double(*std::max_element(h.begin(), h.end()));
            if (ms < best_ms) { best_ms = ms; best_cyc = maxc; }
        }
        const double lane_ops = v.ops_per_inner * iters * double(threads) * blocks;
        const double per_clk_sm = lane_ops / sms / best_cyc;
        const double per_s = lane_ops / (best_ms * 1e-3);
        const double eff_mhz = best_cyc / (best_ms * 1e-3) / 1e6;
        std::printf("%s\"%s\": {\"lane_ops_per_clk_per_sm\": %.2f, \"lane_ops_per_s\": %.4e, \"ms\": %.3f, \"eff_sm_mhz\": %.0f}",
                    first ? "" : ", ", v.name, per_clk_sm, per_s, best_ms, eff_mhz);
        first = false;
    }
    std::printf("}}\n");
    return 0;
}
