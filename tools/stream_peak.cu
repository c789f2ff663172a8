// stream_peak.cu - what HBM bandwidth does a plain streaming kernel reach on this B200 for
// the byte mixes of the add/sub configs? (MEASURED_PEAKS.json's hbm_gbs is a 1:1 copy.)
//   copy   out[i] = a[i]            (read 1 : write 1)
//   add    out[i] = a[i] + b[i]     (read 2 : write 1, the add/sub mix, no carries)
//   read   sum of a[i] and b[i]     (read only)
// 256-bit loads/stores, grid-stride persistent kernel, 537 MB of inputs (> L2), events,
// best of 20 launches after 5 warm-ups. Output: one JSON object.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <algorithm>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    std::fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

struct V4 { uint64_t x, y, z, w; };

__device__ __forceinline__ V4 ld4(const uint64_t* p) {
    V4 v;
    asm volatile("ld.global.L1::no_allocate.L2::evict_first.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(v.x), "=l"(v.y), "=l"(v.z), "=l"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ void st4(uint64_t* p, V4 v) {
    asm volatile("st.global.L1::no_allocate.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(v.x), "l"(v.y), "l"(v.z),
                 "l"(v.w) : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(256) k_stream(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t n4,
                                                uint64_t* sink) {
    uint64_t acc = 0;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += size_t(gridDim.x) * blockDim.x) {
        V4 x = ld4(a + 4 * i);
        if (MODE == 0) {
            st4(out + 4 * i, x);
        } else {
            V4 y = ld4(b + 4 * i);
            if (MODE == 1) {
                st4(out + 4 * i, V4{x.x + y.x, x.y + y.y, x.z + y.z, x.w + y.w});
            } else {
                acc += x.x ^ y.x ^ x.y ^ y.y ^ x.z ^ y.z ^ x.w ^ y.w;
            }
        }
    }
    if (MODE == 2 && acc == 0x123456789ull) sink[0] = acc;
}

template <int MODE>
int run(const char* name, uint64_t* out, const uint64_t* a, const uint64_t* b, size_t n, uint64_t* sink, int sms,
        bool last) {
    const size_t n4 = n / 4;
    int per = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_stream<MODE>, 256, 0));
    const int grid = sms * per;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int it = 0; it < 25; ++it) {
        cudaEventRecord(e0);
        k_stream<MODE><<<grid, 256>>>(out, a, b, n4, sink);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it >= 5) best = std::min(best, ms);
    }
    const double bytes = double(n) * 8 * (MODE == 0 ? 2 : (MODE == 1 ? 3 : 2));
    std::printf("  \"%s\": {\"GBps\": %.1f, \"bytes\": %.0f, \"us\": %.1f}%s\n", name, bytes / (best * 1e-3) / 1e9,
                bytes, best * 1e3, last ? "" : ",");
    return 0;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t n = size_t(1) << 25;  // u64 per operand: 256 MiB each, 537 MB for a + b
    uint64_t *a, *b, *out, *sink;
    CK(cudaMalloc(&a, n * 8));
    CK(cudaMalloc(&b, n * 8));
    CK(cudaMalloc(&out, n * 8));
    CK(cudaMalloc(&sink, 8));
    CK(cudaMemset(a, 1, n * 8));
    CK(cudaMemset(b, 2, n * 8));
    std::printf("{\n");
    run<0>("copy_1r1w", out, a, b, n, sink, sms, false);
    run<1>("add_2r1w", out, a, b, n, sink, sms, false);
    run<2>("read_2r", out, a, b, n, sink, sms, true);
    std::printf("}\n");
    return 0;
}
