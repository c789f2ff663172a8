// step_sweep.cu - throughput of the exact 16x16 column-block MAC step used by
// k_mul_regblk / k_mul_smem (operands in registers), vs warps per SM.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>

constexpr int kK = 16;
__device__ __forceinline__ void mac(uint32_t& lo, uint32_t& mid, uint32_t& hi, uint32_t x, uint32_t y) {
    asm("mad.lo.cc.u32 %0, %3, %4, %0;\n\tmadc.hi.cc.u32 %1, %3, %4, %1;\n\taddc.u32 %2, %2, 0;"
        : "+r"(lo), "+r"(mid), "+r"(hi) : "r"(x), "r"(y));
}

enum { kFull = 0, kLower = 1, kUpper = 2 };
template <int MODE>
__device__ __forceinline__ void mul_step(uint32_t (&acc)[kK][3], const uint32_t (&A)[kK], const uint32_t (&W)[2 * kK]) {
#pragma unroll
    for (int u = 0; u < kK; ++u)
#pragma unroll
        for (int x = 0; x < kK; ++x) {
            if (MODE == kLower && x < u) continue;
            if (MODE == kUpper && x >= u) continue;
            mac(acc[x][0], acc[x][1], acc[x][2], A[u], W[kK + x - u]);
        }
}
__device__ __forceinline__ void add96(uint32_t& lo, uint32_t& mid, uint32_t& hi, uint32_t c0, uint32_t c1, uint32_t c2) {
    asm("add.cc.u32 %0, %0, %3;\n\taddc.cc.u32 %1, %1, %4;\n\taddc.u32 %2, %2, %5;"
        : "+r"(lo), "+r"(mid), "+r"(hi) : "r"(c0), "r"(c1), "r"(c2));
}
// The whole 16-limb pair product of k_mul_regblk on register operands.
template <int TRI>
__global__ void k_pair(uint32_t* out, long long* cyc, uint32_t seed, int iters) {
    constexpr int N = 32, NB = 2, NS = 4;
    uint32_t A[N], B[N];
    for (int i = 0; i < N; ++i) { A[i] = seed * (threadIdx.x + 1u) + i * 7919u; B[i] = seed ^ (threadIdx.x * 31u + i * 104729u); }
    uint32_t sink = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint32_t cr0 = 0, cr1 = 0, cr2 = 0;
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            uint32_t acc[kK][3];
#pragma unroll
            for (int x = 0; x < kK; ++x) acc[x][0] = acc[x][1] = acc[x][2] = 0;
#pragma unroll
            for (int I = 0; I < NB; ++I) {
                const int d = s - I;
                if (d < 0 || d > NB) continue;
                uint32_t Ab[kK], W[2 * kK];
#pragma unroll
                for (int u = 0; u < kK; ++u) Ab[u] = A[I * kK + u];
#pragma unroll
                for (int e = 0; e < 2 * kK; ++e) {
                    const int j = (d - 1) * kK + e;
                    W[e] = (j >= 0 && j < N) ? B[j < 0 ? 0 : (j >= N ? N - 1 : j)] : 0u;
                }
                if (TRI == 0) mul_step<kFull>(acc, Ab, W);
                else if (d == 0) mul_step<kLower>(acc, Ab, W);
                else if (d == NB) mul_step<kUpper>(acc, Ab, W);
                else mul_step<kFull>(acc, Ab, W);
            }
#pragma unroll
            for (int x = 0; x < kK; ++x) {
                add96(acc[x][0], acc[x][1], acc[x][2], cr0, cr1, cr2);
                sink ^= acc[x][0];
                cr0 = acc[x][1]; cr1 = acc[x][2]; cr2 = 0;
            }
        }
        A[it & 31] ^= sink;
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = sink;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int ORDER>
__global__ void k_step(uint32_t* out, long long* cyc, uint32_t seed, int iters) {
    uint32_t A[kK], W[2 * kK];
    for (int i = 0; i < kK; ++i) A[i] = seed * (threadIdx.x + 1u) + i * 7919u;
    for (int i = 0; i < 2 * kK; ++i) W[i] = seed ^ (threadIdx.x * 31u + i * 104729u);
    uint32_t acc[kK][3];
    for (int x = 0; x < kK; ++x) acc[x][0] = acc[x][1] = acc[x][2] = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (ORDER == 0) {
#pragma unroll
            for (int u = 0; u < kK; ++u)
#pragma unroll
                for (int x = 0; x < kK; ++x) mac(acc[x][0], acc[x][1], acc[x][2], A[u], W[kK + x - u]);
        } else {
#pragma unroll
            for (int x = 0; x < kK; ++x)
#pragma unroll
                for (int u = 0; u < kK; ++u) mac(acc[x][0], acc[x][1], acc[x][2], A[u], W[kK + x - u]);
        }
#pragma unroll
        for (int i = 0; i < kK; ++i) A[i] ^= acc[i][0];
    }
    long long t1 = clock64();
    uint32_t r = 0;
    for (int x = 0; x < kK; ++x) r ^= acc[x][0] ^ acc[x][1] ^ acc[x][2];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* out; long long* cyc;
    cudaMalloc(&out, sizeof(uint32_t) * sms * 4096);
    cudaMalloc(&cyc, sizeof(long long) * sms * 64);
    const int iters = 512;
    for (int order = 0; order < 2; ++order)
        for (int wps : {2, 4, 6, 8, 12, 16}) {
            const int threads = 32 * wps;
            auto f = order == 0 ? k_step<0> : k_step<1>;
            f<<<sms, threads>>>(out, cyc, 1u, 4);
            cudaError_t e = cudaDeviceSynchronize();
            f<<<sms, threads>>>(out, cyc, 2u, iters);
            e = cudaGetLastError();
            if (e == cudaSuccess) e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("{\"order\": %d, \"warps\": %d, \"err\": \"%s\"}\n", order, wps, cudaGetErrorString(e)); continue; }
            std::vector<long long> h(sms);
            cudaMemcpy(h.data(), cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
            const double c = double(*std::max_element(h.begin(), h.end()));
            printf("{\"order\": %d, \"warps_per_sm\": %d, \"products_per_clk_sm\": %.2f}\n", order, wps,
                   double(iters) * 256 * threads / c);
        }
    for (int tri = 0; tri < 2; ++tri)
        for (int wps : {4, 8, 12, 16, 20}) {
            const int threads = 32 * wps;
            auto f = tri == 0 ? k_pair<0> : k_pair<1>;
            f<<<sms, threads>>>(out, cyc, 1u, 2);
            cudaError_t e = cudaDeviceSynchronize();
            f<<<sms, threads>>>(out, cyc, 2u, 256);
            e = cudaGetLastError();
            if (e == cudaSuccess) e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("{\"pair_tri\": %d, \"warps\": %d, \"err\": \"%s\"}\n", tri, wps, cudaGetErrorString(e)); continue; }
            std::vector<long long> h(sms);
            cudaMemcpy(h.data(), cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
            const double c = double(*std::max_element(h.begin(), h.end()));
            // tri=0 issues 6 full steps (1536 MACs, zero-padded triangles), tri=1 exactly 1024
            printf("{\"pair_tri\": %d, \"warps_per_sm\": %d, \"macs_per_clk_sm\": %.2f}\n", tri, wps,
                   256.0 * (tri ? 1024 : 1536) * threads / c);
        }
    return 0;
}
