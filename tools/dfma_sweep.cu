// dfma_sweep.cu - throughput of an exact 52x52 -> 104-bit product on the FP64 pipe:
//   h = fma.rz(x, y, 2^104)            (bits(h) = bits(2^104) + hi)
//   c = (2^104 + 2^52) - h             (exact)
//   l = fma.rn(x, y, c)                (bits(l) = bits(2^52) + lo, lo = x*y mod 2^52)
// with the two bit patterns accumulated into 64-bit integer column accumulators.
// Reports exact products per clk per SM vs warps per SM and checks exactness.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ void prod52(double x, double y, uint64_t& acc_lo, uint64_t& acc_hi) {
    const double C104 = 20282409603651670423947251286016.0;               // 2^104
    const double C104p52 = 20282409603651670423947251286016.0 + 4503599627370496.0;  // 2^104 + 2^52
    double h, c, l;
    asm("fma.rz.f64 %0, %1, %2, %3;" : "=d"(h) : "d"(x), "d"(y), "d"(C104));
    asm("sub.rn.f64 %0, %1, %2;" : "=d"(c) : "d"(C104p52), "d"(h));
    asm("fma.rn.f64 %0, %1, %2, %3;" : "=d"(l) : "d"(x), "d"(y), "d"(c));
    acc_lo += uint64_t(__double_as_longlong(l));
    acc_hi += uint64_t(__double_as_longlong(h));
}

template <int C>
__global__ void k_dfma(uint64_t* out, long long* cyc, uint64_t seed, int iters) {
    double x[8], y[8];
    for (int j = 0; j < 8; ++j) {
        const uint64_t v = (seed * (threadIdx.x + 1 + j) * 0x9E3779B97F4A7C15ull) >> 12;  // 52-bit
        x[j] = double(v);
        y[j] = double((v * 0xBF58476D1CE4E5B9ull) >> 12);
    }
    uint64_t lo[C], hi[C];
    for (int j = 0; j < C; ++j) lo[j] = hi[j] = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int j = 0; j < C; ++j) prod52(x[u], y[(u + j) & 7], lo[j], hi[j]);
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = __longlong_as_double(__double_as_longlong(x[u]) ^ (lo[u % C] & 1));
    }
    long long t1 = clock64();
    uint64_t r = 0;
    for (int j = 0; j < C; ++j) r ^= lo[j] ^ hi[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_check(uint64_t* bad, int n) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    uint64_t a = (0x9E3779B97F4A7C15ull * (t + 1)) >> 12, b = (0xBF58476D1CE4E5B9ull * (t + 7)) >> 12;
    if (t % 4 == 0) a = (1ull << 52) - 1;
    if (t % 8 == 0) b = (1ull << 52) - 1;
    if (t % 16 == 1) b = 0;
    uint64_t lo = 0, hi = 0;
    prod52(double(a), double(b), lo, hi);
    const uint64_t rlo = lo - 0x4330000000000000ull, rhi = hi - 0x4670000000000000ull;
    const unsigned __int128 p = (unsigned __int128)a * b;
    if (rlo != uint64_t(p & ((1ull << 52) - 1)) || rhi != uint64_t(p >> 52)) atomicAdd((unsigned long long*)bad, 1ull);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint64_t* out;
    long long* cyc;
    uint64_t* bad;
    cudaMalloc(&out, sizeof(uint64_t) * sms * 1024);
    cudaMalloc(&cyc, sizeof(long long) * sms);
    cudaMalloc(&bad, 8);
    cudaMemset(bad, 0, 8);
    k_check<<<4096, 256>>>(bad, 4096 * 256);
    uint64_t hbad = 0;
    cudaMemcpy(&hbad, bad, 8, cudaMemcpyDeviceToHost);
    printf("{\"exactness_failures\": %llu, \"checked\": %d}\n", (unsigned long long)hbad, 4096 * 256);
    const int iters = 512;
    for (int C : {4, 8}) {
        for (int wps : {4, 8, 12, 16, 24}) {
            const int threads = 32 * wps;
            auto f = C == 4 ? k_dfma<4> : k_dfma<8>;
            f<<<sms, threads>>>(out, cyc, 3, 4);
            f<<<sms, threads>>>(out, cyc, 5, iters);
            cudaError_t e = cudaGetLastError();
            if (e == cudaSuccess) e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("{\"C\": %d, \"warps\": %d, \"err\": \"%s\"}\n", C, wps, cudaGetErrorString(e)); continue; }
            std::vector<long long> h(sms);
            cudaMemcpy(h.data(), cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
            const double c = double(*std::max_element(h.begin(), h.end()));
            printf("{\"C\": %d, \"warps_per_sm\": %d, \"products52_per_clk_sm\": %.2f}\n", C, wps,
                   double(iters) * 8 * C * threads / c);
        }
    }
    return 0;
}
