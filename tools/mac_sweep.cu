// mac_sweep.cu - how many warps / independent column accumulators does the 96-bit
// column MAC (mad.lo.cc + madc.hi.cc + addc -> IMAD.WIDE.U32 w/ carry + IADD3.X) need
// to reach the IMAD.WIDE pipe limit (32 products/clk/SM)? Sweeps warps per SM and the
// number of independent accumulators C per thread; also the no-carry IMAD.WIDE MAC
// (28-bit digits, 64-bit accumulators) for comparison. Prints JSON lines.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>

template <int C>
__global__ void k_mac96(uint32_t* out, long long* cyc, uint32_t seed, int iters) {
    uint32_t lo[C], mid[C], hi[C];
    uint32_t x[8];
    for (int j = 0; j < 8; ++j) x[j] = seed * (threadIdx.x + 3u) + j * 977u;
    for (int j = 0; j < C; ++j) lo[j] = mid[j] = hi[j] = j;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int j = 0; j < C; ++j)
                asm("mad.lo.cc.u32 %0, %3, %4, %0;\n\tmadc.hi.cc.u32 %1, %3, %4, %1;\n\taddc.u32 %2, %2, 0;"
                    : "+r"(lo[j]), "+r"(mid[j]), "+r"(hi[j])
                    : "r"(x[u]), "r"(x[(u + j + 1) & 7]));
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] ^= lo[u % C];
    }
    long long t1 = clock64();
    uint32_t acc = 0;
    for (int j = 0; j < C; ++j) acc ^= lo[j] ^ mid[j] ^ hi[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int C>
__global__ void k_mac64(uint32_t* out, long long* cyc, uint32_t seed, int iters) {
    uint64_t acc[C];
    uint32_t x[8];
    for (int j = 0; j < 8; ++j) x[j] = (seed * (threadIdx.x + 3u) + j * 977u) & 0x0fffffffu;
    for (int j = 0; j < C; ++j) acc[j] = j;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int j = 0; j < C; ++j)
                asm("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[j]) : "r"(x[u]), "r"(x[(u + j + 1) & 7]));
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = (x[u] ^ uint32_t(acc[u % C])) & 0x0fffffffu;
    }
    long long t1 = clock64();
    uint64_t a = 0;
    for (int j = 0; j < C; ++j) a ^= acc[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = uint32_t(a ^ (a >> 32));
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

using kfn = void (*)(uint32_t*, long long*, uint32_t, int);

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(uint32_t) * sms * 2048);
    cudaMalloc(&cyc, sizeof(long long) * sms * 64);
    struct V { const char* name; int C; kfn f; };
    V vs[] = {{"mac96", 1, k_mac96<1>}, {"mac96", 2, k_mac96<2>}, {"mac96", 4, k_mac96<4>},
              {"mac96", 8, k_mac96<8>}, {"mac96", 16, k_mac96<16>},
              {"mac64", 1, k_mac64<1>}, {"mac64", 4, k_mac64<4>}, {"mac64", 16, k_mac64<16>}};
    const int iters = 2048;
    for (const V& v : vs) {
        for (int wps : {4, 8, 16, 32}) {  // warps per SM (one CTA of 32*wps threads per SM)
            const int threads = 32 * wps;
            v.f<<<sms, threads>>>(out, cyc, 1u, 16);
            cudaDeviceSynchronize();
            v.f<<<sms, threads>>>(out, cyc, 2u, iters);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
            std::vector<long long> h(sms);
            cudaMemcpy(h.data(), cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
            const double c = double(*std::max_element(h.begin(), h.end()));
            const double prods = double(iters) * 8 * v.C * threads;
            printf("{\"kind\": \"%s\", \"C\": %d, \"warps_per_sm\": %d, \"products_per_clk_sm\": %.2f}\n", v.name,
                   v.C, wps, prods / c);
        }
    }
    return 0;
}
