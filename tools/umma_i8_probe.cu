// umma_i8_probe.cu - what the 5th-generation tensor core (tcgen05.mma kind::i8, TMEM
// accumulators) delivers for the SHAPES a batched big-integer column product can use.
//
// Question: is a tcgen05 variant of the radix-2^8 column multiply
// (k_mul_imma, legacy mma.sync m16n8k32) worth building? One 4096-bit pair is a
// 512 x 512-byte Toeplitz product: 2^18 byte-MACs, and both operands belong to that pair
// only - no operand is shared across pairs, so an MMA's N (and its reuse of A) is bounded
// by one pair's block count (N <= 16-32 for m = 64). This probe measures, per SM:
//   * clk per tcgen05.mma (M = 128, K = 32 bytes) for N = 16 ... 256, A and B from shared
//     memory (SS) and A from TMEM (TS), one CTA per SM issuing back to back into one
//     TMEM accumulator, with NA distinct A tiles cycled (NA = 1: same A every MMA);
//   * tcgen05.ld.32x32b.x16 throughput (the epilogue's TMEM reads);
// and checks every configuration's accumulator against a host computation.
// Output: one JSON line per configuration.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            std::fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            std::exit(1);                                                                       \
        }                                                                                       \
    } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

// K-major, no-swizzle canonical layout ((8,m),2):((16 B, SBO),LBO): core matrix = 8 rows x
// 16 bytes contiguous; here chunk kappa of rows [8g, 8g+8) sits at (2g + kappa) * 128.
__host__ __device__ constexpr uint32_t tile_off(int r, int k) { return ((r / 8) * 2 + k / 16) * 128 + (r % 8) * 16 + k % 16; }

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
           (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46);  // version 1, no swizzle
}

__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {  // u8 x u8 -> s32, both K-major
    return (2u << 4) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

template <int N, bool TS, int NA, int NCH>
__global__ void __launch_bounds__(128, 1) k_umma(const uint8_t* gA, const uint8_t* gB, int32_t* gD, long long* cyc,
                                                 long long* ldcyc, int iters) {
    constexpr int M = 128;
    constexpr int ATILE = M * 32;
    constexpr int DCOLS = N * NCH;  // NCH independent accumulators, MMA i into accumulator i % NCH
    constexpr int COLS = (DCOLS + (TS ? 8 : 0)) <= 32 ? 32 : (DCOLS + (TS ? 8 : 0)) <= 64 ? 64 : (DCOLS + (TS ? 8 : 0)) <= 128 ? 128 : (DCOLS + (TS ? 8 : 0)) <= 256 ? 256 : 512;
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* sA = sm;                 // NA tiles
    uint8_t* sB = sm + NA * ATILE;    // N x 32
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < NA * ATILE; i += blockDim.x) {
        const int t = i / ATILE, e = i % ATILE, r = e / 32, k = e % 32;
        sA[t * ATILE + tile_off(r, k)] = gA[e] + uint8_t(t);  // tile t = A + t
    }
    for (int i = tid; i < N * 32; i += blockDim.x) sB[tile_off(i / 32, i % 32)] = gB[i];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)),
                     "r"(COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tbase;
    const uint32_t dt = tm, at = tm + DCOLS;
    const uint32_t id = idesc_i8(M, N);
    const uint64_t bd = sdesc(smem_u32(sB), 128, 256);
    if (tid == 0) {
        if (TS) {
            const uint64_t ad = sdesc(smem_u32(sA), 128, 256);
            asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(at), "l"(ad) : "memory");
        }
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint32_t acc = i >= NCH;
            const uint32_t dti = dt + uint32_t((i % NCH) * N);
            if (TS) {
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(dti),
                    "r"(at), "l"(bd), "r"(id), "r"(acc)
                    : "memory");
            } else {
                const uint64_t ad = sdesc(smem_u32(sA + (i % NA) * ATILE), 128, 256);
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(dti),
                    "l"(ad), "l"(bd), "r"(id), "r"(acc)
                    : "memory");
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&bar))
                     : "memory");
        asm volatile(
            "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(
                smem_u32(&bar))
            : "memory");
        long long t1 = clock64();
        cyc[blockIdx.x] = t1 - t0;
    }
    __syncthreads();
    asm volatile(
        "{\n\t.reg .pred p;\nW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W2;\n}" ::"r"(
            smem_u32(&bar))
        : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // epilogue: lane r of warp w reads TMEM lane 32w + r, 16 columns at a time
    uint32_t acc = 0;
    long long l0 = clock64();
    for (int c0 = 0; c0 < DCOLS; c0 += 16) {
        uint32_t v[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(dt + (uint32_t(warp * 32) << 16) + uint32_t(c0)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (blockIdx.x == 0 && c0 < N)
            for (int j = 0; j < 16 && c0 + j < N; ++j) gD[(warp * 32 + (tid & 31)) * N + c0 + j] = int32_t(v[j]);
        acc ^= v[0];
    }
    // TMEM read throughput: 64 more x16 loads per warp, all 4 warps at once
    __syncthreads();
    long long r0 = clock64();
#pragma unroll 1
    for (int rep = 0; rep < 64; ++rep) {
        uint32_t v[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(dt + (uint32_t(warp * 32) << 16) + uint32_t((rep * 16) % DCOLS)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int j = 0; j < 16; ++j) acc += v[j];
    }
    __syncthreads();
    long long r1 = clock64();
    if (tid == 0) ldcyc[blockIdx.x] = r1 - r0;
    if (acc == 0x12345678u) gD[0] = 0;  // keep the loads
    (void)l0;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(COLS) : "memory");
}

template <int N, bool TS, int NA, int NCH = 1>
void run(int sms, int clk_mhz, int per_sm = 1) {
    constexpr int M = 128;
    const int iters = 2048;
    std::vector<uint8_t> A(M * 32), B(N * 32);
    uint32_t s = 12345u + N * 7 + TS * 3 + NA;
    for (auto& x : A) x = uint8_t((s = s * 1664525u + 1013904223u) >> 24) & 0x0F;
    for (auto& x : B) x = uint8_t((s = s * 1664525u + 1013904223u) >> 24) & 0x0F;
    uint8_t *dA, *dB;
    int32_t* dD;
    long long *dc, *dl;
    CK(cudaMalloc(&dA, A.size()));
    CK(cudaMalloc(&dB, B.size()));
    CK(cudaMalloc(&dD, sizeof(int32_t) * M * N));
    CK(cudaMalloc(&dc, sizeof(long long) * sms * per_sm));
    CK(cudaMalloc(&dl, sizeof(long long) * sms * per_sm));
    CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
    const int smem = NA * M * 32 + N * 32;
    CK(cudaFuncSetAttribute(k_umma<N, TS, NA, NCH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_umma<N, TS, NA, NCH><<<sms * per_sm, 128, smem>>>(dA, dB, dD, dc, dl, iters);  // warm
    CK(cudaDeviceSynchronize());
    k_umma<N, TS, NA, NCH><<<sms * per_sm, 128, smem>>>(dA, dB, dD, dc, dl, iters);
    CK(cudaDeviceSynchronize());
    std::vector<int32_t> D(M * N);
    const int nct = sms * per_sm;
    std::vector<long long> c(nct), l(nct);
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(c.data(), dc, nct * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(l.data(), dl, nct * 8, cudaMemcpyDeviceToHost));
    long long bad = 0;
    for (int r = 0; r < M; ++r)
        for (int n = 0; n < N; ++n) {
            long long want = 0;
            const int na = TS ? 1 : NA;  // accumulator 0 takes MMAs i = 0, NCH, ...: A tile i % na
            for (int i = 0; i < iters; i += NCH) {
                const int t = i % na;
                int dot = 0;
                for (int k = 0; k < 32; ++k) dot += int(uint8_t(A[r * 32 + k] + t)) * int(B[n * 32 + k]);
                want += dot;
                if (na == 1) {
                    want = (long long)dot * (iters / NCH);
                    break;
                }
            }
            if (D[r * N + n] != int32_t(want)) ++bad;
        }
    double cm = 0, lm = 0;
    for (int i = 0; i < nct; ++i) cm += c[i], lm += l[i];
    cm /= nct;
    lm /= nct;
    const double clk_per_mma = cm / iters;
    const double macs = double(M) * N * 32;
    // TMEM read: 4 warps x 64 loads x 32 lanes x 16 words x 4 B
    const double ld_bytes = 4.0 * 64 * 32 * 16 * 4;
    std::printf(
        "{\"M\": %d, \"N\": %d, \"K\": 32, \"mode\": \"%s\", \"distinct_A_tiles\": %d, \"accumulators\": %d, \"ctas_per_sm\": %d, \"clk_per_mma\": %.2f, "
        "\"macs_per_clk_sm\": %.1f, \"smem_bytes_per_mma\": %d, \"smem_B_per_clk\": %.1f, "
        "\"tmem_ld_B_per_clk\": %.1f, \"check\": \"%s\", \"mismatches\": %lld}\n",
        M, N, TS ? "TS (A in TMEM)" : "SS (A, B in smem)", TS ? 1 : NA, NCH, per_sm, clk_per_mma, per_sm * macs / clk_per_mma,
        (TS ? 0 : M * 32) + N * 32, ((TS ? 0 : M * 32) + N * 32) / clk_per_mma, ld_bytes / lm, bad ? "FAIL" : "ok", bad);
    (void)clk_mhz;
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
    cudaFree(dc);
    cudaFree(dl);
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
    run<16, false, 1>(sms, clk);
    run<16, false, 4>(sms, clk);
    run<16, true, 1>(sms, clk);
    run<32, false, 1>(sms, clk);
    run<32, false, 4>(sms, clk);
    run<32, true, 1>(sms, clk);
    run<64, false, 1>(sms, clk);
    run<64, false, 4>(sms, clk);
    run<64, true, 1>(sms, clk);
    run<128, false, 1>(sms, clk);
    run<128, true, 1>(sms, clk);
    run<256, false, 1>(sms, clk);
    run<256, false, 4>(sms, clk);
    run<256, true, 1>(sms, clk);
    // independent accumulators (no dependent accumulate between consecutive MMAs)
    run<16, false, 4, 8>(sms, clk);
    run<16, true, 1, 8>(sms, clk);
    run<16, true, 1, 16>(sms, clk);
    run<32, false, 4, 8>(sms, clk);
    run<32, true, 1, 8>(sms, clk);
    run<64, false, 4, 4>(sms, clk);
    run<64, true, 1, 4>(sms, clk);
    // several CTAs per SM, each with its own issuing thread and accumulators
    run<16, false, 4, 8>(sms, clk, 4);
    run<16, true, 1, 8>(sms, clk, 4);
    run<32, true, 1, 4>(sms, clk, 4);
    run<16, true, 1, 1>(sms, clk, 4);
    return 0;
}
