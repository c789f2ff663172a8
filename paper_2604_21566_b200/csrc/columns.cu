// columns.cu - the reference's column pipeline as separate device stages (§8(a) A10-A13):
// gather_columns, compute_partials, align_and_reduce, carry_pass (include/dot/mul.hpp:
// 32-67, src/mul.cpp:12-90). dot_mul_words fuses all four into one register-resident
// kernel (mul_batch.cu, mul_imma.cu); these stages exist so a caller of the reference's
// public pipeline functions gets the same buffers, bit for bit, from the device.
//
//   gather     pair t of column c (i + j = c, c ascending, i ascending) -> m_a[t] = a[i],
//              m_b[t] = b[c - i]; column c starts at S(c) (closed form below).
//   partials   p_lo = (m_a * m_b) mod 2^k, p_hi = floor(m_a * m_b / 2^k) (truncated to 64
//              bits, as the reference's limb_t cast does), elementwise.
//   reduce     col[c] = sum of p_lo over column c + sum of p_hi over column c - 1, mod
//              2^128 (u128 accumulators): one thread per (pair, column).
//   carry      out[c] = (col + carry) mod 2^k, carry = (col + carry) >> k plus 2^(128-k)
//              when the 128-bit add wrapped; the residual carry appends limbs. One thread
//              per pair (the pass is serial by definition).
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"

namespace dotg {

namespace {

typedef unsigned __int128 u128;

// First pair index of column c for m-limb operands (columns 0 .. 2m - 2).
__host__ __device__ __forceinline__ uint64_t col_start(uint64_t c, uint64_t m) {
    if (c <= m) return c * (c + 1) / 2;
    const uint64_t d = c - m;
    return m * (m + 1) / 2 + d * (m - 1) - d * (d - 1) / 2;
}

// grid.x = columns (2m - 1), grid.y = pairs of the batch
__global__ void __launch_bounds__(256) k_gather_columns(uint64_t* ma, uint64_t* mb, const uint64_t* a,
                                                        const uint64_t* b, uint64_t m) {
    const uint64_t c = blockIdx.x, p = blockIdx.y;
    const uint64_t i_lo = c + 1 >= m ? c + 1 - m : 0, i_hi = c < m - 1 ? c : m - 1;
    const uint64_t base = p * m * m + col_start(c, m) - i_lo;
    const uint64_t* pa = a + p * m;
    const uint64_t* pb = b + p * m;
    for (uint64_t i = i_lo + threadIdx.x; i <= i_hi; i += blockDim.x) {
        ma[base + i] = __ldg(pa + i);
        mb[base + i] = __ldg(pb + (c - i));
    }
}

__global__ void __launch_bounds__(256) k_partials(uint64_t* plo, uint64_t* phi, const uint64_t* ma,
                                                  const uint64_t* mb, uint64_t n, unsigned k) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    const uint64_t mask = k == 64 ? ~0ull : ((1ull << k) - 1);
    for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < n; t += stride) {
        const u128 prod = u128(__ldg(ma + t)) * __ldg(mb + t);
        plo[t] = uint64_t(prod) & mask;
        phi[t] = uint64_t(prod >> k);
    }
}

// cols[p][c] as (lo, hi) 64-bit halves of the u128 column sum, c in 0 .. 2m - 1
__global__ void __launch_bounds__(256) k_align_reduce(uint64_t* cols, const uint64_t* plo, const uint64_t* phi,
                                                      uint64_t m, uint64_t batch) {
    const uint64_t ncol = 2 * m;
    const uint64_t idx = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= ncol * batch) return;
    const uint64_t p = idx / ncol, c = idx - p * ncol;
    const uint64_t off = p * m * m;
    u128 s = 0;
    if (c + 1 < ncol) {  // lows of column c (slot 2m - 1 only ever receives highs)
        const uint64_t t0 = col_start(c, m), t1 = col_start(c + 1, m);
        for (uint64_t t = t0; t < t1; ++t) s += __ldg(plo + off + t);
    }
    if (c >= 1) {  // highs of column c - 1
        const uint64_t t0 = col_start(c - 1, m), t1 = col_start(c, m);
        for (uint64_t t = t0; t < t1; ++t) s += __ldg(phi + off + t);
    }
    cols[2 * idx] = uint64_t(s);
    cols[2 * idx + 1] = uint64_t(s >> 64);
}

__global__ void __launch_bounds__(128) k_carry_pass(uint64_t* out, uint32_t* nout, uint64_t cap, const uint64_t* cols,
                                                    uint64_t ncols, uint64_t batch, unsigned k) {
    const uint64_t p = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= batch) return;
    const uint64_t mask = k == 64 ? ~0ull : ((1ull << k) - 1);
    const uint64_t* pc = cols + 2 * p * ncols;
    uint64_t* po = out + p * cap;
    u128 carry = 0;
    uint64_t n = 0;
    for (uint64_t c = 0; c < ncols; ++c) {
        const u128 col = u128(pc[2 * c]) | (u128(pc[2 * c + 1]) << 64);
        const u128 v = col + carry;
        const u128 wrapped = v < col ? u128(1) << (128 - k) : u128(0);
        po[n++] = uint64_t(v) & mask;
        carry = (v >> k) + wrapped;
    }
    while (carry != 0 && n < cap) {
        po[n++] = uint64_t(carry) & mask;
        carry >>= k;
    }
    nout[p] = uint32_t(n);
}

unsigned grid_for(uint64_t n, unsigned threads) {
    const uint64_t need = (n + threads - 1) / threads;
    return unsigned(need < 148ull * 32 ? need : 148ull * 32);
}

}  // namespace

cudaError_t launch_gather_columns(uint64_t* ma, uint64_t* mb, const uint64_t* a, const uint64_t* b, size_t m,
                                  size_t batch, cudaStream_t st) {
    if (batch == 0 || m == 0) return cudaSuccess;
    if (batch > 65535 || 2 * m - 1 > 0x7fffffffull) return cudaErrorInvalidValue;
    k_gather_columns<<<dim3(unsigned(2 * m - 1), unsigned(batch)), m < 256 ? 32 * unsigned((m + 31) / 32) : 256, 0,
                       st>>>(ma, mb, a, b, m);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_partials(uint64_t* plo, uint64_t* phi, const uint64_t* ma, const uint64_t* mb, size_t n,
                            unsigned k, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_partials<<<grid_for(n, 256), 256, 0, st>>>(plo, phi, ma, mb, n, k);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_align_reduce(uint64_t* cols, const uint64_t* plo, const uint64_t* phi, size_t m, size_t batch,
                                cudaStream_t st) {
    if (batch == 0 || m == 0) return cudaSuccess;
    const uint64_t n = 2 * uint64_t(m) * batch;
    k_align_reduce<<<unsigned((n + 255) / 256), 256, 0, st>>>(cols, plo, phi, m, batch);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_carry_pass(uint64_t* out, uint32_t* nout, size_t cap, const uint64_t* cols, size_t ncols,
                              size_t batch, unsigned k, cudaStream_t st) {
    if (batch == 0) return cudaSuccess;
    k_carry_pass<<<unsigned((batch + 127) / 128), 128, 0, st>>>(out, nout, cap, cols, ncols, batch, k);
    count_launch();
    return cudaGetLastError();
}

}  // namespace dotg
