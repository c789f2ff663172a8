// karatsuba.cu - batched Karatsuba over the B200 base-case multiply (§8(f) item 1).
//
// Reference: karatsuba_mul / kara_rec (include/dot/mul.hpp:87-102, src/mul.cpp:161-233):
// split A = A_H * X + A_L (X = 2^(64h), odd sizes padded to even), three half products
// P1 = A_H B_H, P0 = A_L B_L, PD = |A_H - A_L| |B_H - B_L|, mid = P1 + P0 -+ PD (minus
// when the two differences have the same sign), result P1 X^2 + mid X + P0; the base
// case (m <= theta) is dot_mul_4x4 for m == 4 and dot_mul_words otherwise - both equal to
// the exact 2m-limb product the batched column kernels compute.
//
// B200 formulation: breadth-first. Every node of one recursion level has the same size,
// so a level is ONE batched launch: the 3 children of each of the `count` pairs are
// stacked as [lo; hi; |hi - lo|] into a [3*count][h] batch, down to a single batched
// base-case multiply of 3^L * batch pairs, then one combine launch per level on the way
// back up. Launch count is O(levels), not O(3^levels). Split and combine run one warp per
// pair with lane-strided (coalesced) limbs and ballot-lookahead carries.
//
// Two descents share the machinery: the reference's (h = ceil(m / 2) until m <= theta,
// dotg_karatsuba_batch) and the padded one dotg_mul_batch uses for m > 128 and for
// in-between sizes: m padded to base * 2^L with base a tensor-pipe size (mul_imma.cu),
// so every leaf is one exact IMMA multiply.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <vector>

#include "internal.h"

namespace dotg {

namespace {

// ---------------------------------------------------------------------------
// Warp-per-pair split / combine. Limbs are lane-strided (limb i on lane i % 32, so every
// access is coalesced) and processed in 32-limb chunks; each multi-limb add/sub resolves
// its carries with the add kernel's ballot lookahead (device.cuh algebra):
//   C = (((G << 1) | cin) + P) ^ P per chunk, carry out = bit 32, chained over chunks.
// ---------------------------------------------------------------------------
constexpr int kKaraWarps = 8;

// carry-in of this lane and the chunk carry-out for generate/propagate bits (g, p)
__device__ __forceinline__ uint32_t chunk_carry(uint32_t g, uint32_t p, uint32_t& cin, int lane) {
    const uint32_t G = __ballot_sync(0xffffffffu, g), P = __ballot_sync(0xffffffffu, p);
    const uint64_t y = ((uint64_t(G) << 1) | cin) + uint64_t(P);
    cin = uint32_t(y >> 32);
    return ((uint32_t(y) ^ P) >> lane) & 1u;
}

// Both warp kernels walk a pair in 32-limb chunks whose carries chain serially; the loads
// of kGrp chunks are issued together before their carry chain runs, so a warp keeps kGrp
// chunks of memory traffic in flight instead of one (tools/kara_breakdown.py: the level
// passes were 55-87% of a padded product with one chunk per step).
#ifndef DOTG_KARA_GRP
#define DOTG_KARA_GRP 4
#endif
constexpr int kGrp = DOTG_KARA_GRP;

// Children of pair p, parent read as 2h limbs with zero padding above its m limbs:
//   lo = A[0:h], hi = A[h:2h], df = |hi - lo|, sign = (hi < lo).
// Both operands of a level in one launch: blockIdx.y picks the operand (its own output set).
struct KaraSplitArgs {
    const uint64_t* A;
    uint64_t *lo, *hi, *df;
    uint32_t* sign;
};
__global__ void __launch_bounds__(kKaraWarps * 32) k_kara_split_w(const __grid_constant__ KaraSplitArgs x0,
                                                                  const __grid_constant__ KaraSplitArgs x1, size_t m,
                                                                  size_t h, size_t count) {
    const int lane = threadIdx.x & 31;
    const size_t p = size_t(blockIdx.x) * kKaraWarps + (threadIdx.x >> 5);
    if (p >= count) return;
    const KaraSplitArgs& xa = blockIdx.y == 0 ? x0 : x1;
    const uint64_t* __restrict__ A = xa.A;
    uint64_t* lo = xa.lo;
    uint64_t* hi = xa.hi;
    uint64_t* df = xa.df;
    uint32_t* sign = xa.sign;
    const uint64_t* a = A + p * m;
    auto limb = [&](size_t i) -> uint64_t { return i < m ? __ldg(a + i) : 0ull; };
    uint64_t* plo = lo + p * h;
    uint64_t* phi = hi + p * h;
    uint64_t* pdf = df + p * h;
    // pass 1: copy the halves out and find the highest limb where they differ, which
    // decides the sign (compare, limbs.cpp:46-53)
    unsigned top = 0;  // 1 + index of the highest differing limb seen by this lane
    for (size_t base = 0; base < h; base += 32 * kGrp) {
        uint64_t x[kGrp], y[kGrp];
#pragma unroll
        for (int u = 0; u < kGrp; ++u) {
            const size_t i = base + 32 * u + lane;
            x[u] = i < h ? limb(h + i) : 0ull;
            y[u] = i < h ? limb(i) : 0ull;
        }
#pragma unroll
        for (int u = 0; u < kGrp; ++u) {
            const size_t i = base + 32 * u + lane;
            if (i < h) {
                plo[i] = y[u];
                phi[i] = x[u];
                if (x[u] != y[u]) top = unsigned(i) + 1;
            }
        }
    }
    const unsigned hi_diff = __reduce_max_sync(0xffffffffu, top);
    bool neg = false;
    if (hi_diff != 0) {
        const size_t i = hi_diff - 1;
        neg = limb(h + i) < limb(i);  // every lane reads the same limb (broadcast)
    }
    // pass 2: larger minus smaller, borrows by chunk lookahead
    uint32_t cin = 0;
    for (size_t base = 0; base < h; base += 32 * kGrp) {
        uint64_t x[kGrp], y[kGrp];
#pragma unroll
        for (int u = 0; u < kGrp; ++u) {
            const size_t i = base + 32 * u + lane;
            x[u] = i < h ? limb(h + i) : 0ull;
            y[u] = i < h ? limb(i) : 0ull;
        }
#pragma unroll
        for (int u = 0; u < kGrp; ++u) {
            if (base + 32 * u >= h) break;
            const size_t i = base + 32 * u + lane;
            const bool ok = i < h;
            const uint64_t uu = neg ? y[u] : x[u], vv = neg ? x[u] : y[u];
            const uint64_t d = uu - vv;
            const uint32_t bin = chunk_carry(ok && uu < vv, ok && d == 0, cin, lane);
            if (ok) pdf[i] = d - bin;
        }
    }
    if (lane == 0) sign[p] = neg ? 1u : 0u;
}

// Parent product of pair p from its children's products P = [P0; P1; PD] (each
// [count][2h]): out[p] (2m limbs) = P0 + X (P0 + P1 -+ PD) + X^2 P1, truncated to 2m.
// Three chained multi-limb passes per chunk: T = P0 + P1, M = T -+ PD (>= 0, 2h + 1
// limbs), R[h + j] = base + M[j] with base = P0 below 2h, P1 above.
__global__ void __launch_bounds__(kKaraWarps * 32) k_kara_combine_w(const uint64_t* __restrict__ P, size_t h,
                                                                    size_t count, const uint32_t* sa,
                                                                    const uint32_t* sb, uint64_t* out, size_t m) {
    const int lane = threadIdx.x & 31;
    const size_t p = size_t(blockIdx.x) * kKaraWarps + (threadIdx.x >> 5);
    if (p >= count) return;
    const size_t n2 = 2 * h, n_out = 2 * m;
    const uint64_t* p0 = P + p * n2;
    const uint64_t* p1 = P + (count + p) * n2;
    const uint64_t* pd = P + (2 * count + p) * n2;
    const bool minus = sa[p] == sb[p];  // same-sign differences: mid = P0 + P1 - PD
    uint64_t* o = out + p * n_out;
    for (size_t k = lane; k < h && k < n_out; k += 32) o[k] = __ldg(p0 + k);
    uint32_t cT = 0, cM = 0, cR = 0;
    for (size_t base = 0; base < 3 * h; base += 32 * kGrp) {
        uint64_t x0[kGrp], x1[kGrp], dd[kGrp], bk[kGrp];
#pragma unroll
        for (int u = 0; u < kGrp; ++u) {
            const size_t j = base + 32 * u + lane, k = h + j;
            const bool ok = j < 3 * h, low = j < n2;
            x0[u] = ok && low ? __ldg(p0 + j) : 0ull;
            x1[u] = ok && low ? __ldg(p1 + j) : 0ull;
            dd[u] = ok && low ? __ldg(pd + j) : 0ull;
            bk[u] = !ok ? 0ull : (k < n2 ? __ldg(p0 + k) : __ldg(p1 + (k - n2)));
        }
#pragma unroll
        for (int u = 0; u < kGrp; ++u) {
            if (base + 32 * u >= 3 * h) break;
            const size_t j = base + 32 * u + lane, k = h + j;
            const bool ok = j < 3 * h;
            // T = P0 + P1
            const uint64_t ts = x0[u] + x1[u];
            const uint64_t t = ts + chunk_carry(ok && ts < x0[u], ok && ts == ~0ull, cT, lane);
            // M = T -+ PD
            uint64_t mj;
            if (minus) {
                const uint64_t ms = t - dd[u];
                mj = ms - chunk_carry(ok && t < dd[u], ok && ms == 0, cM, lane);
            } else {
                const uint64_t ms = t + dd[u];
                mj = ms + chunk_carry(ok && ms < t, ok && ms == ~0ull, cM, lane);
            }
            // R[h + j] = base + M[j]
            const uint64_t rs = bk[u] + mj;
            const uint64_t r = rs + chunk_carry(ok && rs < bk[u], ok && rs == ~0ull, cR, lane);
            if (ok && k < n_out) o[k] = r;
        }
    }
}

// CTA-per-pair combine for levels with few pairs (a warp per pair leaves most SMs idle
// and walks 3h limbs serially): the same three chains, one after the other over the whole
// CTA, each a segmented add - warp w streams its share of the 32-limb chunks resolved with
// carry-in 0 and stores them, the warps' (G, P) meet in shared memory behind one barrier,
// and a warp whose carry-in is 1 rewrites its segment's carry-dependent prefix (the
// propagating limbs up to the first non-propagating one, which takes +-1; with random
// limbs one chunk). T = P0 + P1 goes to scratch, M = T -+ PD in place, then R[h + j] =
// base + M into the output.
constexpr int kComboWarps = 16;
// x[j] = j < na ? xa[j] : (j - na < nb ? xb[j - na] : 0)
__device__ __forceinline__ uint64_t cat_limb(const uint64_t* xa, size_t na, const uint64_t* xb, size_t nb, size_t j) {
    if (j < na) return xa[j];
    return j - na < nb ? xb[j - na] : 0ull;
}
__device__ void cta_chain(bool sub, uint64_t* d, const uint64_t* xa, size_t na, const uint64_t* xb, size_t nb,
                          const uint64_t* y, size_t ny, size_t n, uint32_t* sh) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, W = blockDim.x >> 5;
    const uint64_t prop = sub ? 0ull : ~0ull;  // a limb that passes a carry / borrow on
    const size_t nch = (n + 31) / 32, cpw = (nch + W - 1) / W;
    const size_t c0 = size_t(w) * cpw < nch ? size_t(w) * cpw : nch;
    const size_t c1 = c0 + cpw < nch ? c0 + cpw : nch;
    uint32_t cin = 0, allp = 1;
    for (size_t cb = c0; cb < c1; cb += kGrp) {
        uint64_t xv[kGrp], yv[kGrp];
#pragma unroll
        for (int u = 0; u < kGrp; ++u) {
            const size_t j = (cb + u) * 32 + lane;
            const bool ok = cb + u < c1 && j < n;
            xv[u] = ok ? cat_limb(xa, na, xb, nb, j) : 0ull;
            yv[u] = ok && j < ny ? y[j] : 0ull;
        }
#pragma unroll
        for (int u = 0; u < kGrp; ++u) {
            if (cb + u >= c1) break;
            const size_t j = (cb + u) * 32 + lane;
            const bool ok = j < n;
            const uint64_t sv = sub ? xv[u] - yv[u] : xv[u] + yv[u];
            const uint32_t g = ok && (sub ? xv[u] < yv[u] : sv < xv[u]), pp = ok && sv == prop;
            const uint32_t ci = chunk_carry(g, pp, cin, lane);
            const uint64_t r = sub ? sv - ci : sv + ci;
            if (ok) d[j] = r;
            allp &= __ballot_sync(0xffffffffu, ok && r != prop) == 0u;
        }
    }
    if (lane == 0) {
        sh[w] = c0 < c1 ? cin : 0u;
        sh[32 + w] = c0 < c1 ? allp : 1u;
    }
    __syncthreads();
    uint32_t c = 0;  // carry into this warp's segment
    for (int i = 0; i < w; ++i) c = sh[i] | (sh[32 + i] & c);
    if (c != 0u) {
        for (size_t cb = c0; cb < c1; ++cb) {
            const size_t j = cb * 32 + lane;
            const bool ok = j < n;
            const uint64_t r = ok ? d[j] : prop;
            const uint32_t np = __ballot_sync(0xffffffffu, r != prop);
            const int q = np ? __ffs(np) - 1 : 32;
            if (ok && lane < q) d[j] = ~prop;  // the propagating limbs flip
            if (lane == q) d[j] = sub ? r - 1 : r + 1;
            if (np) break;
        }
    }
    __syncthreads();  // results visible to the next chain, shared words reusable
}
__global__ void __launch_bounds__(kComboWarps * 32) k_kara_combine_cta(const uint64_t* __restrict__ P, size_t h,
                                                                       size_t count, const uint32_t* sa,
                                                                       const uint32_t* sb, uint64_t* out, size_t m,
                                                                       uint64_t* scratch) {
    __shared__ uint32_t sh[64];
    const size_t p = blockIdx.x;
    const size_t n2 = 2 * h, n3 = 3 * h, n_out = 2 * m;
    const uint64_t* p0 = P + p * n2;
    const uint64_t* p1 = P + (count + p) * n2;
    const uint64_t* pd = P + (2 * count + p) * n2;
    uint64_t* T = scratch + p * n3;
    uint64_t* o = out + p * n_out;
    const bool minus = sa[p] == sb[p];  // same-sign differences: mid = P0 + P1 - PD
    for (size_t k = threadIdx.x; k < h && k < n_out; k += blockDim.x) o[k] = p0[k];
    cta_chain(false, T, p0, n2, nullptr, 0, p1, n2, n3, sh);  // T = P0 + P1
    cta_chain(minus, T, T, n3, nullptr, 0, pd, n2, n3, sh);   // M = T -+ PD (>= 0)
    if (n_out > h)                                            // R[h + j] = (P0[h:2h) ++ P1) + M
        cta_chain(false, o + h, p0 + h, h, p1, n2, T, n3, n3 < n_out - h ? n3 : n_out - h, sh);
}

// CTA-per-pair split for the same few-pair levels: the halves copied out and the highest
// differing limb found by every warp over its share (one barrier), then |hi - lo| as one
// segmented chain (larger minus smaller). blockIdx.y picks the operand as in the warp kernel.
__global__ void __launch_bounds__(kComboWarps * 32) k_kara_split_cta(const __grid_constant__ KaraSplitArgs x0,
                                                                     const __grid_constant__ KaraSplitArgs x1,
                                                                     size_t m, size_t h, size_t count) {
    __shared__ uint32_t sh[64];
    __shared__ unsigned top;
    const KaraSplitArgs& xa = blockIdx.y == 0 ? x0 : x1;
    const size_t p = blockIdx.x;
    const uint64_t* a = xa.A + p * m;
    uint64_t* plo = xa.lo + p * h;
    uint64_t* phi = xa.hi + p * h;
    if (threadIdx.x == 0) top = 0;
    __syncthreads();
    unsigned mine = 0;  // 1 + highest index where the halves differ, this thread's limbs
    for (size_t i = threadIdx.x; i < h; i += blockDim.x) {
        const uint64_t y = a[i], x = h + i < m ? a[h + i] : 0ull;
        plo[i] = y;
        phi[i] = x;
        if (x != y) mine = unsigned(i) + 1;
    }
    mine = __reduce_max_sync(0xffffffffu, mine);
    if ((threadIdx.x & 31) == 0 && mine) atomicMax(&top, mine);
    __syncthreads();
    bool neg = false;
    if (top != 0) {
        const size_t i = top - 1;
        neg = (h + i < m ? a[h + i] : 0ull) < a[i];
    }
    const size_t nh = m > h ? m - h : 0;  // limbs of the upper half actually stored
    if (neg)
        cta_chain(true, xa.df + p * h, a, h, nullptr, 0, a + h, nh, h, sh);  // lo - hi
    else
        cta_chain(true, xa.df + p * h, a + h, nh, nullptr, 0, a, h, h, sh);  // hi - lo
    if (threadIdx.x == 0) xa.sign[p] = neg ? 1u : 0u;
}

// dst[r][0:nd) = src[r][0:ns) zero-extended or truncated: one thread per destination
// limb over the flat [rows][nd] array (coalesced stores; the row index comes from a 32-bit
// division when the array is small enough, which covers every batch that fits in HBM
// for the row widths this serves).
__global__ void __launch_bounds__(256) k_copy_rows(const uint64_t* __restrict__ src, size_t ns,
                                                   uint64_t* __restrict__ dst, size_t nd, size_t rows) {
    const size_t total = rows * nd;
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
        size_t r, c;
        if (total < (size_t(1) << 32)) {
            r = uint32_t(i) / uint32_t(nd);
            c = uint32_t(i) - uint32_t(r) * uint32_t(nd);
        } else {
            r = i / nd;
            c = i - r * nd;
        }
        dst[i] = c < ns ? __ldg(src + r * ns + c) : 0ull;
    }
}

unsigned copy_grid(size_t rows, size_t nd) {
    const size_t need = (rows * nd + 255) / 256;
    return unsigned(need < size_t(148 * 16) ? need : size_t(148 * 16));
}

// ---------------------------------------------------------------------------
// Wide split / combine for the top levels of very large products (few pairs of many
// limbs): a warp per pair would walk a whole 2^23-limb half serially, so these levels are
// composed from the batched long-number add/sub (addsub_long.cu: multi-CTA per number,
// three passes) plus coalesced copy / select kernels. Same results as the warp kernels.
// ---------------------------------------------------------------------------
// dst[r * ds + doff + c] = src ? src[r * ss + soff + c] : 0, for c < n
__global__ void __launch_bounds__(256) k_copy_2d(uint64_t* __restrict__ dst, size_t ds, size_t doff,
                                                 const uint64_t* __restrict__ src, size_t ss, size_t soff, size_t n,
                                                 size_t rows) {
    const size_t total = rows * n, stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
        const size_t r = i / n, c = i - r * n;
        dst[r * ds + doff + c] = src != nullptr ? __ldg(src + r * ss + soff + c) : 0ull;
    }
}

// Rows of dst (n limbs) replaced by the rows of alt where flag[r] != 0.
__global__ void __launch_bounds__(256) k_select_rows(uint64_t* __restrict__ dst, const uint64_t* __restrict__ alt,
                                                     const uint32_t* __restrict__ flag, size_t n, size_t rows) {
    const size_t total = rows * n, stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
        const size_t r = i / n;
        if (__ldg(flag + r) != 0u) dst[i] = __ldg(alt + i);
    }
}

// Mz[r] (3h limbs) = M (2h limbs) ++ top ++ 0...: M = T - PD if the two differences have
// the same sign, else T + PD; top = cT - borrow or cT + carry (the true mid is >= 0 and
// below 2^(64 (2h + 1)), so top is 0 or 1).
__global__ void __launch_bounds__(256) k_make_mid(uint64_t* __restrict__ mz, const uint64_t* __restrict__ mplus,
                                                  const uint64_t* __restrict__ mminus, const uint32_t* cT,
                                                  const uint32_t* cP, const uint32_t* bM, const uint32_t* sa,
                                                  const uint32_t* sb, size_t h, size_t rows) {
    const size_t n2 = 2 * h, n3 = 3 * h, total = rows * n3, stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
        const size_t r = i / n3, c = i - r * n3;
        const bool minus = __ldg(sa + r) == __ldg(sb + r);
        uint64_t v = 0;
        if (c < n2) v = __ldg((minus ? mminus : mplus) + r * n2 + c);
        else if (c == n2) v = uint64_t(__ldg(cT + r)) + (minus ? uint64_t(0) - __ldg(bM + r) : uint64_t(__ldg(cP + r)));
        mz[i] = v;
    }
}

unsigned flat_grid(size_t total) {
    const size_t need = (total + 255) / 256;
    return unsigned(need < size_t(148 * 16) ? need : size_t(148 * 16));
}

// Wide when each warp would walk >= 4096 limbs and there are too few pairs to fill the
// GPU with warps; the long-number kernels take at most 65535 numbers per launch.
#ifndef DOTG_KARA_WIDE_H
#define DOTG_KARA_WIDE_H 4096
#endif
bool kara_wide(size_t h, size_t count) { return h >= DOTG_KARA_WIDE_H && count <= 2048; }

cudaError_t split_wide(const uint64_t* A, size_t m, size_t h, size_t count, uint64_t* lo, uint64_t* hi,
                       uint64_t* df, uint32_t* sign, cudaStream_t st) {
    uint64_t* alt = nullptr;
    cudaError_t e = cudaMallocAsync(&alt, count * h * 8, st);
    if (e != cudaSuccess) return e;
    k_copy_2d<<<flat_grid(count * h), 256, 0, st>>>(lo, h, 0, A, m, 0, h, count);
    k_copy_2d<<<flat_grid(count * (m - h)), 256, 0, st>>>(hi, h, 0, A, m, h, m - h, count);
    if (m - h < h) k_copy_2d<<<flat_grid(count * (2 * h - m)), 256, 0, st>>>(hi, h, m - h, nullptr, 0, 0, 2 * h - m, count);
    count_launch(m - h < h ? 3 : 2);
    e = cudaGetLastError();
    // df = hi - lo, borrow = (hi < lo) = the sign; where negative, df = lo - hi instead
    if (e == cudaSuccess) e = launch_long_batch(true, df, hi, lo, sign, h, count, st);
    if (e == cudaSuccess) e = launch_long_batch(true, alt, lo, hi, nullptr, h, count, st);
    if (e == cudaSuccess) {
        k_select_rows<<<flat_grid(count * h), 256, 0, st>>>(df, alt, sign, h, count);
        count_launch();
        e = cudaGetLastError();
    }
    cudaFreeAsync(alt, st);
    return e;
}

cudaError_t combine_wide(const uint64_t* P, size_t h, size_t count, const uint32_t* sa, const uint32_t* sb,
                         uint64_t* out, size_t m, cudaStream_t st) {
    const size_t n2 = 2 * h, n3 = 3 * h;
    const uint64_t* p0 = P;
    const uint64_t* p1 = P + count * n2;
    const uint64_t* pd = P + 2 * count * n2;
    char* base = nullptr;
    const size_t w2 = count * n2 * 8, w3 = count * n3 * 8, fl = (count * 4 + 255) / 256 * 256;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&base), 3 * w2 + 2 * w3 + 3 * fl, st);
    if (e != cudaSuccess) return e;
    uint64_t* T = reinterpret_cast<uint64_t*>(base);
    uint64_t* Mp = reinterpret_cast<uint64_t*>(base + w2);
    uint64_t* Mm = reinterpret_cast<uint64_t*>(base + 2 * w2);
    uint64_t* Mz = reinterpret_cast<uint64_t*>(base + 3 * w2);
    uint64_t* Rh = reinterpret_cast<uint64_t*>(base + 3 * w2 + w3);
    uint32_t* cT = reinterpret_cast<uint32_t*>(base + 3 * w2 + 2 * w3);
    uint32_t* cP = reinterpret_cast<uint32_t*>(base + 3 * w2 + 2 * w3 + fl);
    uint32_t* bM = reinterpret_cast<uint32_t*>(base + 3 * w2 + 2 * w3 + 2 * fl);
    e = launch_long_batch(false, T, p0, p1, cT, n2, count, st);                 // T = P0 + P1
    if (e == cudaSuccess) e = launch_long_batch(false, Mp, T, pd, cP, n2, count, st);  // T + PD
    if (e == cudaSuccess) e = launch_long_batch(true, Mm, T, pd, bM, n2, count, st);   // T - PD
    if (e == cudaSuccess) {
        k_make_mid<<<flat_grid(count * n3), 256, 0, st>>>(Mz, Mp, Mm, cT, cP, bM, sa, sb, h, count);
        // Rh = P0[h:2h) ++ P1: the parent product's limbs from h up before adding the mid
        k_copy_2d<<<flat_grid(count * h), 256, 0, st>>>(Rh, n3, 0, p0, n2, h, h, count);
        k_copy_2d<<<flat_grid(count * n2), 256, 0, st>>>(Rh, n3, h, p1, n2, 0, n2, count);
        count_launch(3);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = launch_long_batch(false, Rh, Rh, Mz, nullptr, n3, count, st);  // += mid * X
    if (e == cudaSuccess) {
        const size_t no = 2 * m;  // out rows: P0[0:h) ++ Rh, truncated to 2m limbs
        k_copy_2d<<<flat_grid(count * h), 256, 0, st>>>(out, no, 0, p0, n2, 0, h, count);
        k_copy_2d<<<flat_grid(count * (no - h)), 256, 0, st>>>(out, no, h, Rh, n3, 0, no - h, count);
        count_launch(2);
        e = cudaGetLastError();
    }
    cudaFreeAsync(base, st);
    return e;
}

#ifndef DOTG_KARA_CTA_PAIRS
#define DOTG_KARA_CTA_PAIRS 512  // below this many pairs a level's split / combine take a CTA per pair
#endif
size_t kara_cta_pairs() {
    static const size_t v = [] {
        const char* e = std::getenv("DOTG_KARA_CTA_PAIRS");  // A/B knob
        return e ? size_t(std::atoll(e)) : size_t(DOTG_KARA_CTA_PAIRS);
    }();
    return v;
}

// Children of both operands of a level: [lo; hi; |hi - lo|] of A into nA (signs sa), of B
// into nB (signs sb). The warp kernel takes both in one launch (the level's pairs are
// latency-bound warps: twice the warps in flight at once).
cudaError_t kara_split2(const uint64_t* A, const uint64_t* B, size_t m, size_t h, size_t count, uint64_t* nA,
                        uint64_t* nB, uint32_t* sa, uint32_t* sb, cudaStream_t st) {
    if (kara_wide(h, count)) {
        cudaError_t e = split_wide(A, m, h, count, nA, nA + count * h, nA + 2 * count * h, sa, st);
        if (e == cudaSuccess) e = split_wide(B, m, h, count, nB, nB + count * h, nB + 2 * count * h, sb, st);
        return e;
    }
    const KaraSplitArgs xa{A, nA, nA + count * h, nA + 2 * count * h, sa};
    const KaraSplitArgs xb{B, nB, nB + count * h, nB + 2 * count * h, sb};
    if (count < kara_cta_pairs() && h >= 64) {
        k_kara_split_cta<<<dim3(unsigned(count), 2), kComboWarps * 32, 0, st>>>(xa, xb, m, h, count);
    } else {
        const dim3 grid(unsigned((count + kKaraWarps - 1) / kKaraWarps), 2);
        k_kara_split_w<<<grid, kKaraWarps * 32, 0, st>>>(xa, xb, m, h, count);
    }
    count_launch();
    return cudaGetLastError();
}

cudaError_t kara_combine(const uint64_t* P, size_t h, size_t count, const uint32_t* sa, const uint32_t* sb,
                         uint64_t* out, size_t m, cudaStream_t st) {
    if (kara_wide(h, count)) return combine_wide(P, h, count, sa, sb, out, m, st);
    if (count < kara_cta_pairs() && h >= 64) {
        uint64_t* T = nullptr;
        cudaError_t e = cudaMallocAsync(&T, count * 3 * h * 8, st);
        if (e != cudaSuccess) return e;
        k_kara_combine_cta<<<unsigned(count), kComboWarps * 32, 0, st>>>(P, h, count, sa, sb, out, m, T);
        count_launch();
        e = cudaGetLastError();
        cudaError_t e2 = cudaFreeAsync(T, st);
        return e != cudaSuccess ? e : e2;
    }
    k_kara_combine_w<<<unsigned((count + kKaraWarps - 1) / kKaraWarps), kKaraWarps * 32, 0, st>>>(P, h, count, sa,
                                                                                                   sb, out, m);
    count_launch();
    return cudaGetLastError();
}

// The level sizes of a descent: parent m_i (the limbs actually read), half h_i.
struct KaraPlan {
    std::vector<size_t> pm, h;
};

// Peak scratch bytes of a breadth-first run over levels d0.. of `plan`: each level's
// buffers are released (stream-ordered) as soon as the next level has consumed them, so
// the peak is the largest adjacent pair of levels (in practice the leaves: their operands
// plus their products) plus the per-level sign arrays.
size_t kara_bf_bytes(const KaraPlan& plan, size_t d0, size_t batch) {
    auto r256 = [](size_t x) { return (x < 256 ? 256 : x + 255) / 256 * 256; };
    const size_t L = plan.h.size();
    std::vector<size_t> cnt(L + 1);
    cnt[d0] = batch;
    for (size_t d = d0; d < L; ++d) cnt[d + 1] = 3 * cnt[d];
    size_t signs = 0, peak = 0;
    for (size_t d = d0; d < L; ++d) {
        signs += 2 * r256(cnt[d] * 4);
        const size_t in = d > d0 ? 2 * r256(cnt[d] * plan.pm[d] * 8) : 0;
        peak = std::max(peak, in + 2 * r256(3 * cnt[d] * plan.h[d] * 8));
    }
    const size_t cm = plan.h[L - 1];
    peak = std::max(peak, 2 * r256(cnt[L] * cm * 8) + r256(cnt[L] * 2 * cm * 8));
    for (size_t d = d0 + 1; d < L; ++d)  // combine at level d: children's products -> level-d products
        peak = std::max(peak, r256(cnt[d + 1] * 2 * plan.h[d] * 8) + r256(cnt[d] * 2 * plan.pm[d] * 8));
    return peak + signs;
}

cudaError_t run_karatsuba_bf(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t batch,
                             const KaraPlan& plan, size_t d0, cudaStream_t st) {
    struct Level {
        size_t m, h, count;
        uint32_t *sa, *sb;  // signs of this level's differences: [count]
    };
    std::vector<Level> lv;
    std::vector<void*> signs;  // released at the end
    auto alloc = [&](size_t bytes) -> void* {
        void* p = nullptr;
        if (cudaMallocAsync(&p, bytes < 256 ? 256 : bytes, st) != cudaSuccess) return nullptr;
        return p;
    };
    auto release = [&](const void* p) {
        if (p != nullptr) cudaFreeAsync(const_cast<void*>(p), st);
    };
    auto cleanup = [&]() {
        for (void* p : signs) cudaFreeAsync(p, st);
    };
    size_t count = batch, cm = plan.pm.empty() ? 0 : plan.pm[d0];
    const uint64_t* A = a;
    const uint64_t* B = b;
    // Descend: split every level until the base case; a level's operands are released once
    // the next level's split has been issued.
    for (size_t d = d0; d < plan.h.size(); ++d) {
        const size_t h = plan.h[d];
        Level L{plan.pm[d], h, count, nullptr, nullptr};
        uint64_t* nA = static_cast<uint64_t*>(alloc(3 * count * h * 8));
        uint64_t* nB = static_cast<uint64_t*>(alloc(3 * count * h * 8));
        L.sa = static_cast<uint32_t*>(alloc(count * 4));
        L.sb = static_cast<uint32_t*>(alloc(count * 4));
        if (L.sa) signs.push_back(L.sa);
        if (L.sb) signs.push_back(L.sb);
        if (!nA || !nB || !L.sa || !L.sb) {
            release(nA);
            release(nB);
            if (d > d0) {
                release(A);
                release(B);
            }
            cleanup();
            return cudaErrorMemoryAllocation;
        }
        cudaError_t es = kara_split2(A, B, L.m, h, count, nA, nB, L.sa, L.sb, st);
        if (d > d0) {
            release(A);
            release(B);
        }
        if (es != cudaSuccess) {
            release(nA);
            release(nB);
            cleanup();
            return es;
        }
        lv.push_back(L);
        A = nA;
        B = nB;
        cm = h;
        count *= 3;
    }
    // Base case: one batched column multiply of all 3^L * batch leaves.
    uint64_t* P = static_cast<uint64_t*>(alloc(count * 2 * cm * 8));
    if (!P) {
        release(A);
        release(B);
        cleanup();
        return cudaErrorMemoryAllocation;
    }
    cudaError_t e = launch_mul_batch(P, A, B, cm, count, 0, st);
    release(A);
    release(B);
    // Ascend: combine level by level, releasing each level's products once combined.
    for (size_t i = lv.size(); e == cudaSuccess && i-- > 0;) {
        const Level& L = lv[i];
        uint64_t* dst = i == 0 ? out : static_cast<uint64_t*>(alloc(L.count * 2 * L.m * 8));
        if (!dst) {
            e = cudaErrorMemoryAllocation;
            break;
        }
        e = kara_combine(P, L.h, L.count, L.sa, L.sb, dst, L.m, st);
        release(P);
        P = dst;
    }
    if (e != cudaSuccess && P != out) release(P);
    cleanup();
    return e;
}

// Depth-first above the level where the breadth-first scratch fits: the three children
// of the top level run one after another (each as its own, smaller, breadth-first run),
// so the largest products (up to the reference cap of 2^24 limbs, mul.hpp:26-30) stay
// within device memory. Budget: see run_karatsuba.
cudaError_t run_karatsuba_at(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t batch,
                             const KaraPlan& plan, size_t d0, size_t budget, cudaStream_t st) {
    if (kara_bf_bytes(plan, d0, batch) <= budget || d0 + 1 == plan.h.size())
        return run_karatsuba_bf(out, a, b, batch, plan, d0, st);
    const size_t m = plan.pm[d0], h = plan.h[d0];
    uint64_t *nA = nullptr, *nB = nullptr, *P = nullptr;
    uint32_t *sa = nullptr, *sb = nullptr;
    cudaError_t e = cudaMallocAsync(&nA, 3 * batch * h * 8, st);
    if (e == cudaSuccess) e = cudaMallocAsync(&nB, 3 * batch * h * 8, st);
    if (e == cudaSuccess) e = cudaMallocAsync(&sa, batch * 4 < 256 ? 256 : batch * 4, st);
    if (e == cudaSuccess) e = cudaMallocAsync(&sb, batch * 4 < 256 ? 256 : batch * 4, st);
    if (e == cudaSuccess) e = cudaMallocAsync(&P, 3 * batch * 2 * h * 8, st);
    if (e == cudaSuccess) {
        e = kara_split2(a, b, m, h, batch, nA, nB, sa, sb, st);
        // the next level's plan entry describes a child of h limbs (pm[d0 + 1] == h)
        for (int k = 0; k < 3 && e == cudaSuccess; ++k)
            e = run_karatsuba_at(P + size_t(k) * batch * 2 * h, nA + size_t(k) * batch * h,
                                 nB + size_t(k) * batch * h, batch, plan, d0 + 1, budget, st);
    }
    if (e == cudaSuccess) e = kara_combine(P, h, batch, sa, sb, out, m, st);
    for (void* q : {static_cast<void*>(nA), static_cast<void*>(nB), static_cast<void*>(sa), static_cast<void*>(sb),
                    static_cast<void*>(P)})
        if (q != nullptr) cudaFreeAsync(q, st);
    return e;
}

cudaError_t run_karatsuba(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t batch, const KaraPlan& plan,
                          cudaStream_t st) {
    // small runs skip the free-memory query (cudaMemGetInfo costs host time on every call)
    const char* env_budget = std::getenv("DOTG_KARA_BUDGET_MB");
    if (env_budget == nullptr && kara_bf_bytes(plan, 0, batch) <= (size_t(1) << 30))
        return run_karatsuba_bf(out, a, b, batch, plan, 0, st);
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) free_b = size_t(16) << 30;
    // breadth-first while its scratch stays inside the pool's 8 GiB reserve (7 GiB, or 70%
    // of free memory if less): larger scratch is re-mapped by the driver on every call, which
    // cost more than going depth-first now that the top levels split and combine with the
    // multi-CTA long-number passes (tools/mul_max_timing.py: 2^22 limbs 140 ms vs 0.7-0.8 s,
    // 2^24 limbs 1.21 s vs 1.7-1.9 s with a 70%-of-free budget)
    size_t budget = std::min(free_b / 10 * 7, size_t(7) << 30);
    if (env_budget != nullptr) budget = size_t(std::strtoull(env_budget, nullptr, 10)) << 20;
    return run_karatsuba_at(out, a, b, batch, plan, 0, budget, st);
}

}  // namespace

void retain_stream_pool() {
    // keep freed scratch (Karatsuba levels, long-number state) cached in the device's
    // stream-ordered pool instead of returning it to the driver at every sync
    static thread_local int pool_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (pool_dev == dev) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        // up to 8 GiB stays reserved (memory held here is invisible to cudaMalloc users such
        // as torch's allocator, so the cache is bounded; DOTG_POOL_KEEP_GB overrides). Scratch
        // beyond it is re-mapped per call: a 2^21-limb product's 20 GB leaves, for example.
        uint64_t thr = uint64_t(8) << 30;
        if (const char* e = std::getenv("DOTG_POOL_KEEP_GB")) thr = uint64_t(std::strtoull(e, nullptr, 10)) << 30;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    pool_dev = dev;
}

// Copy the rows into aligned temporaries zero-extended to mp >= m limbs, multiply there
// (row-major fast kernels need 32-byte aligned rows of their own sizes), keep the low 2m
// limbs of each product. Any alignment of out / a / b.
cudaError_t mul_padded_rows(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch, size_t mp,
                            cudaStream_t st) {
    if (batch == 0) return cudaSuccess;
    retain_stream_pool();
    uint64_t *pa = nullptr, *pb = nullptr, *po = nullptr;
    cudaError_t e = cudaMallocAsync(&pa, batch * mp * 8, st);
    if (e == cudaSuccess) e = cudaMallocAsync(&pb, batch * mp * 8, st);
    if (e == cudaSuccess) e = cudaMallocAsync(&po, batch * 2 * mp * 8, st);
    if (e == cudaSuccess) {
        k_copy_rows<<<copy_grid(batch, mp), 256, 0, st>>>(a, m, pa, mp, batch);
        k_copy_rows<<<copy_grid(batch, mp), 256, 0, st>>>(b, m, pb, mp, batch);
        count_launch(2);
        e = launch_mul_batch(po, pa, pb, mp, batch, 0, st);
    }
    if (e == cudaSuccess) {
        k_copy_rows<<<copy_grid(batch, 2 * m), 256, 0, st>>>(po, 2 * mp, out, 2 * m, batch);
        count_launch();
        e = cudaGetLastError();
    }
    for (void* q : {static_cast<void*>(pa), static_cast<void*>(pb), static_cast<void*>(po)})
        if (q != nullptr) cudaFreeAsync(q, st);
    return e;
}

// Row-pitched operands / product (views of wider arrays): gather the rows into dense
// scratch, run the dense route, scatter the product rows (two extra coalesced passes).
cudaError_t launch_mul_pitched(uint64_t* out, size_t ldo, const uint64_t* a, size_t lda, const uint64_t* b,
                               size_t ldb, size_t m, size_t batch, cudaStream_t st) {
    if (batch == 0) return cudaSuccess;
    if (ldo == 2 * m && lda == m && ldb == m) return launch_mul_batch(out, a, b, m, batch, 0, st);
    retain_stream_pool();
    uint64_t *pa = nullptr, *pb = nullptr, *po = nullptr;
    cudaError_t e = cudaMallocAsync(&pa, batch * m * 8, st);
    if (e == cudaSuccess) e = cudaMallocAsync(&pb, batch * m * 8, st);
    if (e == cudaSuccess) e = cudaMallocAsync(&po, batch * 2 * m * 8, st);
    if (e == cudaSuccess) {
        k_copy_2d<<<flat_grid(batch * m), 256, 0, st>>>(pa, m, 0, a, lda, 0, m, batch);
        k_copy_2d<<<flat_grid(batch * m), 256, 0, st>>>(pb, m, 0, b, ldb, 0, m, batch);
        count_launch(2);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = launch_mul_batch(po, pa, pb, m, batch, 0, st);
    if (e == cudaSuccess) {
        k_copy_2d<<<flat_grid(batch * 2 * m), 256, 0, st>>>(out, ldo, 0, po, 2 * m, 0, 2 * m, batch);
        count_launch();
        e = cudaGetLastError();
    }
    for (void* q : {static_cast<void*>(pa), static_cast<void*>(pb), static_cast<void*>(po)})
        if (q != nullptr) cudaFreeAsync(q, st);
    return e;
}

// Reference recursion (kara_rec, mul.cpp:176-233): split h = ceil(m / 2) until m <= theta.
cudaError_t launch_karatsuba_batch(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                                   size_t theta, cudaStream_t st) {
    if (batch == 0) return cudaSuccess;
    if (m <= theta) return launch_mul_batch(out, a, b, m, batch, 0, st);
    retain_stream_pool();
    KaraPlan plan;
    for (size_t cm = m; cm > theta; cm = (cm + 1) / 2) {
        plan.pm.push_back(cm);
        plan.h.push_back((cm + 1) / 2);
    }
    return run_karatsuba(out, a, b, batch, plan, st);
}

// Large products for dotg_mul_batch: pad m up to base * 2^L (base a tensor-pipe size),
// so every leaf is an exact tensor-pipe multiply; the top split zero-pads, the top
// combine truncates to 2m limbs.
cudaError_t launch_karatsuba_padded(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                                    size_t base, cudaStream_t st) {
    if (batch == 0) return cudaSuccess;
    retain_stream_pool();
    size_t mp = base;
    int levels = 0;
    while (mp < m) {
        mp *= 2;
        ++levels;
    }
    if (levels == 0) {
        if (m == mp) return launch_mul_batch(out, a, b, m, batch, 0, st);
        return mul_padded_rows(out, a, b, m, batch, mp, st);
    }
    KaraPlan plan;
    size_t cm = m, full = mp;
    for (int d = 0; d < levels; ++d) {
        plan.pm.push_back(cm);
        plan.h.push_back(full / 2);
        full /= 2;
        cm = full;
    }
    return run_karatsuba(out, a, b, batch, plan, st);
}

}  // namespace dotg
