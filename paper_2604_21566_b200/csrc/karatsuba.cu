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
// back up. Launch count is O(levels), not O(3^levels).
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "internal.h"

namespace dotg {

namespace {

typedef unsigned __int128 u128;
typedef __int128 s128;

// Children of pair p (rows of m limbs, read as 2h limbs with a zero pad when m is odd):
//   lo[p] = A[p][0:h], hi[p] = A[p][h:2h], df[p] = |hi - lo|, sign[p] = (hi < lo).
__global__ void k_kara_split(const uint64_t* A, size_t m, size_t h, size_t count, uint64_t* lo, uint64_t* hi,
                             uint64_t* df, uint32_t* sign) {
    const size_t p = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= count) return;
    const uint64_t* a = A + p * m;
    auto limb = [&](size_t i) -> uint64_t { return i < m ? a[i] : 0ull; };
    // compare hi vs lo from the top (limbs.cpp:46-53 restricted to equal lengths)
    int cmp = 0;
    for (size_t i = h; i-- > 0;) {
        const uint64_t x = limb(h + i), y = limb(i);
        if (x != y) {
            cmp = x < y ? -1 : 1;
            break;
        }
    }
    const bool neg = cmp < 0;
    uint64_t* plo = lo + p * h;
    uint64_t* phi = hi + p * h;
    uint64_t* pdf = df + p * h;
    uint32_t bw = 0;
    for (size_t i = 0; i < h; ++i) {
        const uint64_t x = limb(h + i), y = limb(i);
        plo[i] = y;
        phi[i] = x;
        const uint64_t u = neg ? y : x, v = neg ? x : y;  // larger minus smaller
        const uint64_t d = u - v;
        const uint32_t b1 = u < v;
        const uint64_t r = d - bw;
        bw = b1 | (d < uint64_t(bw));
        pdf[i] = r;
    }
    sign[p] = neg ? 1u : 0u;
}

// Parent product of pair p from its children's products P = [P0; P1; PD] (each
// [count][2h]): out[p] (2m limbs) = P0 + X (P0 + P1 -+ PD) + X^2 P1, truncated to 2m.
__global__ void k_kara_combine(const uint64_t* P, size_t h, size_t count, const uint32_t* sa, const uint32_t* sb,
                               uint64_t* out, size_t m) {
    const size_t p = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= count) return;
    const size_t n2 = 2 * h;
    const uint64_t* p0 = P + p * n2;
    const uint64_t* p1 = P + (count + p) * n2;
    const uint64_t* pd = P + (2 * count + p) * n2;
    const bool minus = sa[p] == sb[p];  // same-sign differences: mid = P0 + P1 - PD
    uint64_t* o = out + p * (2 * m);
    s128 vc = 0;   // signed carry of V = P0 + P1 -+ PD (V >= 0, 2h + 1 limbs)
    u128 oc = 0;   // carry of the final sum
    for (size_t k = 0; k < 4 * h; ++k) {
        u128 t = oc + (k < n2 ? p0[k] : p1[k - n2]);
        if (k >= h && k <= 3 * h) {
            const size_t j = k - h;
            uint64_t vj;
            if (j < n2) {
                const s128 s = vc + s128(p0[j]) + s128(p1[j]) + (minus ? -s128(pd[j]) : s128(pd[j]));
                vj = uint64_t(s);
                vc = s >> 64;
            } else {
                vj = uint64_t(vc);  // V's top limb (non-negative)
            }
            t += vj;
        }
        if (k < 2 * m) o[k] = uint64_t(t);
        oc = t >> 64;
    }
}

unsigned blocks_for(size_t n) { return unsigned((n + 127) / 128); }

}  // namespace

cudaError_t launch_karatsuba_batch(uint64_t* out, const uint64_t* a, const uint64_t* b, size_t m, size_t batch,
                                   size_t theta, cudaStream_t st) {
    if (batch == 0) return cudaSuccess;
    if (m <= theta) return launch_mul_batch(out, a, b, m, batch, 0, st);
    struct Level {
        size_t m, h, count;
        uint64_t *A, *B;   // inputs of this level: [count][m]
        uint32_t *sa, *sb; // signs of this level's differences: [count]
    };
    std::vector<Level> lv;
    std::vector<void*> allocs;
    auto alloc = [&](size_t bytes) -> void* {
        void* p = nullptr;
        if (cudaMallocAsync(&p, bytes < 256 ? 256 : bytes, st) != cudaSuccess) return nullptr;
        allocs.push_back(p);
        return p;
    };
    cudaError_t e = cudaSuccess;
    auto cleanup = [&]() {
        for (void* p : allocs) cudaFreeAsync(p, st);
    };
    size_t cm = m, count = batch;
    const uint64_t* A = a;
    const uint64_t* B = b;
    // Descend: split every level until the base case.
    while (cm > theta) {
        const size_t h = (cm + 1) / 2;
        Level L{cm, h, count, nullptr, nullptr, nullptr, nullptr};
        uint64_t* nA = static_cast<uint64_t*>(alloc(3 * count * h * 8));
        uint64_t* nB = static_cast<uint64_t*>(alloc(3 * count * h * 8));
        L.sa = static_cast<uint32_t*>(alloc(count * 4));
        L.sb = static_cast<uint32_t*>(alloc(count * 4));
        if (!nA || !nB || !L.sa || !L.sb) {
            cleanup();
            return cudaErrorMemoryAllocation;
        }
        k_kara_split<<<blocks_for(count), 128, 0, st>>>(A, cm, h, count, nA, nA + count * h, nA + 2 * count * h,
                                                         L.sa);
        k_kara_split<<<blocks_for(count), 128, 0, st>>>(B, cm, h, count, nB, nB + count * h, nB + 2 * count * h,
                                                         L.sb);
        count_launch(2);
        lv.push_back(L);
        A = nA;
        B = nB;
        cm = h;
        count *= 3;
    }
    // Base case: one batched column multiply of all 3^L * batch leaves.
    uint64_t* P = static_cast<uint64_t*>(alloc(count * 2 * cm * 8));
    if (!P) {
        cleanup();
        return cudaErrorMemoryAllocation;
    }
    e = launch_mul_batch(P, A, B, cm, count, 0, st);
    // Ascend: combine level by level.
    for (size_t i = lv.size(); e == cudaSuccess && i-- > 0;) {
        const Level& L = lv[i];
        uint64_t* dst = i == 0 ? out : static_cast<uint64_t*>(alloc(L.count * 2 * L.m * 8));
        if (!dst) {
            e = cudaErrorMemoryAllocation;
            break;
        }
        k_kara_combine<<<blocks_for(L.count), 128, 0, st>>>(P, L.h, L.count, L.sa, L.sb, dst, L.m);
        count_launch();
        e = cudaGetLastError();
        P = dst;
    }
    cleanup();
    return e;
}

}  // namespace dotg
