// device.cuh - sm_100a device helpers shared by the limb kernels.
//
// Carry algebra (restated from the reference's Phase 4, addsub.cpp:61-79, generalised;
// SURVEY.md §8(a)). For one limb, add: s = a + b, g = s < a, p = (s == ~0);
// sub: s = a - b, g = a < b, p = (s == 0). g and p are never both set. For a group of
// lanes with masks G, P and carry-in cin, the carries INTO the lanes are
//     C = (((G << 1) | cin) + P) ^ P
// and the group's carry-out is bit n of ((G << 1) | cin) + P. The operator
// (G,P) o (G',P') = (G' | (P' & G), P & P') composes groups; it is associative.
#pragma once

#include <cstdint>

namespace dotg {

// ---------------------------------------------------------------------------
// Global memory: streaming vector loads/stores (sm_100 has 256-bit LDG/STG).
// Inputs are read once: no L1 allocation; 256-bit loads also mark L2 evict-first
// (ptxas accepts .L2::evict_first only on .v4.b64 / .v8.b32).
// ---------------------------------------------------------------------------
template <int V>
struct Vec {
    uint64_t x[V];
};

template <int V>
__device__ __forceinline__ void ld_stream(const uint64_t* p, uint64_t (&v)[V]) {
    if constexpr (V == 4) {
        asm volatile("ld.global.L1::no_allocate.L2::evict_first.v4.u64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3])
                     : "l"(p));
    } else if constexpr (V == 2) {
        asm volatile("ld.global.L1::no_allocate.v2.u64 {%0,%1}, [%2];"
                     : "=l"(v[0]), "=l"(v[1])
                     : "l"(p));
    } else {
        static_assert(V == 1, "V in {1,2,4}");
        asm volatile("ld.global.L1::no_allocate.u64 %0, [%1];" : "=l"(v[0]) : "l"(p));
    }
}

template <int V>
__device__ __forceinline__ void st_stream(uint64_t* p, const uint64_t (&v)[V]) {
    if constexpr (V == 4) {
        asm volatile("st.global.L1::no_allocate.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(v[0]),
                     "l"(v[1]), "l"(v[2]), "l"(v[3])
                     : "memory");
    } else if constexpr (V == 2) {
        asm volatile("st.global.L1::no_allocate.v2.u64 [%0], {%1,%2};" ::"l"(p), "l"(v[0]), "l"(v[1])
                     : "memory");
    } else {
        static_assert(V == 1, "V in {1,2,4}");
        asm volatile("st.global.L1::no_allocate.u64 [%0], %1;" ::"l"(p), "l"(v[0]) : "memory");
    }
}

// ---------------------------------------------------------------------------
// Limb-level phase 1 + phase 2 (generate / propagate extraction).
// ---------------------------------------------------------------------------
template <bool SUB>
__device__ __forceinline__ uint64_t lane_op(uint64_t a, uint64_t b, uint32_t& g, uint32_t& p) {
    if constexpr (SUB) {
        const uint64_t s = a - b;
        g = a < b;
        p = s == 0;
        return s;
    } else {
        const uint64_t s = a + b;
        g = s < a;
        p = s == ~0ull;
        return s;
    }
}

// The value a propagating limb takes in the output for a given carry-in.
template <bool SUB>
__device__ __forceinline__ uint64_t prop_value(uint32_t cin) {
    // add: s == ~0 -> ~0 + 0 = ~0, ~0 + 1 = 0; sub: s == 0 -> 0 - 0 = 0, 0 - 1 = ~0.
    if constexpr (SUB) return cin ? ~0ull : 0ull;
    else return cin ? 0ull : ~0ull;
}

template <bool SUB>
__device__ __forceinline__ uint64_t apply_carry(uint64_t s, uint32_t c) {
    if constexpr (SUB) return s - uint64_t(c);
    else return s + uint64_t(c);
}

// Fold V limbs of one super-lane into (G, P) (lowest limb first).
template <int V>
__device__ __forceinline__ void fold_gp(const uint32_t (&g)[V], const uint32_t (&p)[V], uint32_t& G,
                                        uint32_t& P) {
    G = g[0];
    P = p[0];
#pragma unroll
    for (int k = 1; k < V; ++k) {
        G = g[k] | (p[k] & G);
        P &= p[k];
    }
}

// Apply the super-lane carry-in c to its V limbs in place (phase 3 + 4 in one step:
// the carry entering limb k+1 is g_k | (p_k & c_k)).
template <bool SUB, int V>
__device__ __forceinline__ void apply_superlane(uint64_t (&s)[V], const uint32_t (&g)[V],
                                                const uint32_t (&p)[V], uint32_t c) {
#pragma unroll
    for (int k = 0; k < V; ++k) {
        const uint64_t v = apply_carry<SUB>(s[k], c);
        c = g[k] | (p[k] & c);
        s[k] = v;
    }
}

// 64-bit mask lookahead for one word of super-lanes with carry-in `cin` and the
// shifted-in generate bit `gin` (the previous word's top generate). Returns the
// carry-into mask; *cout = carry out of this 64-lane word.
__device__ __forceinline__ uint64_t lookahead64(uint64_t G, uint64_t P, uint32_t cin_add, uint32_t gin,
                                                uint32_t& cout) {
    // Y = (G << 1 | gin) + P + cin_add, computed with explicit carry-out.
    const uint64_t gs = (G << 1) | uint64_t(gin);
    const uint64_t t = gs + P;
    const uint32_t c1 = t < P;
    const uint64_t y = t + uint64_t(cin_add);
    const uint32_t c2 = y < t;
    cout = c1 | c2;
    return y ^ P;
}

// ---------------------------------------------------------------------------
// Bulk async copies (cp.async.bulk: the TMA engine without a tensor map) completing on
// shared-memory mbarriers. Source, destination and size must be 16-byte multiples.
// ---------------------------------------------------------------------------
namespace bulk {
__device__ __forceinline__ uint32_t saddr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(bar)) : "memory");
}
__device__ __forceinline__ void init_fence() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     saddr(dst)),
                 "l"(src), "r"(bytes), "r"(saddr(bar))
                 : "memory");
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(saddr(bar)),
        "r"(parity)
        : "memory");
}
// generic-proxy accesses of a buffer ordered before the async proxy's next writes to it
__device__ __forceinline__ void proxy_fence() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
}  // namespace bulk

}  // namespace dotg
