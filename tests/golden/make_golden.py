"""Generate golden vectors from the UNMODIFIED reference (oracle/_ref/libdotref.so).

Run in the build container (where /root/reference exists):
    make -C oracle ref && python tests/golden/make_golden.py

Inputs are numpy PCG64 draws (fixed seeds) in the reference tests' shapes
(test_addsub.cpp:28-40 spiky limbs; testgen.cpp:87-128 categories). Expected values
come from the reference's own DoT path (span-form dot_add_words / dot_sub_words at
Width::w8, dot_mul_words, add_w_limbs / sub_w_limbs) and are cross-checked at
generation time against the reference's oracle (oracle_add / oracle_sub / oracle_mul).
The fixtures are committed so the GPU box (which has no /root/reference) can replay them.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from helpers import CATEGORIES, Reference, category, spiky, uniform  # noqa: E402

ADDSUB_SIZES = [1, 2, 3, 4, 5, 7, 8, 9, 13, 16, 17, 31, 32, 33, 64, 65, 128, 256]
MUL_SIZES = [1, 2, 3, 4, 5, 6, 7, 8, 12, 16, 24, 32, 33, 48, 64]
PER_CAT = 6


def main():
    ref = Reference.load()
    if ref is None:
        raise SystemExit("oracle/_ref/libdotref.so missing: run `make -C oracle ref` first")
    rng = np.random.default_rng(0x601DE7)
    out = {}
    for m in ADDSUB_SIZES:
        A, Bv = [], []
        for cat in CATEGORIES:
            for op in ("add", "sub"):
                a, b = category(rng, cat, op, (PER_CAT // 2, m))
                A.append(a)
                Bv.append(b)
        a = np.concatenate(A)
        b = np.concatenate(Bv)
        n = a.shape[0]
        res = {k: [] for k in ("add_out", "add_flag", "sub_out", "sub_flag", "add_p4", "sub_p4")}
        for i in range(n):
            for sub, key in ((0, "add"), (1, "sub")):
                o, c, chunks, fires = ref.words(sub, a[i], b[i], 8)
                oo, oc = ref.oracle_addsub(sub, a[i], b[i])
                assert np.array_equal(o, oo) and c == oc, "reference DoT path disagrees with its oracle"
                res[key + "_out"].append(o)
                res[key + "_flag"].append(c)
                res[key + "_p4"].append(fires)
        out[f"addsub_m{m}_a"] = a
        out[f"addsub_m{m}_b"] = b
        for k, v in res.items():
            out[f"addsub_m{m}_{k}"] = np.array(v, dtype=np.uint64 if k.endswith("out") else np.uint32)
    for m in MUL_SIZES:
        A, Bv = [], []
        for cat in ("random", "full_propagation", "spiky", "maxed_limbs"):
            a, b = category(rng, cat, "mul", (4, m))
            A.append(a)
            Bv.append(b)
        a = np.concatenate(A)
        b = np.concatenate(Bv)
        prods = []
        for i in range(a.shape[0]):
            p = ref.mul_words(a[i], b[i])
            o = ref.oracle_mul(a[i], b[i])
            assert p.size == 2 * m
            assert np.array_equal(p[: o.size], o) and not p[o.size:].any()
            prods.append(p)
        out[f"mul_m{m}_a"] = a
        out[f"mul_m{m}_b"] = b
        out[f"mul_m{m}_out"] = np.array(prods, dtype=np.uint64)
    # chunk level (add_w_limbs / sub_w_limbs, addsub.hpp:86-89)
    for w in range(1, 9):
        a = spiky(rng, (100, w))
        b = spiky(rng, (100, w))
        cin = rng.integers(0, 2, size=100).astype(np.uint32)
        for sub, key in ((0, "add"), (1, "sub")):
            sums, co, p4 = [], [], []
            for i in range(100):
                s, c, f = ref.chunk(sub, a[i], b[i], int(cin[i]), w)
                sums.append(s)
                co.append(c)
                p4.append(int(f))
            out[f"chunk_w{w}_{key}_sums"] = np.array(sums, dtype=np.uint64)
            out[f"chunk_w{w}_{key}_carry"] = np.array(co, dtype=np.uint32)
            out[f"chunk_w{w}_{key}_p4"] = np.array(p4, dtype=np.uint32)
        out[f"chunk_w{w}_a"] = a
        out[f"chunk_w{w}_b"] = b
        out[f"chunk_w{w}_cin"] = cin
    # 52-bit radix routes (mul.hpp:73-85) and the 64<->52 repacking (limbs.hpp:111-117)
    mask52 = np.uint64((1 << 52) - 1)
    for m in (1, 2, 3, 5, 8, 20):
        a = uniform(rng, (12, m)) & mask52
        b = uniform(rng, (12, m)) & mask52
        a[0] = mask52
        b[0] = mask52
        out["mul52_m%d_a" % m] = a
        out["mul52_m%d_b" % m] = b
        out["mul52_m%d_out" % m] = np.array([ref.mul2("dotref_mul_words52", a[i], b[i], 2 * m) for i in range(12)],
                                            dtype=np.uint64)
    a5 = uniform(rng, (20, 5)) & mask52
    b5 = uniform(rng, (20, 5)) & mask52
    out["mul5x5_a"], out["mul5x5_b"] = a5, b5
    out["mul5x5_out"] = np.array([ref.mul2("dotref_mul_5x5", a5[i], b5[i], 10) for i in range(20)], dtype=np.uint64)
    a4, b4 = uniform(rng, (20, 4)), uniform(rng, (20, 4))
    a4[0] = ~np.uint64(0)
    b4[0] = ~np.uint64(0)
    out["mul4x4_a"], out["mul4x4_b"] = a4, b4
    out["mul4x4_out"] = np.array([ref.mul2("dotref_mul_4x4", a4[i], b4[i], 8) for i in range(20)], dtype=np.uint64)
    for m in (1, 3, 4, 7, 13):
        x = uniform(rng, m)
        p = ref.repack("dotref_pack_64_to_52", x)
        out["pack_m%d_in" % m] = x
        out["pack_m%d_out" % m] = p
        out["pack_m%d_back" % m] = ref.repack("dotref_unpack_52_to_64", p)
    meta = {"dispatch_note_w8": ref.dispatch_note(8)}
    out["meta_dispatch_note_w8"] = np.frombuffer(meta["dispatch_note_w8"].encode(), dtype=np.uint8)
    path = os.path.join(HERE, "reference_vectors.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(out)} arrays)")


if __name__ == "__main__":
    main()
