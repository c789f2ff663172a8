"""Golden vectors for the column-pipeline STAGES (A10-A13), from the UNMODIFIED reference
(oracle/_ref/libdotref.so: gather_columns, compute_partials, align_and_reduce, carry_pass,
mul.hpp:32-67, mul.cpp:12-90).

Run in the build container (where /root/reference exists):
    make -C oracle ref && python tests/golden/make_column_golden.py

Inputs restate the reference's own stage tests (tests/test_mul.cpp):
  * gather / partials / reduce over m in {1..8, 12, 16, 33, 64} with uniform, all-ones and
    52-bit limbs (test_mul.cpp:183-217: lone pair, column sums vs a double loop);
  * carry_pass over 1..12 raw u128 columns per case at k = 64 and k = 52
    (test_mul.cpp:229-241), plus the ~u128 stress and residual cases (242-252): [~0] at
    k = 52 (3 limbs out), [~0, ~0] at k = 64, runs of ~0 columns.
Every reference output is also cross-checked here against the C restatement
(oracle/dot_oracle.c) before it is written. Output: tests/golden/column_vectors.npz.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from helpers import MAX, Oracle, Reference, uniform  # noqa: E402

M52 = np.uint64((1 << 52) - 1)


def main():
    ref = Reference.load()
    if ref is None:
        raise SystemExit("oracle/_ref/libdotref.so missing: run `make -C oracle ref` first")
    orc = Oracle()
    rng = np.random.default_rng(0xC011)
    out = {}
    sizes = [1, 2, 3, 4, 5, 6, 7, 8, 12, 16, 33, 64]
    for m in sizes:
        cases = []
        for kind in ("uniform", "ones", "r52", "lone"):
            if kind == "uniform":
                a, b = uniform(rng, m), uniform(rng, m)
            elif kind == "ones":
                a, b = np.full(m, MAX), np.full(m, MAX)
            elif kind == "r52":
                a, b = uniform(rng, m) & M52, uniform(rng, m) & M52
            else:  # test_mul.cpp:183-196: one nonzero pair a[i] = b[j] = 2^63
                a, b = np.zeros(m, np.uint64), np.zeros(m, np.uint64)
                a[int(rng.integers(0, m))] = np.uint64(1 << 63)
                b[int(rng.integers(0, m))] = np.uint64(1 << 63)
            cases.append((a, b))
        A = np.stack([c[0] for c in cases])
        B = np.stack([c[1] for c in cases])
        for k in (64, 52):
            if k == 52:  # 52-bit radix needs limbs < 2^52 (check_limbs): the r52 / lone rows
                rows = [2]
            else:
                rows = list(range(len(cases)))
            MA, MB, LO, HI, COLS, OUTS, NOUT = [], [], [], [], [], [], []
            for i in rows:
                ma, mb = ref.gather_columns(A[i], B[i])
                oma, omb = orc.gather_columns(A[i], B[i])
                assert np.array_equal(ma, oma) and np.array_equal(mb, omb)
                lo, hi = ref.compute_partials(ma, mb, k)
                olo, ohi = orc.compute_partials(ma, mb, k)
                assert np.array_equal(lo, olo) and np.array_equal(hi, ohi)
                cols = ref.align_and_reduce(lo, hi, m)
                assert np.array_equal(cols, orc.align_and_reduce(lo, hi, m))
                res = ref.carry_pass(cols, k)
                assert np.array_equal(res, orc.carry_pass(cols, k))
                assert res.size == 2 * m  # pipeline columns never leave a residual
                MA.append(ma), MB.append(mb), LO.append(lo), HI.append(hi), COLS.append(cols), OUTS.append(res)
            key = f"m{m}_k{k}"
            out[key + "_a"] = A[rows]
            out[key + "_b"] = B[rows]
            out[key + "_ma"] = np.stack(MA)
            out[key + "_mb"] = np.stack(MB)
            out[key + "_plo"] = np.stack(LO)
            out[key + "_phi"] = np.stack(HI)
            out[key + "_cols"] = np.stack(COLS)
            out[key + "_out"] = np.stack(OUTS)
    # carry_pass over raw u128 columns (test_mul.cpp:229-252)
    for k in (64, 52):
        cases = []
        for _ in range(200):
            n = int(rng.integers(1, 13))
            cases.append(uniform(rng, (n, 2)))
        full = np.full((1, 2), MAX)
        cases += [full, np.full((2, 2), MAX), np.full((5, 2), MAX),
                  np.array([[0, 1 << 63], [MAX, MAX], [0, 0], [MAX, MAX]], np.uint64),
                  np.zeros((10, 2), np.uint64)]
        flat_cols, offs, flat_out, outoffs = [], [0], [], [0]
        for cols in cases:
            res = ref.carry_pass(cols, k)
            assert np.array_equal(res, orc.carry_pass(cols, k))
            flat_cols.append(cols)
            offs.append(offs[-1] + cols.shape[0])
            flat_out.append(res)
            outoffs.append(outoffs[-1] + res.size)
        out[f"carry_k{k}_cols"] = np.concatenate(flat_cols)
        out[f"carry_k{k}_col_offsets"] = np.array(offs, np.int64)
        out[f"carry_k{k}_out"] = np.concatenate(flat_out)
        out[f"carry_k{k}_out_offsets"] = np.array(outoffs, np.int64)
    out["sizes"] = np.array(sizes, np.int64)
    path = os.path.join(HERE, "column_vectors.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(out)} arrays)")


if __name__ == "__main__":
    main()
