"""Write a small corpus in the reference's JSONL exchange format (src/testgen.cpp:195-209:
op, bits, category, a, b, expected as minimal lowercase hex, flag for add/sub; compact
one-object-per-line JSON in that field order) with expected values from the reference's
own oracle (oracle/_ref/libdotref.so). The reference's `dotarith gen` cannot be built here
(CLI11 and nlohmann json are not vendored), so this script stands in for it.

    python tests/golden/make_corpus.py   ->  tests/golden/corpus_small.jsonl
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from helpers import Reference, category  # noqa: E402

CATS = {"random": "random", "full_propagation": "full-propagation", "maxed_limbs": "maxed-limbs",
        "zero_limbs": "zero-limbs", "frequent_carries": "frequent-carries", "frequent_borrows": "frequent-borrows"}


def to_hex(limbs):
    v = 0
    for x in reversed([int(t) for t in limbs]):
        v = (v << 64) | x
    return format(v, "x")


def main():
    ref = Reference.load()
    if ref is None:
        raise SystemExit("oracle/_ref/libdotref.so missing: run `make -C oracle ref` first")
    rng = np.random.default_rng(0xC0BB5)
    lines = []
    for bits in (512, 1024, 4096):
        m = bits // 64
        for op in ("add", "sub", "mul"):
            for cat, name in CATS.items():
                a, b = category(rng, cat, op, (4, m))
                for i in range(4):
                    if op == "mul":
                        exp = ref.oracle_mul(a[i], b[i])
                        rec = {"op": op, "bits": bits, "category": name, "a": to_hex(a[i]), "b": to_hex(b[i]),
                               "expected": to_hex(exp) if exp.size else "0"}
                    else:
                        out, flag = ref.oracle_addsub(op == "sub", a[i], b[i])
                        rec = {"op": op, "bits": bits, "category": name, "a": to_hex(a[i]), "b": to_hex(b[i]),
                               "expected": to_hex(out), "flag": int(flag)}
                    lines.append(json.dumps(rec, separators=(",", ":")))
    path = os.path.join(HERE, "corpus_small.jsonl")
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")
    print(f"wrote {path}: {len(lines)} cases")


if __name__ == "__main__":
    main()
