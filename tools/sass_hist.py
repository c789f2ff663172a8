"""SASS opcode histograms of the product kernels (cuobjdump -sass of the built objects):
which pipes the hot kernels issue to, and the Blackwell mnemonics that are (or are not)
present - UTC*MMA / LDTM (tcgen05), UBLKCP / SYNCS (bulk copies, mbarriers), IMMA
(legacy mma.sync), IMAD.WIDE (the IMAD column MAC). Writes profiles/r02_sass_histograms.json."""
import collections
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "paper_2604_21566_b200", "csrc", "build")
KERNELS = {
    "addsub_batch.o": ["k_addsub_grouped", "k_addsub_timed", "k_addsub_ilf", "k_addsub_ilt", "k_addsub_il_tiny", "k_il_local", "k_il_finish"],
    "mul_batch.o": ["k_mul_kara16", "k_mul_regblk", "k_mul52_regs"],
    "mul_imma.o": ["k_mul_imma"],
    "mul_umma.o": ["k_mul_umma", "k_umma_tile_carries"],
    "addsub_long.o": ["k_long_local", "k_long_finish"],
}
KEY = re.compile(r"^(UTC\w*|LDTM|STTM|UBLKCP|UTMALDG|SYNCS|IMMA|HMMA|IMAD|IADD3|LDS|STS|LDG|STG|SHFL|VOTE|BAR|LOP3|SEL|DFMA|DADD)")


def main():
    out = {}
    for obj, names in KERNELS.items():
        sass = subprocess.run(["cuobjdump", "-sass", os.path.join(OBJ, obj)], capture_output=True, text=True).stdout
        funcs = re.split(r"\n\s+Function : ", sass)
        for f in funcs[1:]:
            mangled = f.split("\n", 1)[0].strip()
            demangled = subprocess.run(["c++filt", mangled], capture_output=True, text=True).stdout.strip()
            if not any(n in demangled for n in names):
                continue
            ops = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", f)
            full = collections.Counter(ops)
            base = collections.Counter(o.split(".")[0] for o in ops)
            short = re.sub(r"\(anonymous namespace\)::", "", demangled).replace("dotg::", "").split("(")[0]
            out[short] = {
                "instructions": sum(base.values()),
                "by_opcode": dict(base.most_common(20)),
                "imad_wide": sum(v for k, v in full.items() if k.startswith("IMAD.WIDE")),
                "tensor": {k: v for k, v in full.items() if k.startswith(("IMMA", "HMMA", "UTC", "LDTM", "STTM"))},
                "tcgen05_present": any(k.startswith(("UTC", "LDTM", "STTM")) for k in full),
                "bulk_copy_mbarrier": {k: v for k, v in full.items() if k.startswith(("UBLKCP", "SYNCS"))},
                "vector_256b_global": sum(v for k, v in full.items() if k.startswith(("LDG.E.ENL2.256", "STG.E.ENL2.256"))
                                          or ".256" in k),
            }
    path = os.path.join(ROOT, "profiles", "r02_sass_histograms.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    for k, v in out.items():
        print(f"{k[:70]:70s} {v['instructions']:6d} instr  tensor={v['tensor']}  tcgen05={v['tcgen05_present']}")


if __name__ == "__main__":
    main()
