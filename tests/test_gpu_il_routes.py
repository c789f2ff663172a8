"""Every interleaved add/sub route, forced one at a time, against the oracle (bit-exact).

The route for an interleaved [m][batch] problem is picked inside the library
(csrc/addsub_batch.cu il_route); DOTG_IL_MODE forces one, read once per process, so each
route runs in its own child: 2 thread per pair, 3 re-read segmented CTAs (k_addsub_il2),
4 two streaming passes, 5 streaming pass with in-CTA fix-up (k_addsub_ilf, in each of its
chunk / pairs-per-lane / double-buffering variants), 6 thread per pair fed by a bulk-copy
ring (k_addsub_ilt; odd batches fall back to thread per pair). Shapes cover ragged m, partial strips,
segments with no rows, in-place calls (out = a), and the carry-stress categories whose propagate runs cross
segment boundaries (the fix-up's rare multi-row branch)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, sys
sys.path.insert(0, ROOT + "/tests")
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2604_21566_b200 as dg
from helpers import CATEGORIES, Oracle, category
orc = Oracle()
bad = []
n = 0
for m, batch in SHAPES:
    rng = np.random.default_rng(9100 + 7 * m + batch)
    for cat in CATEGORIES:
        for op in ("add", "sub"):
            a, b = category(rng, cat, op, (batch, m))
            if cat == "random" and m > 12:  # a propagate run across segment boundaries
                lo, hi = 3, m - 2
                if op == "add":
                    a[::3, lo:hi] = np.uint64(0xFFFFFFFFFFFFFFFF); b[::3, lo:hi] = 0
                else:
                    a[::3, lo:hi] = b[::3, lo:hi]
            want, wf = orc.addsub_batch(op == "sub", a, b)
            ta = torch.from_numpy(np.ascontiguousarray(a.T).view(np.int64)).cuda()
            tb = torch.from_numpy(np.ascontiguousarray(b.T).view(np.int64)).cuda()
            out, fl = dg.addsub_batch(op == "sub", ta, tb, layout="interleaved")
            got = out.cpu().numpy().view(np.uint64).T
            gf = fl.cpu().numpy().view(np.uint32)
            n += 1
            if not (np.array_equal(got, want) and np.array_equal(gf, wf)):
                bad.append([m, batch, cat, op])
            # in place: out aliases a (every route reads a row before it rewrites it)
            dg.addsub_batch(op == "sub", ta, tb, out=ta, flags=fl, layout="interleaved")
            if not (np.array_equal(ta.cpu().numpy().view(np.uint64).T, want)
                    and np.array_equal(fl.cpu().numpy().view(np.uint32), wf)):
                bad.append([m, batch, cat, op, "in place"])
print(json.dumps({"cases": n, "bad": bad[:10]}))
'''.replace("ROOT", repr(ROOT))

SHAPES = [(1, 64), (2, 70), (3, 68), (5, 33), (16, 64), (33, 40), (64, 96), (100, 65), (128, 128), (200, 130), (256, 190),
          (257, 40), (512, 66), (777, 33), (1024, 64), (1500, 40), (2048, 6), (3000, 2)]

SETTINGS = {
    "tpp": {"DOTG_IL_MODE": "2"},
    "tpp_vp2": {"DOTG_IL_MODE": "2", "DOTG_TPP_VP": "2"},
    "tiny": {"DOTG_IL_MODE": "7"},
    "il2": {"DOTG_IL_MODE": "3"},
    "two_pass": {"DOTG_IL_MODE": "4"},
    "ilf": {"DOTG_IL_MODE": "5"},
    "ilf_ppl2": {"DOTG_IL_MODE": "5", "DOTG_ILF_PPL": "2"},
    "ilf_un8": {"DOTG_IL_MODE": "5", "DOTG_ILF_UN": "8", "DOTG_ILF_DB": "0"},
    "ilf_un16": {"DOTG_IL_MODE": "5", "DOTG_ILF_UN": "16", "DOTG_ILF_DB": "0"},
    "ilf_ppl2_single": {"DOTG_IL_MODE": "5", "DOTG_ILF_PPL": "2", "DOTG_ILF_DB": "0"},
    "ilf_wdiv4": {"DOTG_IL_MODE": "5", "DOTG_ILF_WDIV": "4"},
    "ilf_ppl4": {"DOTG_IL_MODE": "5", "DOTG_ILF_PPL": "4"},
    "ilf_g16": {"DOTG_IL_MODE": "5", "DOTG_ILF_G": "16"},
    "ilf_g8_ppl1": {"DOTG_IL_MODE": "5", "DOTG_ILF_G": "8", "DOTG_ILF_PPL": "1"},
    "ilf_ppl4_single": {"DOTG_IL_MODE": "5", "DOTG_ILF_PPL": "4", "DOTG_ILF_DB": "0"},
    "ilt": {"DOTG_IL_MODE": "6"},
    "ilt_p16_r8_s4": {"DOTG_IL_MODE": "6", "DOTG_ILT_P": "16", "DOTG_ILT_R": "8", "DOTG_ILT_STAGES": "4"},
    "ilt_p32_r8_s16": {"DOTG_IL_MODE": "6", "DOTG_ILT_P": "32", "DOTG_ILT_R": "8", "DOTG_ILT_STAGES": "16"},
    "ilt_p16_r32_s4": {"DOTG_IL_MODE": "6", "DOTG_ILT_P": "16", "DOTG_ILT_R": "32", "DOTG_ILT_STAGES": "4"},
    "ilt_p16_r32_s16": {"DOTG_IL_MODE": "6", "DOTG_ILT_P": "16", "DOTG_ILT_R": "32", "DOTG_ILT_STAGES": "16"},
    "ilt_p32_r32": {"DOTG_IL_MODE": "6", "DOTG_ILT_P": "32", "DOTG_ILT_R": "32"},
}


@pytest.mark.parametrize("name", sorted(SETTINGS))
def test_forced_route(cuda, name):
    env = {**os.environ, **SETTINGS[name]}
    code = CHILD.replace("SHAPES", repr(SHAPES))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, cwd=ROOT,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["cases"] > 0 and not res["bad"], (name, res)


# The automatic route at the sizes where it switches to k_addsub_ilt (48 <= m, batch >= 8192
# and even) and just past them: an odd batch (ilf), the smallest ilt batch, ragged m, boxes
# whose last stage is partial; and m <= 3 (k_addsub_il_tiny, batch % 4 == 0, else thread
# per pair) and m = 4 ... 7 (thread per pair).
AUTO_SHAPES = [(48, 8192), (64, 8193), (100, 8194), (130, 8192), (513, 8192), (47, 8192),
               (1, 4096), (2, 4100), (3, 4098), (3, 4097), (4, 4096), (7, 4098)]


def test_auto_route_at_ilt_sizes(cuda):
    code = CHILD.replace("SHAPES", repr(AUTO_SHAPES))
    env = {k: v for k, v in os.environ.items() if not k.startswith(("DOTG_IL", "DOTG_ILT", "DOTG_ILF"))}
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, cwd=ROOT,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["cases"] > 0 and not res["bad"], res
