"""dotg-verify on a reference-format JSONL corpus (tests/golden/corpus_small.jsonl, made
by tests/golden/make_corpus.py with the reference's oracle): all cases match; a corrupted
corpus reports the mismatching case ids with exit code 1; malformed input exits 2
(the reference's dotarith verify behaviour, test_cli.cpp:142-165)."""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "tools", "build", "dotg-verify")
CORPUS = os.path.join(ROOT, "tests", "golden", "corpus_small.jsonl")


def run(*args):
    if not os.path.exists(TOOL):
        subprocess.run(["make", "-C", os.path.join(ROOT, "tools")], check=True)
    return subprocess.run([TOOL, *args], capture_output=True, text=True, timeout=300)


def test_corpus_verifies(cuda):
    r = run("verify", CORPUS)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "216 cases, 0 mismatches" in r.stdout


def test_corrupted_corpus_reports_ids(cuda, tmp_path):
    lines = open(CORPUS).read().splitlines()
    for i in (3, 100, 200):  # flip the last hex digit of the expected value
        head, exp_tail = lines[i].split('"expected":"')
        val, rest = exp_tail.split('"', 1)
        val = val[:-1] + ("0" if val[-1] != "0" else "1")
        lines[i] = head + '"expected":"' + val + '"' + rest
    bad = tmp_path / "bad.jsonl"
    bad.write_text("\n".join(lines) + "\n")
    r = run("verify", str(bad))
    assert r.returncode == 1
    assert "3 mismatches" in r.stdout
    for i in (3, 100, 200):
        assert f"mismatch at case {i}" in r.stdout


def test_malformed_input(cuda, tmp_path):
    p = tmp_path / "broken.jsonl"
    p.write_text('{"op":"add","bits":100,"category":"random","a":"1","b":"2","expected":"3","flag":0}\n')
    r = run("verify", str(p))
    assert r.returncode == 2 and "parse error at line 1" in r.stderr
    assert run("verify", str(tmp_path / "missing.jsonl")).returncode == 2
    assert run("verify", CORPUS, "--width", "16").returncode == 2


def _hex_limbs(text, m):
    v = int(text, 16)
    return np.array([(v >> (64 * i)) & ((1 << 64) - 1) for i in range(m)], dtype=np.uint64)


@pytest.mark.parametrize("width", ["8", "4", "2", "scalar"])
def test_stats_line_matches_reference(cuda, ref, width):
    """The AddSubStats line (dotarith verify prints it for the vector add/sub kernels,
    bench.cpp:160-161) equals the reference's own counters summed over the corpus."""
    import json

    w = 0 if width == "scalar" else int(width)
    chunks = fires = 0
    for line in open(CORPUS):
        c = json.loads(line)
        if c["op"] == "mul":
            continue
        m = c["bits"] // 64
        _, _, ch, fi = ref.words(c["op"] == "sub", _hex_limbs(c["a"], m), _hex_limbs(c["b"], m), w)
        chunks += ch
        fires += fi
    r = run("verify", CORPUS, "--width", width)
    assert r.returncode == 0, r.stdout + r.stderr
    assert f"chunks {chunks}, phase4 triggers {fires} (rate {fires / chunks:.6f})" in r.stdout, r.stdout


def test_bench_rows_and_gate(cuda, tmp_path):
    """dotg-verify bench (dotarith bench over a corpus): one row per (op, bits) group with
    device and host-buffer ns/op and the Phase-4 rate; a group that fails verification
    gets no row and the exit code is 1 (bench.cpp:201-204, dotarith_cli.cpp:120-131)."""
    import json

    groups = {(c["op"], c["bits"]) for c in map(json.loads, open(CORPUS))}
    csv = tmp_path / "rows.csv"
    r = run("bench", CORPUS, "--reps", "3", "--csv", str(csv))
    assert r.returncode == 0, r.stdout + r.stderr
    rows = [ln.split() for ln in r.stdout.splitlines()[1:] if ln.split() and ln.split()[0] in ("add", "sub", "mul")]
    assert {(x[0], int(x[1])) for x in rows} == groups
    for x in rows:
        assert float(x[5]) > 0 and float(x[7]) > 0 and x[-1] == "cuda-events"
    lines = csv.read_text().splitlines()
    assert lines[0].startswith("op,bits,w,kernel") and len(lines) == len(groups) + 1
    # corrupt one add case: its group loses its row, the others still print
    src = open(CORPUS).read().splitlines()
    i = next(k for k, ln in enumerate(src) if json.loads(ln)["op"] == "add")
    c = json.loads(src[i])
    head, tail = src[i].split('"expected":"')
    val, rest = tail.split('"', 1)
    src[i] = head + '"expected":"' + val[:-1] + ("0" if val[-1] != "0" else "1") + '"' + rest
    bad = tmp_path / "bad.jsonl"
    bad.write_text("\n".join(src) + "\n")
    r = run("bench", str(bad), "--reps", "2")
    assert r.returncode == 1 and "failed verification" in r.stderr
    rows = [ln.split() for ln in r.stdout.splitlines()[1:] if ln.split() and ln.split()[0] in ("add", "sub", "mul")]
    assert ("add", c["bits"]) not in {(x[0], int(x[1])) for x in rows} and len(rows) == len(groups) - 1
