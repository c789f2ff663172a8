"""dotg-verify's input handling on CPU (no device call happens before parsing succeeds):
usage errors, unknown width, missing file and malformed JSONL lines exit 2 with the
reference's messages (dotarith_cli.cpp:57-82, testgen.cpp:211-255)."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "tools", "build", "dotg-verify")
CORPUS = os.path.join(ROOT, "tests", "golden", "corpus_small.jsonl")


def run(*args):
    if not os.path.exists(TOOL):
        subprocess.run(["make", "-C", os.path.join(ROOT, "tools")], check=True, capture_output=True)
    return subprocess.run([TOOL, *args], capture_output=True, text=True, timeout=120)


def test_usage_and_width():
    assert run().returncode == 2
    assert run("gen", CORPUS).returncode == 2
    r = run("bench", CORPUS, "--reps", "0")
    assert r.returncode == 2 and "at least one repetition" in r.stderr
    r = run("bench", CORPUS, "--warmup", "3")
    assert r.returncode == 2 and "unknown option" in r.stderr
    r = run("verify", CORPUS, "--reps", "3")  # bench-only option
    assert r.returncode == 2 and "unknown option" in r.stderr
    assert run("bench", CORPUS, "--width").returncode == 2
    r = run("verify", CORPUS, "--width", "16")
    assert r.returncode == 2 and "unknown width" in r.stderr


def test_missing_file(tmp_path):
    r = run("verify", str(tmp_path / "missing.jsonl"))
    assert r.returncode == 2 and "cannot open" in r.stderr


def test_malformed_lines(tmp_path):
    bad = [
        ('{"op":"add","bits":100,"category":"random","a":"1","b":"2","expected":"3","flag":0}', "multiple of 64"),
        ('{"op":"pow","bits":64,"category":"random","a":"1","b":"2","expected":"3","flag":0}', "unknown op"),
        ('{"op":"add","bits":64,"category":"random","a":"1g","b":"2","expected":"3","flag":0}', "invalid character"),
        ('{"op":"add","bits":64,"category":"random","a":"1","b":"2","expected":"3","flag":2}', "flag must be"),
        ('{"op":"add","bits":64,"a":"1","b":"2","expected":"3","flag":0}', "parse error"),
        ('{"op":"add","bits":64,"category":"random","a":"1" "b":"2"}', "expected ',' or '}'"),
        ('{"op":"add","bits":64,"category":"random","a":"1ffffffffffffffff","b":"2","expected":"3","flag":0}',
         "wider than the declared bits"),
    ]
    for i, (line, msg) in enumerate(bad):
        p = tmp_path / f"bad{i}.jsonl"
        p.write_text('{"op":"add","bits":64,"category":"random","a":"1","b":"2","expected":"3","flag":0}\n' + line + "\n")
        r = run("verify", str(p))
        assert r.returncode == 2, (line, r.stdout, r.stderr)
        assert "parse error at line 2" in r.stderr and msg in r.stderr, (line, r.stderr)
