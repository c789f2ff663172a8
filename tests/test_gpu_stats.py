"""Acceptance criterion 4 (acceptance.cpp:157-170): the carry census for k = 1..12 equals
its closed forms (2^k max-sum pairs, 2^(k-1) (2^k - 1) carry pairs; carry_census,
oracle.cpp:65-78, here cross-checked by brute force for small k) and the Monte-Carlo
carry frequency of 10^7 random 64-bit additions is 0.5 +/- 0.001 - counted on the device,
through the API and through `dotg-verify stats` (dotarith stats)."""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_census_and_monte_carlo(cuda):
    import paper_2604_21566_b200 as dg
    from paper_2604_21566_b200 import api

    for k in range(1, 7):
        n = 1 << k
        x, y = np.meshgrid(np.arange(n), np.arange(n))
        s = x + y
        assert api.carry_census(k) == (int((s == n - 1).sum()), int((s >= n).sum()))
    rep = api.run_stats(12, 10_000_000, 1)
    assert all(r["match"] for r in rep["census"]) and len(rep["census"]) == 12
    assert rep["mc_within_tolerance"], rep["mc_carry_freq"]
    assert api.carry_census(16) == (1 << 16, (1 << 15) * ((1 << 16) - 1))
    for bad in (0, 17):
        with pytest.raises(dg.InvalidArgument):
            api.carry_census(bad)


def test_verify_tool_stats(cuda):
    tool = os.path.join(ROOT, "tools", "build", "dotg-verify")
    if not os.path.exists(tool):
        subprocess.run(["make", "-C", os.path.join(ROOT, "tools")], check=True)
    r = subprocess.run([tool, "stats"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count(" yes") == 13 and "monte-carlo: 10000000 samples" in r.stdout
    assert subprocess.run([tool, "stats", "--k-max", "17"], capture_output=True, timeout=60).returncode == 2
