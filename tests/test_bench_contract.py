"""bench.py contract checks that run without a GPU: the reference arm (CPU) prints one
JSON line with the driver's keys, on the same metric/config as our arm."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "impl"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GB/s"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    import bench

    assert d["metric"] == bench.METRIC
    assert d["config"]["workload"] == bench.c2_config()["workload"]
    assert d["steps"] == 1 and d["warmup"] >= 3  # W >= 3 enforced


def test_reference_arm_two_ranks_gloo():
    """The N > 1 launch shape of the reference arm on CPU (torchrun, gloo, world size 2):
    rank 0 alone works and prints ONE JSON line, the other rank exits 0."""
    env = {**os.environ, "MASTER_ADDR": "127.0.0.1"}
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", "29573", "bench.py", "--impl", "reference",
                        "--gpus", "2", "--steps", "1", "--warmup", "3"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0


def test_strong_scaling_slices():
    """Rank slices of the named batches partition them exactly (no pair lost or repeated),
    and the rotation count keeps > L2 bytes between reuses of a copy."""
    import bench

    for B in (1 << 20, 1 << 18, 65536, 16384, 1000, 7):
        for world in (1, 2, 3, 4, 8):
            spans = [bench.rank_slice(B, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == B
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            assert max(hi - lo for lo, hi in spans) - min(hi - lo for lo, hi in spans) <= 1
    for nbytes in (1 << 20, 67 << 20, 537 << 20):
        k = bench.rotations(nbytes)
        assert k >= 1 and (k == 1 or k * nbytes >= 2 * bench.L2_BYTES)
