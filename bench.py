#!/usr/bin/env python
"""bench.py - B200 limb arithmetic (DigitsOnTurbo hot path) benchmark.

Headline workload (BASELINE.json configs[1], "C2"): the carry-stress add/sub sweep -
(m, B) in (4, 2^20), (16, 2^18), (64, 2^16), (256, 2^14); each limb all-ones with p=1/2
else uniform, 1% of pairs forced to a full-length carry chain; sub swaps pairs so a >= b.
One step = batched add at all four sizes, then batched sub at all four sizes, through the
device C ABI (one dotg_addsub_grouped launch, replayed as a CUDA graph). Metric:
algorithmic GB/s (24m + 4 bytes per pair-op), roofline = measured HBM copy bandwidth.

The same JSON line reports every other config under "configs", each with its own
roofline, e2e (host C ABI, pinned buffers, copies timed) and reference CPU baseline:
C1 (4096-bit add/sub), C3/C4 (1024/4096-bit mul, products/s vs the measured IMAD.WIDE
roofline), C5 (one 2^30-limb add/sub), plus the interleaved layout.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--only C1,C3,C4,C5,IL,R52,WIDE] [--no-secondary]

N > 1: launched by torch.distributed.run, one rank per GPU. Strong scaling: rank r runs
the contiguous slice [B*r/N, B*(r+1)/N) of every named batch (no collective on the data
path; C5 is split by limb range and exchanges 8 bytes per rank through
dotg_add_words_sharded); value = the whole named workload / max-over-ranks time. The
weak-scaling figure (full sweep on every rank) is reported as "weak_scaling".
--impl reference times the reference's own CPU implementation (oracle/_ref/libdotref.so:
span-form dot_add_words / dot_sub_words at Width::w8 and dot_mul_words) on all host
cores; under torchrun only rank 0 works.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK_GBS = 6650.0  # B200_PROFILING.md fallback, used only without MEASURED_PEAKS.json
IMAD_WIDE_PER_CLK_SM = 32.0  # measured: profiles/r01_imad_peak.json (cc_chain_products)
IMMA_U8_MACS_PER_CLK_SM = 2048.0  # measured: profiles/r01_imma_peak.json (mma.sync m16n8k32 u8)
IMMA_ROUTE_M = (32, 64, 128)  # m the library multiplies on the tensor pipe (mul_batch.cu)
C2_SIZES = [(4, 1 << 20), (16, 1 << 18), (64, 1 << 16), (256, 1 << 14)]
METRIC = "add/sub GB/s vs HBM peak (C2 carry-stress sweep, 4/16/64/256 limbs)"
DATA = ("synthetic (seeded splitmix64, BASELINE.json configs[1] distribution: limb all-ones p=0.5 else uniform, "
        "1% forced full carry chains, sub swapped to a>=b)")


C2_WORKING_SET = sum(4 * B * m * 8 for m, B in C2_SIZES)  # distinct input bytes per step (a, b, sa, sb)


def c2_config(ungrouped=False):
    """The workload description, identical in both arms (ours and --impl reference)."""
    return {"workload": "C2 carry-stress add+sub sweep (BASELINE.json configs[1])",
            "sizes_m_batch": C2_SIZES, "layout": "row-major [batch][m] (reference Limbs layout)",
            "step": ("8 launches: add at 4 sizes then sub at 4 sizes" if ungrouped else
                     "add at 4 sizes + sub at 4 sizes (GPU: one dotg_addsub_grouped launch)"),
            "l2": (f"inputs larger than L2: each step reads {C2_WORKING_SET / 1e6:.0f} MB of distinct inputs "
                   "(126 MB L2), every buffer touched once per step")}


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------
def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j.get("hbm_gbs", HBM_FALLBACK_GBS)), "measured", float(j.get("sm_max_mhz", 1965.0))
    return HBM_FALLBACK_GBS, "fallback", 1965.0


def traffic_table():
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled during the timed region:
    NVML polled every 5 ms from a thread (plus one sample at start and stop, so even a
    millisecond-long region is covered); `nvidia-smi -lms` only where NVML is missing."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0, period_ms=5):
        self.index, self.period_ms = index, period_ms
        self.proc = None
        self.nvml = None
        self.lines = []
        self.samples = []  # (sm_mhz, max_mhz, reasons set)
        self._stop = threading.Event()

    def _nvml_sample(self):
        n = self.nvml
        sm = n.nvmlDeviceGetClockInfo(self.h, n.NVML_CLOCK_SM)
        mx = n.nvmlDeviceGetMaxClockInfo(self.h, n.NVML_CLOCK_SM)
        bits = n.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        masks = (n.nvmlClocksEventReasonHwSlowdown, n.nvmlClocksEventReasonHwThermalSlowdown,
                 n.nvmlClocksEventReasonSwThermalSlowdown, n.nvmlClocksEventReasonSwPowerCap)
        self.samples.append((float(sm), float(mx), {nm for nm, b in zip(self.NAMES, masks) if bits & b}))

    def _poll(self):
        while not self._stop.is_set():
            try:
                self._nvml_sample()
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(self.period_ms / 1000.0)

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self._nvml_sample()
            threading.Thread(target=self._poll, daemon=True).start()
            return
        except Exception:  # noqa: BLE001
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms=50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.nvml is not None:
            try:
                self._nvml_sample()
            except Exception:  # noqa: BLE001
                pass
            self._stop.set()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            for ln in self.lines:
                parts = [x.strip() for x in ln.split(",")]
                if len(parts) < 6:
                    continue
                try:
                    rs = {n for n, v in zip(self.NAMES, parts[2:6]) if v.lower().startswith("active")}
                    self.samples.append((float(parts[0]), float(parts[1]), rs))
                except ValueError:
                    continue
        sm = [x[0] for x in self.samples]
        mx = [x[1] for x in self.samples]
        reasons = set().union(*[x[2] for x in self.samples]) if self.samples else set()
        load = [v for v in sm if v > 400] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml" if self.nvml is not None else "nvidia-smi"}


# ---------------------------------------------------------------------------
# reference CPU arm (oracle/_ref/libdotref.so, or the oracle port without it)
# ---------------------------------------------------------------------------
class CpuRef:
    def __init__(self):
        ref_so = os.path.join(ROOT, "oracle", "_ref", "libdotref.so")
        orc_so = os.path.join(ROOT, "oracle", "liboracle.so")
        self.threads = os.cpu_count() or 1
        if os.path.exists(ref_so):
            self.kind = "reference"
            L = ctypes.CDLL(ref_so)
            L.dotref_batch.restype = ctypes.c_int
            L.dotref_batch.argtypes = [ctypes.c_int, ctypes.c_int] + [ctypes.c_void_p] * 4 + [ctypes.c_size_t] * 2 + [
                ctypes.c_int]
            L.dotref_dispatch_note.restype = ctypes.c_char_p
            L.dotref_dispatch_note.argtypes = [ctypes.c_int]
            self.note = L.dotref_dispatch_note(8).decode()
        elif os.path.exists(orc_so):
            self.kind = "port"
            L = ctypes.CDLL(orc_so)
            self.threads = 1
            self.note = "oracle port (scalar)"
        else:
            raise SystemExit("neither oracle/_ref/libdotref.so nor oracle/liboracle.so is built")
        self.L = L

    def words(self, sub, out, a, b):
        """One long number, span form (dot_add_words / dot_sub_words, Width::w8, single
        thread: the reference's carry chain is serial). Returns the carry/borrow."""
        P = lambda x: ctypes.c_void_p(x.ctypes.data)  # noqa: E731
        if self.kind == "reference":
            L = self.L
            L.dotref_words.restype = ctypes.c_int
            L.dotref_words.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                                       ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                                       ctypes.c_void_p, ctypes.c_void_p]
            c = L.dotref_words(int(sub), P(out), out.size, P(a), a.size, P(b), b.size, 8, None, None)
            if c < 0:
                raise RuntimeError("reference words failed")
            return int(c)
        self.L.dotor_words.restype = ctypes.c_uint
        self.L.dotor_words.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_size_t, ctypes.c_uint, ctypes.c_void_p, ctypes.c_void_p]
        return int(self.L.dotor_words(int(sub), P(out), P(a), P(b), a.size, 8, None, None))

    def run(self, op, a, b, out, flags):
        """op 0 add, 1 sub, 2 mul on [B, m] numpy uint64 arrays (reference DoT path)."""
        B, m = a.shape
        P = lambda x: None if x is None else ctypes.c_void_p(x.ctypes.data)  # noqa: E731
        if self.kind == "reference":
            rc = self.L.dotref_batch(op, 0, P(out), P(a), P(b), P(flags), m, B, self.threads)
            if rc != 0:
                raise RuntimeError("reference batch failed")
        else:
            if op == 2:
                self.L.dotor_mul_batch(P(out), P(a), P(b), ctypes.c_size_t(m), ctypes.c_size_t(B))
            else:
                self.L.dotor_addsub_batch(op, P(out), P(a), P(b), P(flags), ctypes.c_size_t(m), ctypes.c_size_t(B))


def host_c2_inputs():
    """C2 inputs on the host via the oracle's splitmix64 twin (same values as the device
    generator in paper_2604_21566_b200/workloads.py)."""
    import numpy as np

    L = ctypes.CDLL(os.path.join(ROOT, "oracle", "liboracle.so"))
    L.dotor_fill_splitmix64.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_uint64]

    def fill(n, seed, off):
        x = np.empty(n, np.uint64)
        L.dotor_fill_splitmix64(ctypes.c_void_p(x.ctypes.data), n, seed, off)
        return x

    MAX = np.uint64(0xFFFFFFFFFFFFFFFF)
    sets = []
    for m, B in C2_SIZES:
        s, n = 0xC2 + m, B * m

        def operand(off):
            v = fill(n, s, off)
            sel = fill(n, s, off + n)
            v[(sel & np.uint64(1)) == 1] = MAX
            return v.reshape(B, m)

        a, b = operand(0), operand(2 * n)
        a[::100] = MAX
        b[::100] = 0
        b[::100, 0] = 1
        ne = a != b
        idx = (m - 1) - np.argmax(ne[:, ::-1], axis=1)
        r = np.arange(B)
        lt = (ne.any(axis=1) & (a[r, idx] < b[r, idx]))[:, None]
        sa, sb = np.where(lt, b, a), np.where(lt, a, b)
        sets.append((m, B, a, b, np.ascontiguousarray(sa), np.ascontiguousarray(sb)))
    return sets


def c2_bytes():
    return sum(2 * (B * (24 * m + 4)) for m, B in C2_SIZES)


def cpu_c2_measure(cpu, sets, min_seconds=3.0, max_reps=200):
    """Time the reference on the full C2 step (add + sub at all sizes), repeated until
    min_seconds of CPU work; returns (GB/s, reps, seconds)."""
    import numpy as np

    outs = [(np.empty_like(a), np.empty(B, np.uint32)) for (m, B, a, b, sa, sb) in sets]
    reps, t0 = 0, time.perf_counter()
    while True:
        for (m, B, a, b, sa, sb), (o, f) in zip(sets, outs):
            cpu.run(0, a, b, o, f)
        for (m, B, a, b, sa, sb), (o, f) in zip(sets, outs):
            cpu.run(1, sa, sb, o, f)
        reps += 1
        dt = time.perf_counter() - t0
        if dt >= min_seconds or reps >= max_reps:
            break
    return c2_bytes() * reps / dt / 1e9, reps, dt


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    cpu = CpuRef()
    sets = host_c2_inputs()
    import numpy as np

    outs = [(np.empty_like(a), np.empty(B, np.uint32)) for (m, B, a, b, sa, sb) in sets]

    def step():
        for (m, B, a, b, sa, sb), (o, f) in zip(sets, outs):
            cpu.run(0, a, b, o, f)
        for (m, B, a, b, sa, sb), (o, f) in zip(sets, outs):
            cpu.run(1, sa, sb, o, f)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    gbs = c2_bytes() * args.steps / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs,
        "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u64", "data": DATA,
        "config": c2_config(),
        "sharding": "reference CPU path on rank 0's host (all host threads); other ranks idle",
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": cpu.threads, "kind": cpu.kind,
                         "sample": f"full C2 step (add+sub, 4 sizes) x {args.steps} steps; route {cpu.note}"},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
class Launcher:
    """Pre-bound ctypes calls of the device C ABI (keeps Python off the critical path)."""

    def __init__(self, torch, lib, stream):
        self.torch, self.lib = torch, lib
        self.stream = ctypes.c_void_p(stream.cuda_stream)

    def addsub(self, sub, out, a, b, flags, m, B):
        fn = self.lib.dotg_sub_batch if sub else self.lib.dotg_add_batch
        args = (ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()),
                ctypes.c_void_p(flags.data_ptr()), m, B, 0, self.stream)
        return lambda: fn(*args)

    def grouped(self, problems):
        """problems: list of (sub, out, a, b, flags, m, B) -> one dotg_addsub_grouped call."""
        from paper_2604_21566_b200._lib import AddSubProblem

        arr = (AddSubProblem * len(problems))()
        for i, (sub, out, a, b, flags, m, B) in enumerate(problems):
            arr[i] = AddSubProblem(int(sub), 0, out.data_ptr(), a.data_ptr(), b.data_ptr(), flags.data_ptr(), m, B)
        fn, n, st = self.lib.dotg_addsub_grouped, len(problems), self.stream
        self._keep = arr
        return lambda: fn(arr, n, st)

    def mul(self, out, a, b, m, B):
        fn = self.lib.dotg_mul_batch
        args = (ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()), m, B,
                0, self.stream)
        return lambda: fn(*args)


def device_index():
    """This rank's GPU: LOCAL_RANK, or 0 for every rank in the shared-GPU rehearsal."""
    return 0 if os.environ.get("DOTG_BENCH_SHARED_GPU") == "1" else env_int("LOCAL_RANK", 0)


def reduce_scalar(dist, x, op):
    """max / min of a host scalar over ranks (a CUDA tensor for NCCL, a CPU one for gloo)."""
    import torch

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.MIN)
    return float(t.item())


def timed_steps(torch, dist, world, stream, calls, steps, warmup):
    """Run `calls` (zero-arg callables, one device launch sequence each) per step:
    W warm-up steps, then K timed steps bracketed by barrier + synchronize and timed
    with CUDA events on the launching stream (max over ranks). A second pass of K steps
    records an event pair around every call to get per-kernel durations (the roofline's
    launch duration) without slowing the lean timed loop. Returns
    (ms_per_step, [mean ms per call])."""
    for _ in range(warmup):
        for c in calls:
            rc = c()
            if rc != 0:
                raise RuntimeError(f"dotg call failed rc={rc}")
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(steps):
        for c in calls:
            c()
    t1.record(stream)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    total_ms = t0.elapsed_time(t1)
    if dist is not None and world > 1:
        total_ms = reduce_scalar(dist, total_ms, "max")
    evs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in calls]
           for _ in range(steps)]
    for s in range(steps):
        for i, c in enumerate(calls):
            evs[s][i][0].record(stream)
            c()
            evs[s][i][1].record(stream)
    torch.cuda.synchronize()
    per_call = [sum(evs[s][i][0].elapsed_time(evs[s][i][1]) for s in range(steps)) / steps for i in range(len(calls))]
    return total_ms / steps, per_call


L2_BYTES = 126 * 1000 * 1000  # B200 L2 (126 MB): inputs per timed step must exceed it


def rank_slice(B, rank, world):
    """Contiguous pair range [lo, hi) of the named batch that `rank` processes (strong
    scaling: the batch partitioned into G contiguous slices)."""
    return B * rank // world, B * (rank + 1) // world


def rotations(input_bytes):
    """How many distinct copies of a per-rank input set to rotate through so that the
    bytes read between two uses of the same copy exceed the L2 (timing rule: inputs
    larger than L2 between timed iterations)."""
    return max(1, -(-2 * L2_BYTES // max(1, input_bytes)))


def make_rotating(fns):
    """One zero-arg callable that runs fns[0], fns[1], ... in turn (one per step)."""
    state = {"i": 0}

    def call():
        f = fns[state["i"] % len(fns)]
        state["i"] += 1
        return f()

    return call


def capture_graph(torch, dg, lib, stream, make_call):
    """Capture make_call(launcher)() once into a CUDA graph; returns (replay_fn,
    kernels per replay) or (None, None) when capture is unavailable."""
    try:
        cap = torch.cuda.Stream()
        cap.wait_stream(stream)
        call = make_call(Launcher(torch, lib, cap))
        with torch.cuda.stream(cap):
            assert call() == 0
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        n0 = dg.kernel_launches()
        with torch.cuda.graph(graph, stream=cap):
            call()
        nk = dg.kernel_launches() - n0
        torch.cuda.synchronize()
        return (lambda: (graph.replay(), 0)[1]), nk, graph
    except Exception as e:  # noqa: BLE001
        print(f"graph capture unavailable ({e}); direct launches", file=sys.stderr)
        return None, None, None


def hbm_roofline(alg_bytes, launch_s, peak, kernel, peak_kind="measured (MEASURED_PEAKS.json hbm_gbs)",
                 traffic=None, **extra):
    achieved = alg_bytes / launch_s / 1e9
    r = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
         "traffic": traffic, "kernel": kernel, "algorithmic_bytes_per_launch": alg_bytes,
         "launch_us_avg": launch_s * 1e6, "peak_kind": peak_kind}
    r.update(extra)
    return r


# tcgen05.mma kind::i8 dense rate (tools/umma_i8_probe.cu, profiles/r02_umma_i8_probe.jsonl: N = 128 / 256)
UMMA_U8_MACS_PER_CLK_SM = 8192
# dotg_mul_batch on the mma.sync Karatsuba route before the tcgen05 kernel (profiles/r02_umma_wide_variants.txt)
WIDE_PRIOR_US = {(1024, 1024): 223.8, (2048, 256): 210.0, (4096, 64): 206.6}


def per_launch_us(torch, dg, lib, stream, make_calls, reps=4):
    """Device time of ONE launch when launches run back to back (the GPU never waits for
    the host): the calls make_calls(launcher) returns - one per rotating input set - are
    captured `reps` times into one CUDA graph; per launch = graph time / launches, CUDA
    events on the launching stream, best of 3 replays. (Bracketing a single launch with
    events from Python also times the host's launch submission when the GPU is idle -
    ~6 us on a ~17 us kernel.)"""
    fn, nk, graph = capture_graph(torch, dg, lib, stream,
                                  lambda Lc: (lambda cs=make_calls(Lc): [c() for _ in range(reps) for c in cs][-1]))
    if fn is None:
        return None
    n = reps * len(make_calls(Launcher(torch, lib, stream)))
    fn()
    torch.cuda.synchronize()
    best = None
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) * 1e3 / n
        best = t if best is None else min(best, t)
    del graph
    return best


def pinned_like(torch, t):
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    return h


def run_ours(args, rank, world, dist):
    import torch

    import paper_2604_21566_b200 as dg
    from paper_2604_21566_b200 import workloads as W

    lib = dg.lib()  # raises if libdotg.so is missing: no fallback
    torch.cuda.set_device(device_index())
    hbm_peak, peak_kind, sm_max = peaks()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    stream = torch.cuda.current_stream()
    L = Launcher(torch, lib, stream)
    if args.only:
        res = run_secondary(args, torch, dg, W, L, stream, rank, world, dist, hbm_peak, sm_max, sms)
        if rank == 0:
            print(json.dumps({"only": args.only, "configs": res}), flush=True)
        return 0

    # ---- headline: C2 sweep, device-resident ----
    bufs = []
    for m, B in C2_SIZES:
        a, b, sa, sb = W.c2_inputs(m, B)
        bufs.append(dict(m=m, B=B, a=a, b=b, sa=sa, sb=sb, oa=torch.empty_like(a), os=torch.empty_like(a),
                         fa=torch.empty(B, dtype=torch.int32, device="cuda"),
                         fs=torch.empty(B, dtype=torch.int32, device="cuda")))
    probs = [(False, x["oa"], x["a"], x["b"], x["fa"], x["m"], x["B"]) for x in bufs]
    probs += [(True, x["os"], x["sa"], x["sb"], x["fs"], x["m"], x["B"]) for x in bufs]
    call_bytes = [x["B"] * (24 * x["m"] + 4) for x in bufs] * 2
    full_step_bytes = sum(call_bytes)
    assert full_step_bytes == c2_bytes()

    # This rank's share of every batch (strong scaling: the named batches split into G
    # contiguous slices, no collective). At N = 1 the slice is the whole batch. With small
    # slices several copies rotate so every step still reads more than the L2.
    def slice_probs(copy):
        out = []
        for (sub, o, a_, b_, f, m, B), x in zip(probs, bufs * 2):
            lo, hi = rank_slice(B, rank, world)
            if copy == 0:
                out.append((sub, o[lo:hi], a_[lo:hi], b_[lo:hi], f[lo:hi], m, hi - lo))
            else:
                out.append((sub, torch.empty_like(o[lo:hi]), a_[lo:hi].clone(), b_[lo:hi].clone(),
                            torch.empty_like(f[lo:hi]), m, hi - lo))
        return out

    my_pairs = [rank_slice(B, rank, world) for m, B in C2_SIZES]
    my_bytes = sum(2 * (hi - lo) * (24 * m + 4) for (m, B), (lo, hi) in zip(C2_SIZES, my_pairs))
    my_inputs = sum(2 * 2 * (hi - lo) * m * 8 for (m, B), (lo, hi) in zip(C2_SIZES, my_pairs))
    nrot = rotations(my_inputs) if world > 1 else 1
    sets = [slice_probs(i) for i in range(nrot)]
    single_calls = [L.addsub(*q) for q in sets[0]]
    graph_launches = None
    graphs = []
    if args.ungrouped:
        calls = [make_rotating([(lambda ps=ps: [L.addsub(*q)() for q in ps][-1]) for ps in sets])]
    elif args.no_graph:
        calls = [make_rotating([L.grouped(ps) for ps in sets])]
    else:
        replays = []
        for ps in sets:
            fn, nk, g = capture_graph(torch, dg, lib, stream, lambda Lc, ps=ps: Lc.grouped(ps))
            if fn is None:
                replays = None
                break
            replays.append(fn)
            graphs.append(g)
            graph_launches = nk
        calls = [make_rotating(replays)] if replays else [make_rotating([L.grouped(ps) for ps in sets])]
    working_set = sum(4 * x["a"].numel() * 8 for x in bufs)  # distinct inputs read per full step (a, b, sa, sb)

    sampler = ClockSampler(device_index())
    sampler.start()
    time.sleep(0.2)
    launches0 = dg.kernel_launches()
    ms_step, per_call = timed_steps(torch, dist if world > 1 else None, world, stream, calls, args.steps,
                                    args.warmup)
    # launches inside the lean timed region (the event pass repeats it once more); graph
    # replays do not pass the library's launch counter: launches per captured step x steps
    launches = (dg.kernel_launches() - launches0 - args.warmup * len(calls)) // 2
    if graph_launches is not None:
        launches = graph_launches * args.steps
    clocks = sampler.stop()
    # value = the whole named sweep (all ranks' slices together) / max-over-ranks step time
    value = full_step_bytes / (ms_step * 1e-3) / 1e9
    achieved = my_bytes / (ms_step * 1e-3) / 1e9  # this rank's kernel: its bytes per launch / launch time
    weak = None
    if world > 1:
        # weak scaling (extra key): every rank runs the FULL sweep on its own GPU
        fn, nk, g = capture_graph(torch, dg, lib, stream, lambda Lc: Lc.grouped(probs))
        graphs.append(g)
        wcalls = [fn] if fn is not None else [L.grouped(probs)]
        wms, _ = timed_steps(torch, dist, world, stream, wcalls, args.steps, args.warmup)
        weak = {"value": full_step_bytes * world / (wms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": wms,
                "per_rank": "the full C2 sweep on every rank (no collective)"}
    # one size alone per launch: dotg_add_batch / dotg_sub_batch of this rank's slice,
    # back to back over 3 rotating copies of the inputs (> L2 between reuses)
    per_size = {}
    for i, x in enumerate(bufs):
        lo, hi = my_pairs[i]
        bts = (hi - lo) * (24 * x["m"] + 4)
        row = {}
        for op, (o, a_, b_, f) in (("add", (x["oa"], x["a"], x["b"], x["fa"])),
                                   ("sub", (x["os"], x["sa"], x["sb"], x["fs"]))):
            copies = [(o[lo:hi], a_[lo:hi], b_[lo:hi], f[lo:hi])]
            copies += [(torch.empty_like(o[lo:hi]), a_[lo:hi].clone(), b_[lo:hi].clone(), torch.empty_like(f[lo:hi]))
                       for _ in range(max(2, rotations(2 * (hi - lo) * x["m"] * 8)) - 1)]
            us = per_launch_us(torch, dg, lib, stream,
                               lambda Lc, cp=copies, sub=op == "sub": [Lc.addsub(sub, *c_, x["m"], hi - lo)
                                                                      for c_ in cp])
            del copies
            if us is not None:
                row.update({f"{op}_gbs": bts / (us * 1e-6) / 1e9, f"{op}_us": us,
                            f"{op}_frac": bts / (us * 1e-6) / 1e9 / hbm_peak})
        row["note"] = ("one dotg_add_batch / dotg_sub_batch launch of this size alone, launches back to back "
                       "over rotating input copies (CUDA graph, events on the stream)")
        per_size[f"m{x['m']}"] = row
    traffic = traffic_table().get("C2_per_launch_bytes_grouped" if not args.ungrouped else "C2_per_launch_bytes")
    # the same byte mix without carries: a plain 2-read / 1-write streaming add measured
    # live (tools/stream_peak.cu) - the practical ceiling for this kernel's traffic
    mix_peak = None
    sp = os.path.join(ROOT, "tools", "build", "stream_peak")
    if os.path.exists(sp) and rank == 0 and world == 1:
        try:
            r = subprocess.run([sp], capture_output=True, text=True, timeout=120)
            probe = json.loads(r.stdout)
            mix_peak = {"GBps": probe["add_2r1w"]["GBps"], "frac": achieved / probe["add_2r1w"]["GBps"],
                        "copy_1r1w_GBps": probe["copy_1r1w"]["GBps"], "read_GBps": probe["read_2r"]["GBps"],
                        "source": "tools/stream_peak.cu: out = a + b, 256-bit ld/st, 805 MB, best of 20"}
        except Exception as e:  # noqa: BLE001
            mix_peak = {"error": str(e)[:200]}
    # stress level of the sweep: AddSubStats counters of the reference's
    # w8 chunking, derived on the device from the step's own inputs and outputs
    stress = {}
    if world == 1:
        ctr = torch.zeros(2, dtype=torch.int64, device="cuda")
        for x in bufs:
            row = {}
            for sub, o, a_, b_ in ((0, x["oa"], x["a"], x["b"]), (1, x["os"], x["sa"], x["sb"])):
                ctr.zero_()
                rc = lib.dotg_addsub_stats(sub, ctypes.c_void_p(o.data_ptr()), ctypes.c_void_p(a_.data_ptr()),
                                           ctypes.c_void_p(b_.data_ptr()), x["m"], x["B"], 0, 8,
                                           ctypes.c_void_p(ctr.data_ptr()), ctypes.c_void_p(stream.cuda_stream))
                if rc == 0:
                    c = ctr.cpu().tolist()
                    row["sub" if sub else "add"] = {"chunks": c[0], "phase4_triggers": c[1],
                                                    "phase4_fraction": c[1] / max(1, c[0])}
            stress[f"m{x['m']}"] = row
    # phase split (the reference's collect_ticks pass, bench.cpp:227-247): %clock64 laps
    # of the timed team kernel over the same inputs, in AddSubStats buckets
    phase_split = {}
    if world == 1 and not args.no_phase:
        for x in bufs:
            row = {}
            for op, (a_, b_) in (("add", (x["a"], x["b"])), ("sub", (x["sa"], x["sb"]))):
                try:
                    r = dg.addsub_phase_ticks(op == "sub", a_, b_)
                    row[op] = {"pct": {k: round(v, 2) for k, v in r["pct"].items()},
                               "carry_to_add_ratio": r["carry_to_add_ratio"]}
                except Exception as e:  # noqa: BLE001
                    row[op] = {"error": str(e)[:200]}
            phase_split[f"m{x['m']}"] = row
        phase_split["unit"] = ("share of SM-clock cycles per warp task (timed team kernel, laps at phase "
                               "boundaries); reference (PAPER.md:754-761, EMR 512-bit add): load 18.7 / add 13.8 / "
                               "carry_gen 25.8 / carry_add 20.7 / store 21.0 %, carry-to-add 4.9 random")

    # ---- e2e: this rank's share through the host-buffer C ABI (pinned host arrays) ----
    e2e = None
    if not args.no_e2e:
        from paper_2604_21566_b200._lib import AddSubProblem

        hsets = []
        for x, (lo, hi) in zip(bufs, my_pairs):
            hs = {k: pinned_like(torch, x[k][lo:hi]) for k in ("a", "b", "sa", "sb")}
            hs["o"] = torch.empty(hs["a"].shape, dtype=torch.int64, pin_memory=True)
            hs["os"] = torch.empty(hs["a"].shape, dtype=torch.int64, pin_memory=True)
            hs["f"] = torch.empty(hi - lo, dtype=torch.int32, pin_memory=True)
            hs["fs"] = torch.empty(hi - lo, dtype=torch.int32, pin_memory=True)
            hsets.append((x["m"], hi - lo, hs))
        hprobs = (AddSubProblem * 8)()
        for i, (m, B, hs) in enumerate(hsets):
            hprobs[i] = AddSubProblem(0, 0, hs["o"].data_ptr(), hs["a"].data_ptr(), hs["b"].data_ptr(),
                                      hs["f"].data_ptr(), m, B)
            hprobs[4 + i] = AddSubProblem(1, 0, hs["os"].data_ptr(), hs["sa"].data_ptr(), hs["sb"].data_ptr(),
                                          hs["fs"].data_ptr(), m, B)

        def e2e_step():
            rc = lib.dotg_addsub_grouped_host(hprobs, 8)
            assert rc == 0, lib.dotg_last_error()

        e2e_step()
        # correctness spot check of the e2e path against the device result
        lo, hi = my_pairs[-1]
        assert torch.equal(hsets[-1][2]["os"], bufs[-1]["os"][lo:hi].cpu()), "e2e result mismatch"
        lo, hi = my_pairs[0]
        assert torch.equal(hsets[0][2]["o"], bufs[0]["oa"][lo:hi].cpu()), "e2e result mismatch"
        e_steps = max(3, min(args.steps, 20))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e_steps):
            e2e_step()
        dt = time.perf_counter() - t0
        if world > 1:
            dt = reduce_scalar(dist, dt, "max")
        h2d = sum(2 * 2 * B * m * 8 for m, B, _ in hsets)
        d2h = sum(2 * (B * m * 8 + 4 * B) for m, B, _ in hsets)
        e2e = {"value": full_step_bytes * e_steps / dt / 1e9, "unit": "GB/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "steps": e_steps,
               "api": "dotg_addsub_grouped_host: the 8 host problems through one H2D / kernel / D2H stream "
                      "pipeline (pinned host buffers)",
               "bound": "PCIe: one integer op per byte moved; the kernel-only path runs ~85x faster than the "
                        "link can feed it"}
        # the PCIe ceiling of this step: the same bytes moved with no kernels at all
        # (uploads on one stream, downloads concurrently on another, 24 MB chunks)
        try:
            xa = torch.empty(h2d // 8, dtype=torch.int64, pin_memory=True)
            xb = torch.empty(d2h // 8, dtype=torch.int64, pin_memory=True)
            ya, yb = torch.empty_like(xa, device="cuda"), torch.empty_like(xb, device="cuda")
            s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
            ch = 3 << 20

            def xfer():
                with torch.cuda.stream(s1):
                    for i in range(0, xa.numel(), ch):
                        ya[i:i + ch].copy_(xa[i:i + ch], non_blocking=True)
                with torch.cuda.stream(s2):
                    for i in range(0, xb.numel(), ch):
                        xb[i:i + ch].copy_(yb[i:i + ch], non_blocking=True)
                torch.cuda.synchronize()

            xfer()
            t0 = time.perf_counter()
            for _ in range(5):
                xfer()
            tx = (time.perf_counter() - t0) / 5
            e2e["transfer_only_GBps"] = my_bytes / tx / 1e9
            e2e["frac_of_transfer_only"] = e2e["value"] / world / e2e["transfer_only_GBps"]
            del xa, xb, ya, yb
        except Exception as ex:  # noqa: BLE001
            e2e["transfer_only_GBps"] = None
            e2e["transfer_note"] = str(ex)[:200]
        del hsets

    # ---- CPU baseline (rank 0, N = 1 only) ----
    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = CpuRef()
            hsets_cpu = host_c2_inputs()
            gbs, reps, dt = cpu_c2_measure(cpu, hsets_cpu, min_seconds=args.cpu_seconds)
            cpu_baseline = {"value": gbs, "unit": "GB/s", "cores": cpu.threads, "kind": cpu.kind,
                            "sample": f"full C2 step (add+sub at 4 sizes, {c2_bytes() / 1e6:.0f} MB) x {reps} reps "
                                      f"({dt:.1f} s), span-form dot_add_words/dot_sub_words route {cpu.note}"}
            del hsets_cpu
        except Exception as e:  # noqa: BLE001
            cpu_baseline = {"value": None, "unit": "GB/s", "cores": 0, "kind": "unavailable", "sample": str(e)}

    # per-call latency of the drop-in span form on ONE 4096-bit number (how the reference's
    # own callers use dot_add_words, e.g. Karatsuba's add_at, mul.cpp:169-174), beside the
    # reference's span call on one core; and one device-resident call (batch of 1)
    latency = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            import numpy as np

            m1 = 64
            ha1 = np.ascontiguousarray(bufs[2]["a"][0].cpu().numpy().view(np.uint64))
            hb1 = np.ascontiguousarray(bufs[2]["b"][0].cpu().numpy().view(np.uint64))
            ho1 = np.empty(m1, np.uint64)
            c1 = ctypes.c_uint32(0)
            P1 = lambda x: ctypes.c_void_p(x.ctypes.data)  # noqa: E731
            for _ in range(20):
                lib.dotg_add_words_host(P1(ho1), P1(ha1), P1(hb1), m1, ctypes.byref(c1))
            n1 = 2000
            t0 = time.perf_counter()
            for _ in range(n1):
                lib.dotg_add_words_host(P1(ho1), P1(ha1), P1(hb1), m1, ctypes.byref(c1))
            host_us = (time.perf_counter() - t0) / n1 * 1e6
            d_o = torch.empty(m1, dtype=torch.int64, device="cuda")
            d_c = torch.empty(1, dtype=torch.int32, device="cuda")
            da1, db1 = bufs[2]["a"][0], bufs[2]["b"][0]
            dcall = lambda: lib.dotg_add_batch(ctypes.c_void_p(d_o.data_ptr()), ctypes.c_void_p(da1.data_ptr()),  # noqa: E731
                                               ctypes.c_void_p(db1.data_ptr()), ctypes.c_void_p(d_c.data_ptr()), m1,
                                               1, 0, L.stream)
            for _ in range(20):
                dcall()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(n1):
                dcall()
            torch.cuda.synchronize()
            dev_us = (time.perf_counter() - t0) / n1 * 1e6
            cpu = CpuRef()
            ref_ns = None
            if cpu.kind == "reference":
                co = np.empty(m1, np.uint64)
                cpu.words(0, co, ha1, hb1)
                t0 = time.perf_counter()
                for _ in range(n1):
                    cpu.words(0, co, ha1, hb1)
                ref_ns = (time.perf_counter() - t0) / n1 * 1e9
            latency = {"m": m1, "dropin_host_span_us": host_us, "device_call_us": dev_us,
                       "reference_span_ns_incl_ctypes": ref_ns,
                       "note": "one 4096-bit add per call: host span form (operands through mapped pinned memory, one launch, one sync) and the "
                               "device-pointer C ABI back to back (launch-bound), vs the reference's span call "
                               "through ctypes on one core (~53 ns natively, profiles/r01_cpu_table.json). Single "
                               "small numbers belong on the CPU or in a batch / CUDA graph."}
        except Exception as e:  # noqa: BLE001
            latency = {"error": str(e)[:200]}

    # free the headline buffers before the secondary configs
    del bufs, calls, single_calls, sets, graphs
    torch.cuda.synchronize()
    torch.cuda.empty_cache()

    secondary = {}
    if not args.no_secondary:
        secondary = run_secondary(args, torch, dg, W, L, stream, rank, world, dist, hbm_peak, sm_max, sms)

    line = {
        "metric": METRIC,
        "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": DATA,
        "config": c2_config(args.ungrouped),
        "sharding": (f"rank r of {world} runs pairs [B*r/{world}, B*(r+1)/{world}) of every C2 batch (contiguous "
                     "slices, no collective on the data path); value = the whole named sweep / max-over-ranks step "
                     f"time; {nrot} rotating copies of each rank's slice keep > L2 bytes per step"
                     if world > 1 else "one GPU runs the whole named sweep"),
        "roofline": hbm_roofline(my_bytes, ms_step * 1e-3, hbm_peak,
                                 "k_addsub_grouped (persistent batched add/sub, warp-ballot lookahead)",
                                 peak_kind=f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)", traffic=traffic,
                                 per_size=per_size, mix_peak=mix_peak,
                                 traffic_steady=(traffic_table().get("C2_steady_per_launch_bytes")
                                                 if world == 1 and not args.ungrouped else None),
                                 traffic_steady_note=("ncu --cache-control none over consecutive launches of this "
                                                      "kernel in the bench command: DRAM read + write per launch in "
                                                      "steady state (profiles/r02_ncu_headline_steady.csv); "
                                                      "traffic is one --set full capture with caches flushed"),
                                 note="achieved = this rank's algorithmic bytes per step launch / the launch's "
                                      "CUDA-event time on the launching stream (one launch per step)"),
        "cpu_baseline": cpu_baseline,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "launch_mode": ("one CUDA-graph replay per step (the captured dotg_addsub_grouped launch)"
                        if graph_launches is not None else "direct C-ABI launches"),
        "clocks": clocks,
        "carry_stress": stress,
        "phase_split": phase_split,
        "call_latency": latency,
        "configs": secondary,
    }
    if weak is not None:
        line["weak_scaling"] = weak
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def run_secondary(args, torch, dg, W, L, stream, rank, world, dist, hbm_peak, sm_max, sms):
    import numpy as np

    out = {}
    steps = max(3, min(args.steps, 50))
    warm = max(3, args.warmup)
    dd = dist if world > 1 else None
    lib = dg.lib()
    rank0 = rank == 0
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731

    def want(k):
        return not args.only or k in args.only.split(",")

    def host_u64(t):
        return t.cpu().numpy().view(np.uint64)

    # ---------------- C1: 4096-bit add + sub, B = 65536 ----------------
    if want("C1"):
        B, m = W.C1["batch"], 64
        lo, hi = rank_slice(B, rank, world)
        nb = hi - lo
        byts = nb * (24 * m + 4)  # one op over this rank's slice
        # 3 rotating input sets (>= 2 x L2 of inputs between reuses of a set)
        nset = max(3, rotations(2 * 2 * nb * m * 8))
        sets = []
        for r in range(nset):
            a = W.fill(B * m, 0xC1 + 17 * r, 0).view(-1, m)[lo:hi].clone()
            b = W.fill(B * m, 0xC1 + 17 * r, 1 << 40).view(-1, m)[lo:hi].clone()
            sa, sb = W.swap_for_sub(a, b)
            sets.append(dict(a=a, b=b, sa=sa, sb=sb, o=torch.empty_like(a), o2=torch.empty_like(a),
                             f=torch.empty(nb, dtype=torch.int32, device="cuda"),
                             f2=torch.empty(nb, dtype=torch.int32, device="cuda")))
        calls = [L.grouped([(False, x["o"], x["a"], x["b"], x["f"], m, nb), (True, x["o2"], x["sa"], x["sb"], x["f2"],
                                                                             m, nb)]) for x in sets]
        ms, per = timed_steps(torch, dd, world, stream, calls, steps, warm)
        x0 = sets[0]
        # back-to-back launch times (graph over the rotating sets): add+sub grouped, add, sub
        us_g = per_launch_us(torch, dg, lib, stream, lambda Lc: [
            Lc.grouped([(False, x["o"], x["a"], x["b"], x["f"], m, nb), (True, x["o2"], x["sa"], x["sb"], x["f2"], m,
                                                                         nb)]) for x in sets])
        per1 = [per_launch_us(torch, dg, lib, stream, lambda Lc, sub=sub: [
            Lc.addsub(sub, x["o2" if sub else "o"], x["sa" if sub else "a"], x["sb" if sub else "b"],
                      x["f2" if sub else "f"], m, nb) for x in sets]) * 1e-3 for sub in (False, True)]
        launch_s = (us_g * 1e-6) if us_g is not None else statistics.mean(per) * 1e-3
        c1 = {"metric": "add/sub GB/s (4096-bit, B=65536)", "value": B * (24 * m + 4) * 2 * len(calls) / (ms * 1e-3)
              / 1e9, "unit": "GB/s",
              "step": f"{len(calls)} rotating input sets; per set add + sub in one dotg_addsub_grouped launch",
              "roofline": hbm_roofline(2 * byts, launch_s, hbm_peak,
                                       "k_addsub_grouped (add + sub of one C1 set, 2 problems, one launch)",
                                       traffic=traffic_table().get("C1_per_launch_bytes") if world == 1 else None,
                                       single_launch={"add_gbs": byts / (per1[0] * 1e-3) / 1e9,
                                                      "sub_gbs": byts / (per1[1] * 1e-3) / 1e9,
                                                      "add_frac": byts / (per1[0] * 1e-3) / 1e9 / hbm_peak,
                                                      "sub_frac": byts / (per1[1] * 1e-3) / 1e9 / hbm_peak,
                                                      "add_us": per1[0] * 1e3, "sub_us": per1[1] * 1e3}),
              "frac_hbm_back_to_back": 2 * byts * len(calls) / (ms * 1e-3) / 1e9 / hbm_peak}
        if not args.no_e2e:
            from paper_2604_21566_b200._lib import AddSubProblem

            hs = {k: pinned_like(torch, x0[k]) for k in ("a", "b", "sa", "sb")}
            ho = torch.empty_like(hs["a"], pin_memory=True)
            ho2 = torch.empty_like(hs["a"], pin_memory=True)
            hf = torch.empty(nb, dtype=torch.int32, pin_memory=True)
            hf2 = torch.empty(nb, dtype=torch.int32, pin_memory=True)
            hp = (AddSubProblem * 2)()
            hp[0] = AddSubProblem(0, 0, ho.data_ptr(), hs["a"].data_ptr(), hs["b"].data_ptr(), hf.data_ptr(), m, nb)
            hp[1] = AddSubProblem(1, 0, ho2.data_ptr(), hs["sa"].data_ptr(), hs["sb"].data_ptr(), hf2.data_ptr(), m,
                                  nb)
            assert lib.dotg_addsub_grouped_host(hp, 2) == 0, lib.dotg_last_error()
            torch.cuda.synchronize()
            assert torch.equal(ho, x0["o"].cpu()) and torch.equal(ho2, x0["o2"].cpu()), "C1 e2e mismatch"
            reps = 10
            if dd is not None:
                dist.barrier()
            t0 = time.perf_counter()
            for _ in range(reps):
                lib.dotg_addsub_grouped_host(hp, 2)
            dt = (time.perf_counter() - t0) / reps
            if dd is not None:
                dt = reduce_scalar(dist, dt, "max")
            c1["e2e"] = {"value": B * (24 * m + 4) * 2 / dt / 1e9, "unit": "GB/s",
                         "h2d_bytes_per_step": 4 * nb * m * 8, "d2h_bytes_per_step": 2 * (nb * m * 8 + 4 * nb),
                         "api": "dotg_addsub_grouped_host (add + sub of the whole batch, pinned host buffers)"}
            if rank0 and world == 1 and not args.no_cpu:
                try:
                    cpu = CpuRef()
                    ha, hb = hs["a"].numpy().view(np.uint64), hs["b"].numpy().view(np.uint64)
                    hsa, hsb = hs["sa"].numpy().view(np.uint64), hs["sb"].numpy().view(np.uint64)
                    co, cf = np.empty_like(ha), np.empty(nb, np.uint32)
                    co2, cf2 = np.empty_like(ha), np.empty(nb, np.uint32)
                    cpu.run(0, ha, hb, co, cf)
                    cpu.run(1, hsa, hsb, co2, cf2)
                    assert np.array_equal(co, ho.numpy().view(np.uint64)) and np.array_equal(
                        co2, ho2.numpy().view(np.uint64)), "C1 cpu/gpu mismatch"
                    assert np.array_equal(cf, hf.numpy().view(np.uint32)) and np.array_equal(
                        cf2, hf2.numpy().view(np.uint32)), "C1 cpu/gpu flag mismatch"
                    reps, t0 = 0, time.perf_counter()
                    while True:
                        cpu.run(0, ha, hb, co, cf)
                        cpu.run(1, hsa, hsb, co2, cf2)
                        reps += 1
                        if time.perf_counter() - t0 >= 2.0:
                            break
                    cdt = (time.perf_counter() - t0) / reps
                    c1["cpu_baseline"] = {"value": 2 * byts / cdt / 1e9, "unit": "GB/s", "cores": cpu.threads,
                                          "kind": cpu.kind,
                                          "sample": f"all {nb} pairs, add + sub (span-form dot_add_words / "
                                                    f"dot_sub_words, route {cpu.note}) x {reps} reps; results "
                                                    "bit-identical to the GPU's"}
                except Exception as e:  # noqa: BLE001
                    c1["cpu_baseline"] = {"value": None, "kind": "unavailable", "sample": str(e)[:200]}
            del hs, ho, ho2
        out["C1"] = c1
        del sets, calls
        torch.cuda.empty_cache()

    # ---------------- C3 / C4: batched multiply ----------------
    imad_peak_pps = sms * IMAD_WIDE_PER_CLK_SM * sm_max * 1e6  # u32 products / s at max clock
    for name, gen, m in (("C3", W.c3_inputs, 16), ("C4", W.c4_inputs, 64)):
        if not want(name):
            continue
        fa, fb = gen()
        Bn = fa.shape[0]
        lo, hi = rank_slice(Bn, rank, world)
        nb = hi - lo
        # rotating input copies so that every step reads more than the L2 between two uses of
        # the same operands (timing rule), at N = 1 too
        nrot = rotations(2 * nb * m * 8)
        rot = ([(fa, fb)] if world == 1 else []) + [(fa[lo:hi].clone(), fb[lo:hi].clone())
                                                    for _ in range(nrot - (1 if world == 1 else 0))]
        outs = [torch.empty((nb, 2 * m), dtype=torch.int64, device="cuda") for _ in rot]
        # one CUDA-graph replay of the captured dotg_mul_batch launch per step (as the headline)
        replays, mgraphs = [], []
        for o, (a_, b_) in zip(outs, rot):
            fn, _, g = capture_graph(torch, dg, lib, stream, lambda Lc, o=o, a_=a_, b_=b_: Lc.mul(o, a_, b_, m, nb))
            if fn is None:
                replays = None
                break
            replays.append(fn)
            mgraphs.append(g)
        calls = [make_rotating(replays if replays else [L.mul(o, a_, b_, m, nb) for o, (a_, b_) in zip(outs, rot)])]
        ms, per = timed_steps(torch, dd, world, stream, calls, steps, warm)
        # the kernel's launch duration with launches back to back (8 per graph over rotating
        # sets, events on the stream); the per-call event pair above also times the idle gap
        # before each replay
        b2b = per_launch_us(torch, dg, lib, stream,
                            lambda Lc: [Lc.mul(o, a_, b_, m, nb) for o, (a_, b_) in zip(outs, rot)] * 2)
        launch_ms = b2b * 1e-3 if b2b else per[0]
        pairs_s = nb / (launch_ms * 1e-3)
        prods = 4 * m * m
        o, (a, b) = outs[0], rot[0]
        res = {"metric": f"{64 * m}-bit mul products/s (pairs/s)", "value": Bn / (ms * 1e-3),
               "unit": "pairs/s", "kernel_pairs_s": pairs_s, "kernel_us": launch_ms * 1e3,
               "kernel_us_event_per_call": per[0] * 1e3,
               "timing": "value: one CUDA-graph replay of the launch per step; kernel_us: launches back to back "
                         "in one graph over rotating inputs, events on the stream",
               "u32_products_per_s": pairs_s * prods,
               "imad_roofline_u32_products_per_s": imad_peak_pps,
               "frac_imad": pairs_s * prods / imad_peak_pps,
               "hbm_gbs": nb * 32 * m / (per[0] * 1e-3) / 1e9,
               "note": "roofline = SMs x 32 IMAD.WIDE.U32/clk/SM (measured, tools/imad_peak.cu) x max SM clock",
               "l2": f"{len(rot)} rotating input sets of {2 * nb * m * 8 / 1e6:.0f} MB: more than the L2 is read "
                     "between two uses of the same operands"}
        roof = {"bound": "imad", "achieved": pairs_s * prods / 1e12, "peak": imad_peak_pps / 1e12,
                "unit": "T u32-products/s", "frac": pairs_s * prods / imad_peak_pps, "traffic": None,
                "algorithmic_units_per_launch": f"{nb} pairs x {prods} u32 products", "launch_us_avg": launch_ms * 1e3}
        if m in IMMA_ROUTE_M:
            # tensor-pipe kernel (k_mul_imma): radix-2^8 products, (8m)^2 byte-MACs per pair
            imma_peak = sms * IMMA_U8_MACS_PER_CLK_SM * sm_max * 1e6
            res.update({"pipe": "imma (mma.sync m16n8k32 u8, k_mul_imma)",
                        "u8_macs_per_s": pairs_s * (8 * m) ** 2,
                        "imma_roofline_u8_macs_per_s": imma_peak,
                        "frac_imma": pairs_s * (8 * m) ** 2 / imma_peak,
                        "note": "frac_imad: u32-product equivalents vs the IMAD.WIDE roofline (148 x 32/clk x "
                                "max clock); frac_imma: byte MACs vs the measured u8 IMMA rate (148 x 2048/clk "
                                "x max clock, tools/imma_peak.cu)"})
            roof["kernel"] = "k_mul_imma<16> (mma.sync u8 column sums)"
        else:
            res["pipe"] = "imad (IMAD.WIDE.U32 96-bit column MAC)"
            roof["kernel"] = "k_mul_kara16 (IMAD.WIDE.U32 columns, one in-register Karatsuba level)"
        res["roofline"] = roof
        if not args.no_e2e:
            # e2e: pinned host arrays through dotg_mul_batch_host (copies inside the timed region)
            ha, hb = pinned_like(torch, a), pinned_like(torch, b)
            ho = torch.empty(o.shape, dtype=torch.int64, pin_memory=True)
            assert lib.dotg_mul_batch_host(P(ho), P(ha), P(hb), m, nb) == 0
            torch.cuda.synchronize()
            assert torch.equal(ho, o.cpu()), "mul e2e mismatch"
            reps = 5
            if dd is not None:
                dist.barrier()
            t0 = time.perf_counter()
            for _ in range(reps):
                lib.dotg_mul_batch_host(P(ho), P(ha), P(hb), m, nb)
            dt = (time.perf_counter() - t0) / reps
            if dd is not None:
                dt = reduce_scalar(dist, dt, "max")
            res["e2e"] = {"value": Bn / dt, "unit": "pairs/s", "h2d_bytes_per_step": 2 * nb * m * 8,
                          "d2h_bytes_per_step": nb * 2 * m * 8, "api": "dotg_mul_batch_host"}
            if rank0 and world == 1 and not args.no_cpu:
                try:
                    cpu = CpuRef()
                    nsamp = Bn // 16
                    if name == "C4":  # half random, half all-ones pairs, as in the config
                        idx = np.concatenate([np.arange(nsamp // 2), np.arange(Bn // 2, Bn // 2 + nsamp // 2)])
                    else:
                        idx = np.arange(nsamp)
                    sa_ = np.ascontiguousarray(ha.numpy().view(np.uint64)[idx])
                    sb_ = np.ascontiguousarray(hb.numpy().view(np.uint64)[idx])
                    so_ = np.empty((nsamp, 2 * m), np.uint64)
                    cpu.run(2, sa_, sb_, so_, None)  # warm
                    t0 = time.perf_counter()
                    cpu.run(2, sa_, sb_, so_, None)
                    cdt = time.perf_counter() - t0
                    assert np.array_equal(so_, ho.numpy().view(np.uint64)[idx]), "cpu/gpu mismatch"
                    res["cpu_baseline"] = {"value": nsamp / cdt, "unit": "pairs/s", "cores": cpu.threads,
                                           "kind": cpu.kind,
                                           "sample": f"{nsamp} pairs of the same batch"
                                                     f"{' (half random, half all-ones)' if name == 'C4' else ''}, "
                                                     "dot_mul_words; results bit-identical to the GPU's"}
                except Exception as e:  # noqa: BLE001
                    res["cpu_baseline"] = {"value": None, "kind": "unavailable", "sample": str(e)[:200]}
            del ha, hb, ho
        out[name] = res
        del fa, fb, rot, outs, calls, a, b, o
        torch.cuda.empty_cache()

    # ---------------- interleaved layout (north star's batch-interleaved subsystem) ----------------
    if want("IL") and world == 1 and not args.no_layouts:
        il = {}
        # back-to-back launches over 3 rotating input copies (> L2 between reuses)
        for m, B in [(64, 1 << 16)] + [(mm, (1 << 22) // mm) for mm in (4, 16, 128, 256, 512)]:
            sets = []
            for r in range(3):
                a = W.fill(B * m, 0x1A + m + 7 * r, 0).view(m, B)  # [m][batch]
                b = W.fill(B * m, 0x1A + m + 7 * r, 1 << 40).view(m, B)
                sets.append((a, b, torch.empty_like(a), torch.empty(B, dtype=torch.int32, device="cuda")))
            byts = B * (24 * m + 4)
            row = {}
            for sub in (0, 1):
                fn = lib.dotg_sub_batch if sub else lib.dotg_add_batch

                def mk(Lc, fn=fn, sets=sets):
                    return [(lambda args_=(P(o), P(a), P(b), P(f), m, B, 1, Lc.stream): fn(*args_))
                            for a, b, o, f in sets]
                us = per_launch_us(torch, dg, lib, stream, mk)
                op = "sub" if sub else "add"
                row[f"{op}_gbs"] = byts / (us * 1e-6) / 1e9
                row[f"{op}_frac"] = byts / (us * 1e-6) / 1e9 / hbm_peak
            il[f"m{m}_B{B}"] = row
            del sets
        # interleaved multiply at the C3 / C4 shapes
        for m, B in ((16, 1 << 18), (32, 1 << 17), (64, 1 << 16)):
            sets = []
            for r in range(2):
                a = W.fill(B * m, 0x1B + m + 7 * r, 0).view(m, B)
                b = W.fill(B * m, 0x1B + m + 7 * r, 1 << 40).view(m, B)
                sets.append((a, b, torch.empty((2 * m, B), dtype=torch.int64, device="cuda")))

            def mk(Lc, sets=sets, m=m, B=B):
                return [(lambda args_=(P(o), P(a), P(b), m, B, 1, Lc.stream): lib.dotg_mul_batch(*args_))
                        for a, b, o in sets]
            us = per_launch_us(torch, dg, lib, stream, mk)
            il[f"mul_m{m}_B{B}"] = {"pairs_s": B / (us * 1e-6), "us": us,
                                    "frac_imad": B / (us * 1e-6) * 4 * m * m / imad_peak_pps}
            del sets
        out["interleaved"] = {"layout": "[m][batch] (limb i of pair p at i*batch + p)", "per_shape": il,
                              "peak": hbm_peak, "timing": "back-to-back launches over rotating input copies "
                                                          "(CUDA graph, events on the stream)"}
        torch.cuda.empty_cache()

    # ---------------- 256-bit base cases: dot_mul_5x5 / dot_mul_4x4 shapes ----------------
    if want("R52") and world == 1 and not args.no_layouts:
        r52 = {}
        Bq = 1 << 21
        for name, m, fn, mask in (("mul52_5x5", 5, lib.dotg_mul52_batch, (1 << 52) - 1),
                                  ("mul64_4x4", 4, None, None)):
            a = W.fill(Bq * m, 0x52 + m, 0).view(Bq, m)
            b = W.fill(Bq * m, 0x52 + m, 1 << 40).view(Bq, m)
            if mask is not None:
                a &= mask
                b &= mask
            o = torch.empty((Bq, 2 * m), dtype=torch.int64, device="cuda")

            def mk(Lc, fn=fn, o=o, a=a, b=b, m=m):
                if fn is None:
                    return [Lc.mul(o, a, b, m, Bq)]
                args_ = (P(o), P(a), P(b), m, Bq, Lc.stream)
                return [lambda: fn(*args_)]
            us = per_launch_us(torch, dg, lib, stream, mk)
            byts = Bq * 32 * m
            r52[name] = {"pairs_s": Bq / (us * 1e-6), "us": us, "hbm_gbs": byts / (us * 1e-6) / 1e9,
                         "frac_hbm": byts / (us * 1e-6) / 1e9 / hbm_peak, "batch": Bq}
            del a, b, o
        out["base_case_256bit"] = r52
        torch.cuda.empty_cache()

    # ---------------- wide products on tcgen05 (mul_umma.cu; Karatsuba leaves above 4096 limbs) ----------------
    if want("WIDE") and world == 1 and not args.no_layouts:
        wide = {}
        tensor_peak = sms * UMMA_U8_MACS_PER_CLK_SM * sm_max * 1e6  # byte-MACs / s at max clock
        for m, B in ((1024, 1024), (2048, 256), (4096, 64)):
            sets = []
            for r in range(rotations(2 * B * m * 8)):  # more than the L2 read between reuses
                a = W.fill(B * m, 0x3C + m + 7 * r, 0).view(B, m)
                b = W.fill(B * m, 0x3C + m + 7 * r, 1 << 40).view(B, m)
                sets.append((a, b, torch.empty((B, 2 * m), dtype=torch.int64, device="cuda")))

            def mk(Lc, sets=sets, m=m, B=B):
                return [(lambda args_=(P(o), P(a), P(b), m, B, 0, Lc.stream): lib.dotg_mul_batch(*args_))
                        for a, b, o in sets]
            us = per_launch_us(torch, dg, lib, stream, mk)
            macs = B * (8 * m) ** 2
            wide[f"m{m}_B{B}"] = {"pairs_s": B / (us * 1e-6), "us": us, "byte_macs_per_s": macs / (us * 1e-6),
                                  "frac_tensor_u8": macs / (us * 1e-6) / tensor_peak,
                                  "prior_route_us": WIDE_PRIOR_US.get((m, B))}
            del sets
        out["wide_products"] = {
            "kernel": "k_mul_umma: tcgen05.mma.cta_group::1.kind::i8 M=128, Hankel core-matrix ring (A) and "
                      "byte-reversed a-chunk arrays (B) in shared memory, column sums in TMEM, in-CTA carry resolve",
            "per_shape": wide, "tensor_peak_byte_macs_per_s": tensor_peak,
            "peak_note": "148 SMs x 8192 u8 MACs/clk/SM (tools/umma_i8_probe.cu, N=128/256) x max SM clock; "
                         "schoolbook byte-MACs (8m)^2 per pair counted",
            "prior_route_note": "prior_route_us: the same call on the mma.sync Karatsuba route (DOTG_MUL_UMMA=0), "
                                "profiles/r02_umma_wide_variants.txt",
            "timing": "back-to-back calls over rotating input sets (more than the L2 read between reuses; CUDA graph, events on the stream)"}
        torch.cuda.empty_cache()

    # ---------------- C5: one 2^30-limb add / sub ----------------
    if not args.no_c5 and want("C5"):
        from paper_2604_21566_b200.sharded import CommShardedWords, ShardedWords, shard_bounds

        M5 = W.C5_M
        lo, hi = shard_bounds(M5, rank, world)
        n_local = hi - lo
        free = torch.cuda.mem_get_info()[0]
        if world > 1:  # the skip decision must be the same on every rank (collectives follow)
            free = int(reduce_scalar(dist, float(free), "min"))
        if free < 3 * n_local * 8 + (1 << 30):
            out["C5"] = {"skipped": f"needs {3 * n_local * 8 / 2**30:.0f} GiB free per GPU"}
            return out
        shared = os.environ.get("DOTG_BENCH_SHARED_GPU") == "1"
        comm = CommShardedWords() if world > 1 and not shared else None
        res = {}
        for sub in (False, True):
            a, b = W.c5_shard_inputs(sub, lo, hi) if world > 1 else W.c5_inputs(sub)
            o = torch.empty_like(a)
            c = torch.empty(1, dtype=torch.int32, device="cuda")
            if world == 1:
                fn = lib.dotg_sub_words if sub else lib.dotg_add_words
                args_ = (P(o), P(a), P(b), n_local, P(c), L.stream)
                call = lambda fn=fn, args_=args_: fn(*args_)  # noqa: E731
                mode = "single GPU: dotg_add_words / dotg_sub_words (tiled local pass, chunk scan, fix-up)"
            elif comm is not None:
                def call(sub=sub, a=a, b=b, o=o, c=c):
                    comm.run(sub, o, a, b, carry=c, stream=stream)
                    return 0
                mode = (f"{world} limb-range shards: one dotg_{'sub' if sub else 'add'}_words_sharded call per "
                        "rank (C++: local pass, 8-byte ncclAllGather, fix-up on one stream)")
            else:
                sw = ShardedWords()
                state = sw.state_for(n_local, a.device)

                def call(sub=sub, a=a, b=b, o=o, sw=sw, state=state):
                    sw.run(sub, o, a, b, state=state)
                    return 0
                mode = f"{world} limb-range shards, gloo exchange (shared-GPU rehearsal)"
            ms, per = timed_steps(torch, dd, world, stream, [call], 3, 2)
            carry = int(c.item()) if world == 1 or comm is not None else None
            r = {"ms": ms, "gbs": 24 * M5 / (ms * 1e-3) / 1e9,
                 "frac_hbm_per_gpu": 24 * n_local / (ms * 1e-3) / 1e9 / hbm_peak, "carry": carry, "mode": mode}
            r["roofline"] = hbm_roofline(24 * n_local, per[0] * 1e-3, hbm_peak,
                                         "k_long_local + k_long_scan_chunks + k_long_shard_agg + k_long_finish "
                                         "(one long add/sub; k_long_local carries ~90% of the time)",
                                         traffic=traffic_table().get("C5_per_op_bytes") if world == 1 else None)
            if world == 1 and not args.no_e2e and rank0:
                # e2e through the host span form on pinned 8 GiB host arrays, and the
                # reference's span-form dot_add_words on the same host arrays (1 thread)
                ha, hb = pinned_like(torch, a), pinned_like(torch, b)
                del a, b, o
                torch.cuda.empty_cache()
                ho = torch.empty(ha.shape, dtype=torch.int64, pin_memory=True)
                hfn = lib.dotg_sub_words_host if sub else lib.dotg_add_words_host
                hc = ctypes.c_uint32(0)
                assert hfn(P(ho), P(ha), P(hb), M5, ctypes.byref(hc)) == 0, lib.dotg_last_error()
                assert hc.value == carry, "C5 e2e carry mismatch"
                reps = 2
                t0 = time.perf_counter()
                for _ in range(reps):
                    hfn(P(ho), P(ha), P(hb), M5, ctypes.byref(hc))
                dt = (time.perf_counter() - t0) / reps
                r["e2e"] = {"value": 24 * M5 / dt / 1e9, "unit": "GB/s", "h2d_bytes_per_step": 16 * M5,
                            "d2h_bytes_per_step": 8 * M5 + 4,
                            "api": f"dotg_{'sub' if sub else 'add'}_words_host (pinned 8 GiB host operands)"}
                if not args.no_cpu:
                    try:
                        cpu = CpuRef()
                        hav, hbv = ha.numpy().view(np.uint64), hb.numpy().view(np.uint64)
                        co = np.empty(M5, np.uint64)
                        t0 = time.perf_counter()
                        cc = cpu.words(int(sub), co, hav, hbv)
                        cdt = time.perf_counter() - t0
                        assert cc == carry and np.array_equal(co, ho.numpy().view(np.uint64)), "C5 cpu/gpu mismatch"
                        r["cpu_baseline"] = {"value": 24 * M5 / cdt / 1e9, "unit": "GB/s", "cores": 1,
                                             "kind": cpu.kind,
                                             "sample": f"all 2^30 limbs, one span-form dot_{'sub' if sub else 'add'}"
                                                       f"_words call (route {cpu.note}; the reference's carry "
                                                       "chain is serial, so 1 thread); bit-identical to the GPU"}
                        del co
                    except Exception as e:  # noqa: BLE001
                        r["cpu_baseline"] = {"value": None, "kind": "unavailable", "sample": str(e)[:200]}
                del ha, hb, ho
            else:
                del a, b, o
            res["sub" if sub else "add"] = r
            torch.cuda.empty_cache()
        if comm is not None:
            comm.close()
        out["C5"] = {"metric": "one 2^30-limb add/sub GB/s (whole number, all GPUs)", "unit": "GB/s",
                     "n_limbs": M5, "shard_limbs": n_local, "run": list(W.C5_RUN), **res}
    return out


def cpu_ref_table():
    """BASELINE.md §4 CPU columns (part of the CPU-baseline leg): the reference's own
    DoT path (oracle/_ref/libdotref.so) on this host, 1 thread and all threads, per
    config, on bounded samples of the configs' inputs (device generators, copied to the
    host). add/sub in algorithmic GB/s (24m + 4 B per pair-op), mul in pairs/s, C5 in
    GB/s (24 B per limb, single thread: the reference's carry chain is serial)."""
    import numpy as np
    import torch

    from paper_2604_21566_b200 import workloads as W

    L = ctypes.CDLL(os.path.join(ROOT, "oracle", "_ref", "libdotref.so"))
    L.dotref_batch.restype = ctypes.c_int
    L.dotref_batch.argtypes = [ctypes.c_int, ctypes.c_int] + [ctypes.c_void_p] * 4 + [ctypes.c_size_t] * 2 + [ctypes.c_int]
    L.dotref_words.restype = ctypes.c_int
    L.dotref_words.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t,
                               ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    L.dotref_dispatch_note.restype = ctypes.c_char_p
    L.dotref_dispatch_note.argtypes = [ctypes.c_int]
    NT = os.cpu_count() or 1
    P = lambda x: None if x is None else ctypes.c_void_p(x.ctypes.data)  # noqa: E731

    def host(t):
        return t.cpu().numpy().view(np.uint64).copy()

    def best_of(fn, reps=3):
        fn()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        return min(ts)

    def batch_rate(op, a, b, threads):
        B, m = a.shape
        out = np.empty((B, 2 * m if op == 2 else m), np.uint64)
        fl = None if op == 2 else np.empty(B, np.uint32)
        dt = best_of(lambda: L.dotref_batch(op, 0, P(out), P(a), P(b), P(fl), m, B, threads))
        return dt

    res = {"cpu": open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": \t"),
           "threads_all": NT, "route": L.dotref_dispatch_note(8).decode(), "rows": []}

    def row(cfg, unit, sample, v1, vn):
        res["rows"].append({"config": cfg, "unit": unit, "sample": sample, "one_thread": v1, "all_threads": vn})

    # C1: 4096-bit add + sub, sample 16384 of 65536 pairs
    a, b, sa, sb = W.c1_inputs()
    n = 16384
    ha, hb, hsa, hsb = host(a[:n]), host(b[:n]), host(sa[:n]), host(sb[:n])
    byts = 2 * n * (24 * 64 + 4)
    # the reference bench's methodology on one core: ns per op, mean +- Student-t CI95
    # over 7 repetitions, span form and value form (bench.cpp:95-104, 216-225)
    t_975_6 = 2.447
    for impl, form in ((0, "span"), (2, "value")):
        out_ = np.empty_like(ha)
        fl_ = np.empty(n, np.uint32)
        L.dotref_batch(0, impl, P(out_), P(ha), P(hb), P(fl_), 64, n, 1)
        ts = []
        for _ in range(7):
            t0 = time.perf_counter()
            L.dotref_batch(0, impl, P(out_), P(ha), P(hb), P(fl_), 64, n, 1)
            ts.append((time.perf_counter() - t0) / n * 1e9)
        mean = statistics.mean(ts)
        ci = t_975_6 * statistics.stdev(ts) / len(ts) ** 0.5
        res["rows"].append({"config": f"C1 add m=64, {form} form, 1 thread", "unit": "ns/op", "sample": f"{n} ops x 7",
                            "one_thread": mean, "ci95": ci, "all_threads": None})
    for th in (1, NT):
        dt = batch_rate(0, ha, hb, th) + batch_rate(1, hsa, hsb, th)
        if th == 1:
            v1 = byts / dt / 1e9
        else:
            vn = byts / dt / 1e9
    row("C1 add+sub m=64", "GB/s", f"{n} pairs add + sub", v1, vn)
    del a, b, sa, sb

    # C2: the four carry-stress sizes, 1/4 of each batch
    tot_b, tot_t = 0, {1: 0.0, NT: 0.0}
    for m, B in W.C2_SIZES:
        a, b, sa, sb = W.c2_inputs(m, B)
        n = B // 4
        ha, hb, hsa, hsb = host(a[:n]), host(b[:n]), host(sa[:n]), host(sb[:n])
        byts = 2 * n * (24 * m + 4)
        vals = {}
        for th in (1, NT):
            dt = batch_rate(0, ha, hb, th) + batch_rate(1, hsa, hsb, th)
            vals[th] = byts / dt / 1e9
            tot_t[th] += dt
        tot_b += byts
        row(f"C2 add+sub m={m}", "GB/s", f"{n} of {B} pairs add + sub", vals[1], vals[NT])
        del a, b, sa, sb
    row("C2 sweep (all sizes)", "GB/s", "1/4 of every batch", tot_b / tot_t[1] / 1e9, tot_b / tot_t[NT] / 1e9)

    # C3 / C4 multiplication (dot_mul_words)
    for name, gen, n in (("C3 mul m=16", W.c3_inputs, 16384), ("C4 mul m=64", W.c4_inputs, 2048)):
        a, b = gen()
        half = a.shape[0] // 2
        if name.startswith("C4"):  # half random, half all-ones pairs, as in the config
            idx = torch.cat([torch.arange(0, n // 2), torch.arange(half, half + n // 2)]).cuda()
            ha, hb = host(a[idx]), host(b[idx])
        else:
            ha, hb = host(a[:n]), host(b[:n])
        vals = {th: n / batch_rate(2, ha, hb, th) for th in (1, NT)}
        row(name, "pairs/s", f"{n} pairs", vals[1], vals[NT])
        del a, b

    # C5: one long add / sub, single thread (the reference's carry chain is serial)
    m5 = 1 << 28
    run = (3 << 25, 5 << 25)
    for sub in (False, True):
        a_d, b_d = W.c5_inputs(sub, m=m5, run=run)
        ha, hb = host(a_d), host(b_d)
        del a_d, b_d
        out = np.empty(m5, np.uint64)
        dt = best_of(lambda: L.dotref_words(int(sub), P(out), m5, P(ha), m5, P(hb), m5, 8, None, None), reps=2)
        row(f"C5 {'sub' if sub else 'add'} (2^28-limb sample)", "GB/s", f"{m5} limbs, run of 2^26 limbs",
            24 * m5 / dt / 1e9, None)
        del ha, hb, out

    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c5", action="store_true")
    ap.add_argument("--no-layouts", action="store_true", help="skip the interleaved-layout rows")
    ap.add_argument("--no-phase", action="store_true", help="skip the phase-tick split")
    ap.add_argument("--only", default="", help="comma list of C1,C3,C4,C5: run only those secondary configs")
    ap.add_argument("--ungrouped", action="store_true", help="one launch per (size, op) instead of one grouped launch")
    ap.add_argument("--no-graph", action="store_true", help="direct launches instead of one CUDA-graph replay per step")
    ap.add_argument("--cpu-seconds", type=float, default=5.0)
    ap.add_argument("--cpu-table", action="store_true",
                    help="print the CPU reference table (1 thread / all threads per config) and exit")
    args = ap.parse_args()
    if args.cpu_table:
        print(json.dumps(cpu_ref_table(), indent=1))
        return 0
    args.warmup = max(3, args.warmup)
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist

        # DOTG_BENCH_SHARED_GPU=1: every rank on GPU 0 with gloo - a control-flow rehearsal
        # of the multi-rank bench on a one-GPU box (numbers meaningless, no kernel waits on
        # another rank's kernel: the exchanges are host-orchestrated collectives)
        shared = os.environ.get("DOTG_BENCH_SHARED_GPU") == "1"
        if args.impl == "ours":
            torch.cuda.set_device(device_index())
        dist.init_process_group("nccl" if args.impl == "ours" and not shared else "gloo")
    try:
        if args.impl == "reference":
            return run_reference(args, rank, world)
        return run_ours(args, rank, world, dist)
    finally:
        if dist is not None:
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
