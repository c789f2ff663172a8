#!/usr/bin/env python
"""bench.py - B200 limb arithmetic (DigitsOnTurbo hot path) benchmark.

Headline workload (BASELINE.json configs[1], "C2"): the carry-stress add/sub sweep -
(m, B) in (4, 2^20), (16, 2^18), (64, 2^16), (256, 2^14); each limb all-ones with p=1/2
else uniform, 1% of pairs forced to a full-length carry chain; sub swaps pairs so a >= b.
One step = batched add at all four sizes, then batched sub at all four sizes, through the
device C ABI (dotg_add_batch / dotg_sub_batch). Metric: algorithmic GB/s
(24m + 4 bytes per pair-op), roofline = measured HBM copy bandwidth.

The same JSON line also reports C1 (4096-bit add/sub), C3/C4 (1024/4096-bit mul,
products/s vs the measured IMAD.WIDE roofline) and C5 (one 2^30-limb add/sub) under
"configs".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--only C2] [--no-secondary]

N > 1: launched by torch.distributed.run, one rank per GPU; every rank runs the full
batch sweep on its own GPU (weak scaling, no collective on the data path); value = the
bytes of all ranks / max-over-ranks time. --impl reference times the reference's own
CPU implementation (oracle/_ref/libdotref.so: span-form dot_add_words / dot_sub_words
at Width::w8 and dot_mul_words) on all host cores; under torchrun only rank 0 works.
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


def c2_config(ungrouped=False, working_set=None):
    cfg = {"workload": "C2 carry-stress add+sub sweep (BASELINE.json configs[1])",
           "sizes_m_batch": C2_SIZES, "layout": "row-major [batch][m] (reference Limbs layout)",
           "step": ("8 launches: add at 4 sizes then sub at 4 sizes" if ungrouped else
                    "one dotg_addsub_grouped call = one persistent launch: add at 4 sizes + sub at 4 sizes"),
           "per_rank": "full sweep on every rank (weak scaling, no collective)"}
    if working_set is not None:
        cfg["l2"] = (f"inputs larger than L2: each step reads {working_set / 1e6:.0f} MB of distinct inputs "
                     "(126 MB L2), every buffer touched once per step")
    return cfg


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
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u64", "data": DATA,
        "config": c2_config(),
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


def run_ours(args, rank, world, dist):
    import numpy as np
    import torch

    import paper_2604_21566_b200 as dg
    from paper_2604_21566_b200 import workloads as W

    lib = dg.lib()  # raises if libdotg.so is missing: no fallback
    torch.cuda.set_device(device_index())
    if args.only:
        stream = torch.cuda.current_stream()
        hbm_peak, _, sm_max = peaks()
        sms = torch.cuda.get_device_properties(0).multi_processor_count
        res = run_secondary(args, torch, dg, W, Launcher(torch, lib, stream), stream, world, dist, hbm_peak,
                            sm_max, sms)
        if rank == 0:
            print(json.dumps({"only": args.only, "configs": res}), flush=True)
        return 0
    stream = torch.cuda.current_stream()
    L = Launcher(torch, lib, stream)
    hbm_peak, peak_kind, sm_max = peaks()
    sms = torch.cuda.get_device_properties(0).multi_processor_count

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
    step_bytes = sum(call_bytes)
    # per-problem launches (event-bracketed breakdown, and --ungrouped timing)
    single_calls = [L.addsub(*q) for q in probs]
    if args.ungrouped:
        calls = single_calls
    else:
        calls = [L.grouped(probs)]  # the whole sweep = one persistent launch
    # The step as a CUDA graph (one replay per step): same kernel, same bytes, without the
    # host launch path between consecutive steps. --no-graph keeps direct launches.
    graph_launches = None
    if not args.ungrouped and not args.no_graph:
        try:
            cap = torch.cuda.Stream()
            cap.wait_stream(stream)
            Lc = Launcher(torch, lib, cap)
            cap_call = Lc.grouped(probs)
            with torch.cuda.stream(cap):
                assert cap_call() == 0
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            n0 = dg.kernel_launches()
            with torch.cuda.graph(graph, stream=cap):
                cap_call()
            graph_launches = dg.kernel_launches() - n0
            torch.cuda.synchronize()
            calls = [lambda: (graph.replay(), 0)[1]]
        except Exception as e:  # noqa: BLE001
            graph_launches = None
            print(f"graph capture unavailable ({e}); direct launches", file=sys.stderr)
    calls_meta = list(range(len(calls)))
    assert step_bytes == c2_bytes()
    working_set = sum(4 * x["a"].numel() * 8 for x in bufs)  # distinct inputs read per step (a, b, sa, sb)

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
    value = step_bytes * world / (ms_step * 1e-3) / 1e9
    # average launch duration of the batched add/sub kernel = lean-loop step time / launches
    # (inter-launch gaps included: conservative); per_size uses event-bracketed launches.
    achieved = step_bytes / (ms_step * 1e-3) / 1e9
    _, per_single = timed_steps(torch, None, 1, stream, single_calls, max(3, args.steps // 4), 2)
    per_size = {f"m{x['m']}": {"add_gbs": call_bytes[i] / (per_single[i] * 1e-3) / 1e9,
                               "sub_gbs": call_bytes[i] / (per_single[i + 4] * 1e-3) / 1e9}
                for i, x in enumerate(bufs)}
    traffic = traffic_table().get("C2_per_launch_bytes_grouped" if not args.ungrouped else "C2_per_launch_bytes")
    # the same byte mix without carries: a plain 2-read / 1-write streaming add measured
    # live (tools/stream_peak.cu) - the practical ceiling for this kernel's traffic
    mix_peak = None
    sp = os.path.join(ROOT, "tools", "build", "stream_peak")
    if os.path.exists(sp) and rank == 0:
        try:
            import subprocess

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

    # ---- e2e: the same step through the host-buffer C ABI (pinned host arrays) ----
    e2e = None
    if not args.no_e2e:
        hsets = []
        for x in bufs:
            hs = {}
            for k in ("a", "b", "sa", "sb"):
                h = torch.empty(x[k].shape, dtype=torch.int64, pin_memory=True)
                h.copy_(x[k])
                hs[k] = h
            hs["o"] = torch.empty(x["a"].shape, dtype=torch.int64, pin_memory=True)
            hs["os"] = torch.empty(x["a"].shape, dtype=torch.int64, pin_memory=True)
            hs["f"] = torch.empty(x["B"], dtype=torch.int32, pin_memory=True)
            hs["fs"] = torch.empty(x["B"], dtype=torch.int32, pin_memory=True)
            hsets.append((x["m"], x["B"], hs))
        from paper_2604_21566_b200._lib import AddSubProblem

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
        # correctness spot check of the e2e path against the device result (last call = sub m=256)
        m, B, hs = hsets[-1]
        assert torch.equal(hs["os"], bufs[-1]["os"].cpu()), "e2e result mismatch"
        assert torch.equal(hsets[0][2]["o"], bufs[0]["oa"].cpu()), "e2e result mismatch"
        e_steps = max(3, min(args.steps, 20))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e_steps):
            e2e_step()
        dt = time.perf_counter() - t0
        if world > 1:
            dt = reduce_scalar(dist, dt, "max")
        h2d = sum(2 * 2 * B * m * 8 for m, B in C2_SIZES)
        d2h = sum(2 * (B * m * 8 + 4 * B) for m, B in C2_SIZES)
        e2e = {"value": step_bytes * world * e_steps / dt / 1e9, "unit": "GB/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "steps": e_steps,
               "api": "dotg_addsub_grouped_host: the 8 host problems through one H2D / kernel / D2H stream "
                      "pipeline (pinned host buffers)"}
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
            e2e["transfer_only_GBps"] = step_bytes / tx / 1e9
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
            sets = host_c2_inputs()
            gbs, reps, dt = cpu_c2_measure(cpu, sets, min_seconds=args.cpu_seconds)
            cpu_baseline = {"value": gbs, "unit": "GB/s", "cores": cpu.threads, "kind": cpu.kind,
                            "sample": f"full C2 step (add+sub at 4 sizes, {c2_bytes() / 1e6:.0f} MB) x {reps} reps "
                                      f"({dt:.1f} s), span-form dot_add_words/dot_sub_words route {cpu.note}"}
            del sets
        except Exception as e:  # noqa: BLE001
            cpu_baseline = {"value": None, "unit": "GB/s", "cores": 0, "kind": "unavailable", "sample": str(e)}

    # free the headline buffers before the secondary configs
    del bufs, calls, single_calls
    torch.cuda.empty_cache()

    secondary = {}
    if not args.no_secondary:
        secondary = run_secondary(args, torch, dg, W, L, stream, world, dist, hbm_peak, sm_max, sms, rank == 0)

    line = {
        "metric": METRIC,
        "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": DATA,
        "config": c2_config(args.ungrouped, working_set),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic,
                     "kernel": "k_addsub_grouped (persistent batched add/sub, warp-ballot lookahead)",
                     "algorithmic_bytes_per_launch": step_bytes / len(calls_meta),
                     "launch_us_avg": ms_step * 1e3 / len(calls_meta), "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
                     "per_size": per_size, "mix_peak": mix_peak},
        "cpu_baseline": cpu_baseline,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "launch_mode": ("one CUDA-graph replay per step (the captured dotg_addsub_grouped launch)"
                        if graph_launches is not None else "direct C-ABI launches"),
        "clocks": clocks,
        "carry_stress": stress,
        "configs": secondary,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def run_secondary(args, torch, dg, W, L, stream, world, dist, hbm_peak, sm_max, sms, rank0=True):
    out = {}
    steps = max(3, min(args.steps, 50))
    warm = max(3, args.warmup)
    dd = dist if world > 1 else None

    def want(k):
        return not args.only or k in args.only.split(",")

    # C1: 4096-bit add + sub (rotate 3 input sets -> 300 MB between reuses > L2)
    sets = []
    for r in range(3 if want("C1") else 0):
        a = W.fill(W.C1["batch"] * 64, 0xC1 + 17 * r, 0).view(-1, 64)
        b = W.fill(W.C1["batch"] * 64, 0xC1 + 17 * r, 1 << 40).view(-1, 64)
        sa, sb = W.swap_for_sub(a, b)
        sets.append((a, b, sa, sb, torch.empty_like(a), torch.empty(a.shape[0], dtype=torch.int32, device="cuda")))
    B = W.C1["batch"]
    calls = []
    if not want("C1"):
        sets = []
    outs2 = []
    for a, b, sa, sb, o, f in sets:
        # add and sub of one set: one grouped launch (two problems, separate outputs)
        o2, f2 = torch.empty_like(o), torch.empty_like(f)
        outs2.append((o2, f2))
        calls.append(L.grouped([(False, o, a, b, f, 64, B), (True, o2, sa, sb, f2, 64, B)]))
    if sets:
        ms, per = timed_steps(torch, dd, world, stream, calls, steps, warm)
    byts = B * (24 * 64 + 4)
    if sets:
        nops = 2 * len(calls)
        out["C1"] = {"metric": "add/sub GB/s (4096-bit, B=65536)", "value": byts * nops * world / (ms * 1e-3) / 1e9,
                     "unit": "GB/s", "kernel_gbs": byts * nops / (sum(per) * 1e-3) / 1e9,
                     "frac_hbm": byts * nops / (sum(per) * 1e-3) / 1e9 / hbm_peak,
                     "frac_hbm_back_to_back": byts * nops / (ms * 1e-3) / 1e9 / hbm_peak,
                     "launch_us": statistics.mean(per) * 1e3,
                     "step": "3 rotating input sets (300 MB apart > L2); per set add + sub in one dotg_addsub_grouped "
                             "launch"}
    del outs2
    del sets, calls
    torch.cuda.empty_cache()

    imad_peak_pps = sms * IMAD_WIDE_PER_CLK_SM * sm_max * 1e6  # u32 products / s at max clock
    for name, gen, m in (("C3", W.c3_inputs, 16), ("C4", W.c4_inputs, 64)):
        if not want(name):
            continue
        a, b = gen()
        Bn = a.shape[0]
        o = torch.empty((Bn, 2 * m), dtype=torch.int64, device="cuda")
        calls = [L.mul(o, a, b, m, Bn)]
        ms, per = timed_steps(torch, dd, world, stream, calls, steps, warm)
        pairs_s = Bn / (per[0] * 1e-3)
        prods = 4 * m * m
        out[name] = {"metric": f"{64 * m}-bit mul products/s (pairs/s)", "value": Bn * world / (ms * 1e-3),
                     "unit": "pairs/s", "kernel_pairs_s": pairs_s, "kernel_us": per[0] * 1e3,
                     "u32_products_per_s": pairs_s * prods,
                     "imad_roofline_u32_products_per_s": imad_peak_pps,
                     "frac_imad": pairs_s * prods / imad_peak_pps,
                     "hbm_gbs": Bn * 32 * m / (per[0] * 1e-3) / 1e9,
                     "note": "roofline = SMs x 32 IMAD.WIDE.U32/clk/SM (measured, tools/imad_peak.cu) x max SM clock"}
        if m in IMMA_ROUTE_M:
            # tensor-pipe kernel (k_mul_imma): radix-2^8 products, (8m)^2 byte-MACs per pair
            imma_peak = sms * IMMA_U8_MACS_PER_CLK_SM * sm_max * 1e6
            out[name].update({"pipe": "imma (mma.sync m16n8k32 u8, k_mul_imma)",
                              "u8_macs_per_s": pairs_s * (8 * m) ** 2,
                              "imma_roofline_u8_macs_per_s": imma_peak,
                              "frac_imma": pairs_s * (8 * m) ** 2 / imma_peak,
                              "note": "frac_imad: u32-product equivalents vs the IMAD.WIDE roofline (148 x 32/clk x "
                                      "max clock); frac_imma: byte MACs vs the measured u8 IMMA rate (148 x 2048/clk "
                                      "x max clock, tools/imma_peak.cu)"})
        else:
            out[name]["pipe"] = "imad (IMAD.WIDE.U32 96-bit column MAC)"
        if not args.no_e2e:
            # e2e: pinned host arrays through dotg_mul_batch_host (copies inside the timed region)
            ha = torch.empty(a.shape, dtype=torch.int64, pin_memory=True)
            hb = torch.empty(b.shape, dtype=torch.int64, pin_memory=True)
            ho = torch.empty(o.shape, dtype=torch.int64, pin_memory=True)
            ha.copy_(a)
            hb.copy_(b)
            lib = dg.lib()
            P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
            assert lib.dotg_mul_batch_host(P(ho), P(ha), P(hb), m, Bn) == 0
            assert torch.equal(ho, o.cpu()), "mul e2e mismatch"
            reps = 5
            t0 = time.perf_counter()
            for _ in range(reps):
                lib.dotg_mul_batch_host(P(ho), P(ha), P(hb), m, Bn)
            dt = (time.perf_counter() - t0) / reps
            out[name]["e2e"] = {"value": Bn * world / dt, "unit": "pairs/s", "h2d_bytes_per_step": 2 * Bn * m * 8,
                                "d2h_bytes_per_step": Bn * 2 * m * 8, "api": "dotg_mul_batch_host"}
            if rank0 and world == 1 and not args.no_cpu:
                try:
                    cpu = CpuRef()
                    import numpy as np

                    nsamp = Bn // 16
                    sa_ = ha[:nsamp].numpy().view(np.uint64)
                    sb_ = hb[:nsamp].numpy().view(np.uint64)
                    so_ = np.empty((nsamp, 2 * m), np.uint64)
                    cpu.run(2, sa_, sb_, so_, None)  # warm
                    t0 = time.perf_counter()
                    cpu.run(2, sa_, sb_, so_, None)
                    cdt = time.perf_counter() - t0
                    assert np.array_equal(so_, ho[:nsamp].numpy().view(np.uint64)), "cpu/gpu mismatch"
                    out[name]["cpu_baseline"] = {"value": nsamp / cdt, "unit": "pairs/s", "cores": cpu.threads,
                                                 "kind": cpu.kind,
                                                 "sample": f"{nsamp} pairs of the same batch, dot_mul_words"}
                except Exception as e:  # noqa: BLE001
                    out[name]["cpu_baseline"] = {"value": None, "kind": "unavailable", "sample": str(e)}
            del ha, hb, ho
        del a, b, o, calls
        torch.cuda.empty_cache()

    if not args.no_c5 and want("C5"):
        from paper_2604_21566_b200.sharded import ShardedWords, shard_bounds

        M5 = W.C5_M
        rank = dist.get_rank() if world > 1 else 0
        lo, hi = shard_bounds(M5, rank, world)
        n_local = hi - lo
        free = torch.cuda.mem_get_info()[0]
        if world > 1:  # the skip decision must be the same on every rank (collectives follow)
            free = int(reduce_scalar(dist, float(free), "min"))
        if free < 3 * n_local * 8 + (1 << 30):
            out["C5"] = {"skipped": f"needs {3 * n_local * 8 / 2**30:.0f} GiB free per GPU"}
            return out
        res = {}
        for sub in (False, True):
            a, b = W.c5_shard_inputs(sub, lo, hi) if world > 1 else W.c5_inputs(sub)
            o = torch.empty_like(a)
            c = torch.empty(1, dtype=torch.int32, device="cuda")
            if world == 1:
                fn = dg.lib().dotg_sub_words if sub else dg.lib().dotg_add_words
                args_ = (ctypes.c_void_p(o.data_ptr()), ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()),
                         n_local, ctypes.c_void_p(c.data_ptr()), L.stream)
                call = lambda: fn(*args_)  # noqa: E731
            else:
                # limb-range shards: local pass, 8-byte NCCL all-gather, boundary fix-up
                sw = ShardedWords()
                state = sw.state_for(n_local, a.device)

                def call():
                    sw.run(sub, o, a, b, state=state)
                    return 0
            ms, per = timed_steps(torch, dd, world, stream, [call], 3, 2)
            carry = int(c.item()) if world == 1 else None
            res["sub" if sub else "add"] = {"ms": ms, "gbs": 24 * M5 / (ms * 1e-3) / 1e9,
                                            "frac_hbm_per_gpu": 24 * M5 / world / (ms * 1e-3) / 1e9 / hbm_peak,
                                            "carry": carry}
            del a, b, o
            torch.cuda.empty_cache()
        out["C5"] = {"metric": "one 2^30-limb add/sub GB/s (whole number, all GPUs)", "unit": "GB/s",
                     "n_limbs": M5, "shard_limbs": n_local, "run": list(W.C5_RUN),
                     "mode": "single GPU tiled path" if world == 1 else
                             f"{world} limb-range shards, NCCL all_gather of 8-byte (G,P) per rank",
                     **res}
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
