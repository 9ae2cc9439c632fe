#!/usr/bin/env python3
"""Benchmark for the B200 batched FFT (+ fused ABFT) — the driver's contract.

    python bench.py --gpus N --steps K --warmup W [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)

Headline workload (BASELINE.json configs[1], "C2"): FP64 complex 1-D forward
FFT sweep N = 2^8 .. 2^20, each with B = 2^26 / N signals (1 GiB in, 1 GiB
out, both larger than the 126 MB L2, so no flush is needed). One step = the
13 transforms of the sweep. ``value`` = algorithmic GFLOP/s (5 N log2 N per
transform) over the whole job (all ranks), inputs resident in HBM; ``e2e`` =
the same metric through the public API (execute_plan on pinned host numpy
batches: H2D + kernels + D2H inside the timed region). Weak scaling: every
rank transforms its own 1 GiB shard per N; no data crosses NVLink.

Extra keys: per-N GB/s and roofline fractions, the fused-ABFT overhead on
C3 (N = 4096, 1 GiB, T = 8) and C5 (N = 2^16, 2048 signals/GPU, T = 8, with
the NCCL fault-counter all-reduce when N > 1), clocks sampled during the
timed region, the dominant kernel's roofline, and the reference CPU path
timed on this host.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FLOP = lambda n: 5.0 * n * np.log2(n)  # noqa: E731


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--sweep", default="8-20", help="log2 N range of the C2 sweep")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-abft", action="store_true")
    ap.add_argument("--cpu-fraction", type=float, default=0.25,
                    help="fraction of each N's batch the CPU baseline transforms")
    return ap.parse_args()


def sweep_sizes(spec):
    a, b = (int(v) for v in spec.split("-"))
    return [2 ** k for k in range(a, b + 1)]


# ---------------------------------------------------------------------------
# distributed plumbing


class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None

    def init(self, device_backend=True):
        import torch
        import torch.distributed as dist

        if device_backend:
            torch.cuda.set_device(self.local)
        if self.world > 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            if device_backend:  # eager NCCL communicator (its handle feeds tfft_allreduce_stats)
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
                dist.barrier()
            else:
                dist.init_process_group("gloo")
            self.pg = dist
        return self

    def barrier(self):
        if self.pg is not None:
            self.pg.barrier()

    def max(self, v):
        if self.pg is None:
            return v
        import torch

        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, v):
        if self.pg is None:
            return v
        import torch

        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        self.pg.all_reduce(t)
        return float(t.item())

    def close(self):
        if self.pg is not None:
            self.pg.destroy_process_group()


# ---------------------------------------------------------------------------
# clocks during the timed region


class Clocks:
    """SM clock and throttle reasons sampled during the timed region: NVML
    polled every 5 ms from a thread (the timed region is tens of ms), with
    nvidia-smi (-lms 50) as the fallback."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self.thread = None
        self.proc = None

    def start(self):
        try:
            import threading

            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self.stop_evt = threading.Event()

            def poll():
                while not self.stop_evt.is_set():
                    self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                    try:
                        bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    except Exception:  # older bindings
                        bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                    for name, attr in self.REASONS:
                        if bits & getattr(nv, attr, 0):
                            self.reasons.add(name)
                    self.stop_evt.wait(0.005)

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
        except Exception:
            self.thread = None
            self._start_smi()

    def _start_smi(self):
        fields = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                  "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                  "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        self.path = ROOT / "gpurun_out" / f"clocks_rank{self.index}.csv"
        try:
            self.path.parent.mkdir(exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={fields}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=self.fh, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.thread is not None:
            self.stop_evt.set()
            self.thread.join(timeout=2)
            sm = self.samples
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                    "reasons": sorted(self.reasons), "samples": len(sm), "source": "nvml 5 ms"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        self.proc.terminate()
        self.proc.wait(timeout=5)
        self.fh.close()
        sm, mx, reasons = [], [], set()
        for line in self.path.read_text().splitlines():
            f = [v.strip() for v in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for (name, _), val in zip(self.REASONS, f[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi 50 ms"}


# ---------------------------------------------------------------------------
# our arm


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def run_ours(args, dist):
    import torch

    import paper_2412_05824_b200 as tf
    from paper_2412_05824_b200 import _lib, abft as A, fft_core

    lib = _lib.load()
    sizes = sweep_sizes(args.sweep)
    total_elems = 2 ** 26  # 1 GiB of complex128 per rank per N
    x = torch.randn(total_elems * 2, dtype=torch.float64, device="cuda").view(torch.complex128)
    y = torch.empty_like(x)
    plans = {n: tf.build_plan(tf.select_params(n, total_elems // n, "double"), "double") for n in sizes}
    for n in sizes:  # plan creation (twiddle upload) outside the timed region
        fft_core.device_execute(plans[n], x.view(-1, n)[:1], y.view(-1, n)[:1])
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()

    def step(events=None):
        for i, n in enumerate(sizes):
            if events is not None:
                events[i][0].record(stream)
            fft_core.device_execute(plans[n], x.view(-1, n), y.view(-1, n))
            if events is not None:
                events[i][1].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    per_n = [[] for _ in sizes]
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in sizes]
          for _ in range(args.steps)]
    clocks = Clocks(dist.local)
    dist.barrier()
    torch.cuda.synchronize()
    launches0 = lib.tfft_launch_count()
    clocks.start()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for s in range(args.steps):
        step(ev[s])
    t1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop()
    launches = lib.tfft_launch_count() - launches0
    elapsed = t0.elapsed_time(t1) / 1e3
    for s in range(args.steps):
        for i in range(len(sizes)):
            per_n[i].append(ev[s][i][0].elapsed_time(ev[s][i][1]) / 1e3)
    elapsed = dist.max(elapsed)
    flops_rank = sum(FLOP(n) * (total_elems // n) for n in sizes)
    value = flops_rank * dist.world * args.steps / elapsed / 1e9
    peak, peak_src = peaks()
    sweep = []
    for i, n in enumerate(sizes):
        t = statistics.median(per_n[i])
        b = total_elems // n
        gbs = 2 * n * b * 16 / t / 1e9
        sweep.append({"n": n, "batch": b, "ms": round(t * 1e3, 4), "gflops": round(FLOP(n) * b / t / 1e9, 1),
                      "gbs": round(gbs, 1), "hbm_frac": round(gbs / peak, 4),
                      "kernel": _kernel_label("double", n)})
    dom = max(range(len(sizes)), key=lambda i: statistics.mean(per_n[i]))
    dn = sweep[dom]
    roofline = {"bound": "hbm", "achieved": dn["gbs"], "peak": peak, "unit": "GB/s",
                "frac": round(dn["gbs"] / peak, 4), "traffic": None,
                "kernel": f"{dn['kernel']} (N={dn['n']}, B={dn['batch']})",
                "algorithmic_bytes_per_launch": 2 * dn["n"] * dn["batch"] * 16,
                "peak_source": peak_src}
    prof = ROOT / "profiles" / "traffic.json"
    if prof.exists():
        tr = json.loads(prof.read_text()).get(str(dn["n"]))
        if tr:
            roofline["traffic"] = tr["bytes"] if isinstance(tr, dict) else tr
            roofline["traffic_unit"] = "bytes per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum)"

    out = {
        "metric": "FFT GFLOP/s (5 N log2 N per transform), C2 FP64 sweep N=2^8..2^20",
        "value": round(value, 1), "unit": "GFLOP/s", "n_gpus": dist.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(elapsed / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64 (complex128)", "data": "synthetic (torch.randn)",
        "config": {"workload": "C2: FP64 complex 1-D forward FFT, N=2^8..2^20, B=2^26/N (1 GiB in per N per GPU)",
                   "transforms_per_step": len(sizes), "bytes_per_step_per_gpu": 2 * total_elems * 16 * len(sizes),
                   "l2": "inputs 1 GiB > 126 MB L2 (no flush needed)", "parallelism": f"batch-shard x{dist.world}"},
        "gb_per_s": round(2 * total_elems * 16 * len(sizes) * dist.world * args.steps / elapsed / 1e9, 1),
        "sweep": sweep, "roofline": roofline, "clocks": clk, "gpu_launches": int(launches),
    }
    del x, y
    torch.cuda.empty_cache()
    out["sweep_fp32"] = fp32_sweep(args, dist, peak)
    if not args.no_abft:
        out["abft"] = abft_overheads(args, dist)
        out["abft_T_sweep"] = abft_t_sweep(args, dist)
        out["c4"] = c4_config(args, dist, peak)
    out["c1"] = c1_config(args, dist)
    if not args.no_e2e:
        out["e2e"] = e2e(args, dist, sizes, plans, total_elems)
    return out


def _time_loop(fn, steps, warmup, dist):
    import torch

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    torch.cuda.synchronize()
    dist.barrier()
    return dist.max(a.elapsed_time(b) / 1e3 / steps)


def abft_overheads(args, dist):
    """Fused two-sided ABFT overhead: C3 (N=4096) and C5 (N=2^16) at T=8."""
    import torch

    import paper_2412_05824_b200 as tf
    from paper_2412_05824_b200 import _lib, abft as A, fft_core, shard

    res = {}
    cases = [("C3_fp32_n4096", 4096, 32768, "single", 8), ("C3_fp64_n4096", 4096, 16384, "double", 8),
             ("C5_fp32_n65536", 65536, 2048, "single", 8)]
    for name, n, b, prec, T in cases:
        dt = torch.complex64 if prec == "single" else torch.complex128
        rdt = torch.float32 if prec == "single" else torch.float64
        x = torch.randn(b * n * 2, dtype=rdt, device="cuda").view(dt).view(b, n)
        y = torch.empty_like(x)
        plan = tf.build_plan(tf.select_params(n, b, prec), prec)
        ntx = -(-b // plan.bs)
        nwin = -(-ntx // T)
        sums = A._DeviceSums(b, nwin)
        ctr = fft_core._Counters()
        delta = A.default_delta(prec)
        offset = dist.rank * b  # global signal indices of this shard (weights w_j = j + 1)

        def plain():
            fft_core.device_execute(plan, x, y)

        comm = shard._nccl_comm(dist.pg, "cuda") if dist.pg is not None else None
        lib = _lib.load()

        def fused():
            A.protected_device(plan, x, y, delta=delta, group_size=T, counters=ctr, sums=sums,
                               signal_offset=offset)
            if comm is not None:
                # the only collective: the triggered-signal count (int64 SUM) and
                # the max divergence (its non-negative double bits, MAX) over
                # NVLink, in one grouped NCCL launch on this stream
                d = ctr.dev
                rc = lib.tfft_allreduce_stats(d.data_ptr() + 8, 1, d.data_ptr() + 16, comm,
                                              torch.cuda.current_stream().cuda_stream)
                _lib.check(rc, "tfft_allreduce_stats")

        steps = max(args.steps, 5)
        tp = _time_loop(plain, steps, args.warmup, dist)
        tfz = _time_loop(fused, steps, args.warmup, dist)
        gbs = 2 * n * b * (8 if prec == "single" else 16) / tp / 1e9
        api = None
        if name.startswith("C5"):
            api = c5_public_api(plan, x, b, T, dist, steps, args.warmup)
        inj = injected_api(plan, x, b, T, prec, dist)
        res[name] = {"n": n, "batch_per_gpu": b, "T": T, "bs": plan.bs, "plain_ms": round(tp * 1e3, 4),
                     "fused_ms": round(tfz * 1e3, 4), "overhead_pct": round(100 * (tfz / tp - 1), 2),
                     "plain_gbs": round(gbs, 1),
                     "path": "K5 with fused two-sided ABFT (window sums in TMEM) + one window-finisher launch"
                             if n <= 4096 else ("K7" if prec == "double" else "K4") + " transform + one-sweep checksums"}
        if api is not None:
            res[name]["public_api"] = api
        res[name]["injected"] = inj
        del x, y, sums
        torch.cuda.empty_cache()
    return res


def _kernel_label(prec, n):
    logn = int(np.log2(n))
    if logn <= 8:
        return "k1_single_pass"
    if logn <= (13 if prec == "single" else 12):
        return "k5_single_pass"
    if logn <= 22:
        return ("k7" if logn <= 20 else "k4/k3") + "_two_pass"
    return "stage_passes"


def fp32_sweep(args, dist, peak):
    """FP32 N=2^8..2^20 at 1 GiB per N (north_star: FP32 and FP64 2^8..2^20),
    device-resident, CUDA events, median of the timed steps."""
    import torch

    import paper_2412_05824_b200 as tf
    from paper_2412_05824_b200 import fft_core

    total = 2 ** 27  # complex64 elements = 1 GiB
    x = torch.randn(total * 2, dtype=torch.float32, device="cuda").view(torch.complex64)
    y = torch.empty_like(x)
    rows = []
    for n in sweep_sizes(args.sweep):
        b = total // n
        plan = tf.build_plan(tf.select_params(n, b, "single"), "single")
        xv, yv = x.view(-1, n), y.view(-1, n)
        t = _time_loop(lambda: fft_core.device_execute(plan, xv, yv), max(args.steps, 5), args.warmup, dist)
        gbs = 2 * n * b * 8 / t / 1e9
        rows.append({"n": n, "batch": b, "ms": round(t * 1e3, 4), "gflops": round(FLOP(n) * b / t / 1e9, 1),
                     "gbs": round(gbs, 1), "hbm_frac": round(gbs / peak, 4), "kernel": _kernel_label("single", n)})
    del x, y
    torch.cuda.empty_cache()
    return rows


def abft_t_sweep(args, dist):
    """C3 (N=4096, 1 GiB, fault-free) fused-ABFT overhead for T in {1,2,4,8,16,32}."""
    import torch

    import paper_2412_05824_b200 as tf
    from paper_2412_05824_b200 import abft as A, fft_core

    res = {}
    for prec, b in (("single", 32768), ("double", 16384)):
        dt = torch.complex64 if prec == "single" else torch.complex128
        rdt = torch.float32 if prec == "single" else torch.float64
        n = 4096
        x = torch.randn(b * n * 2, dtype=rdt, device="cuda").view(dt).view(b, n)
        y = torch.empty_like(x)
        plan = tf.build_plan(tf.select_params(n, b, prec), prec)
        tp = _time_loop(lambda: fft_core.device_execute(plan, x, y), max(args.steps, 5), args.warmup, dist)
        row = {"plain_ms": round(tp * 1e3, 4)}
        for T in (1, 2, 4, 8, 16, 32):
            nwin = -(-(-(-b // plan.bs)) // T)
            sums = A._DeviceSums(b, nwin)
            delta = A.default_delta(prec)
            tf_ = _time_loop(lambda: A.protected_device(plan, x, y, delta=delta, group_size=T,
                                                        counters=sums.counters, sums=sums),
                             max(args.steps, 5), args.warmup, dist)
            row[f"T{T}"] = {"ms": round(tf_ * 1e3, 4), "overhead_pct": round(100 * (tf_ / tp - 1), 2)}
        res[f"C3_{'fp32' if prec == 'single' else 'fp64'}_n4096"] = row
        del x, y
        torch.cuda.empty_cache()
    return res


def c4_config(args, dist, peak):
    """C4: large N under injection. N=2^22 (two stages, bs=1) and 2^23 (three
    stages, curated (256,128,256) bs=16), FP32 and FP64, 2 GiB in. Clean: plain
    vs protected (device). Injected: run_protected through the public API on
    the device batch with one exponent/mantissa fault per verification window
    (T=2 at 2^22: 32 FP32 / 16 FP64 injections), wall clock of the whole call
    (transform, checksums, host replay, corrections or recomputations)."""
    import torch

    import paper_2412_05824_b200 as tf
    from paper_2412_05824_b200 import abft as A, fft_core

    out = {}
    for logn in (22, 23):
        n = 2 ** logn
        for prec, bpc in (("single", 8), ("double", 16)):
            b = 2 ** 31 // (n * bpc)
            dt = torch.complex64 if prec == "single" else torch.complex128
            rdt = torch.float32 if prec == "single" else torch.float64
            x = torch.randn(b * n * 2, dtype=rdt, device="cuda").view(dt).view(b, n)
            y = torch.empty_like(x)
            plan = tf.build_plan(tf.select_params(n, b, prec), prec)
            T = 2 if logn == 22 else 1
            nwin = -(-(-(-b // plan.bs)) // T)
            sums = A._DeviceSums(b, nwin)
            delta = A.default_delta(prec)
            steps = max(2, min(args.steps, 5))
            tp = _time_loop(lambda: fft_core.device_execute(plan, x, y), steps, 1, dist)
            tq = _time_loop(lambda: A.protected_device(plan, x, y, delta=delta, group_size=T,
                                                       counters=sums.counters, sums=sums), steps, 1, dist)
            gbs = 2 * n * b * bpc / tp / 1e9
            row = {"n": n, "batch": b, "bs": plan.bs, "stages": [st.span for st in plan.stages], "T": T, "plain_ms": round(tp * 1e3, 3), "plain_gbs": round(gbs, 1),
                   "hbm_frac": round(gbs / peak, 4), "protected_clean_ms": round(tq * 1e3, 3),
                   "clean_overhead_pct": round(100 * (tq / tp - 1), 2), "path": _kernel_label(prec, n)}
            if logn == 22:
                batch = tf.SignalBatch(x)
                rng = np.random.default_rng(0xC4)
                # mantissa-top bit: the per-signal test fires and the fault is corrected online
                bit = 24 if prec == "single" else 51  # FP32: exponent bit 1 (x4 or /4), FP64: mantissa top bit
                specs = []
                for w in range(nwin):
                    tx = w * T + int(rng.integers(0, T))
                    specs.append(tf.FaultSpec(transaction=tx, signal=tx * plan.bs, element=int(rng.integers(0, n)),
                                              stage=int(rng.integers(0, 2)), part="re", bit=bit))
                # warm-up: left row, workspaces and the FP64 correction plan
                # (built on first use) outside the timed calls
                warm = tf.FaultInjector(seu=False)
                for sp in specs:
                    warm.arm(sp, plan=plan, batch=batch)
                tf.run_protected(plan, batch, group_size=T, injector=warm)
                specs = [tf.FaultSpec(**{k: getattr(sp, k) for k in ("transaction", "signal", "element", "stage",
                                                                      "part", "bit")}) for sp in specs]
                torch.cuda.synchronize()
                inj = tf.FaultInjector(seu=False)
                for sp in specs:
                    inj.arm(sp, plan=plan, batch=batch)
                stats = tf.RunStats()
                t0 = time.perf_counter()
                tf.run_protected(plan, batch, group_size=T, injector=inj, stats=stats)
                torch.cuda.synchronize()
                ti = dist.max(time.perf_counter() - t0)
                t0 = time.perf_counter()
                tf.run_protected(plan, batch, group_size=T)
                torch.cuda.synchronize()
                tc = dist.max(time.perf_counter() - t0)
                row["injected"] = {"injections": len(specs), "bit": bit, "events": len(stats.events),
                                   "corrections": stats.corrections, "recomputations": stats.recomputations,
                                   "api_clean_ms": round(tc * 1e3, 2), "api_injected_ms": round(ti * 1e3, 2),
                                   "injection_overhead_pct": round(100 * (ti / tc - 1), 1),
                                   "per_event_ms": round((ti - tc) * 1e3 / max(len(stats.events), 1), 3),
                                   "call": "run_protected(SignalBatch(device tensor), group_size=T, injector)"}
            out[f"{'fp32' if prec == 'single' else 'fp64'}_2p{logn}"] = row
            del x, y, sums
            torch.cuda.empty_cache()
    return out


def injected_api(plan, x, b, T, prec, dist, reps=3):
    """ABFT under injection through the public API (run_protected on the
    device batch): one mantissa-top-bit fault in EVERY verification window
    (stage 0, random element), min wall time of `reps` calls, against the
    same call without faults. Detected faults are corrected online (batched
    correction of single-trigger windows, the serial replay for the rest)."""
    import torch

    import paper_2412_05824_b200 as tf

    n = x.shape[1]
    batch = tf.SignalBatch(x)
    ntx = -(-b // plan.bs)
    nwin = -(-ntx // T)
    rng = np.random.default_rng(0xC3)
    bit = 24 if prec == "single" else 51  # FP32: exponent bit 1 (x4 or /4), FP64: mantissa top bit
    specs = []
    for w in range(nwin):
        tx = min(w * T + int(rng.integers(T)), ntx - 1)
        sig = tx * plan.bs + int(rng.integers(min(plan.bs, b - tx * plan.bs)))
        specs.append(dict(transaction=tx, signal=sig, element=int(rng.integers(n)), stage=0, part="re", bit=bit))

    def injector():
        i = tf.FaultInjector(seu=False)
        for sp in specs:
            i.arm(tf.FaultSpec(**sp), plan=plan, batch=batch)
        return i

    tf.run_protected(plan, batch, group_size=T, injector=injector())  # warm (correction plan, workspaces)
    tc, ti, stats = [], [], None
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tf.run_protected(plan, batch, group_size=T)
        torch.cuda.synchronize()
        tc.append(time.perf_counter() - t0)
        j, stats = injector(), tf.RunStats()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tf.run_protected(plan, batch, group_size=T, injector=j, stats=stats)
        torch.cuda.synchronize()
        ti.append(time.perf_counter() - t0)
    c, i = dist.max(min(tc)), dist.max(min(ti))
    return {"injections": len(specs), "bit": bit, "events": len(stats.events), "corrections": stats.corrections,
            "recomputations": stats.recomputations, "api_clean_ms": round(c * 1e3, 3),
            "api_injected_ms": round(i * 1e3, 3), "injection_overhead_pct": round(100 * (i / c - 1), 1),
            "call": "run_protected(SignalBatch(device tensor), group_size=T[, injector])"}


def c5_public_api(plan, x, b, T, dist, steps, warmup):
    """C5 through the public sharded API (shard.run_protected_sharded on this
    rank's device-resident shard of a world*b-signal batch): transform +
    checksums + decisions + the counter all-reduce (NCCL C ABI when N > 1),
    host synchronisation included. Wall clock per call, max over ranks."""
    import torch
    import torch.distributed as tdist

    import paper_2412_05824_b200 as tf
    from paper_2412_05824_b200 import shard

    world = dist.world
    global_b = b * world
    s0, s1, _ = shard.shard_bounds(global_b, plan.bs, T, world, dist.rank)
    xs = x[: s1 - s0]
    batch = tf.SignalBatch(xs)
    pg = dist.pg if dist.pg is not None else None

    def call():
        if pg is None:
            return tf.run_protected(plan, batch, group_size=T)
        return shard.run_protected_sharded(plan, batch, global_b=global_b, rank=dist.rank, world=world, dist=tdist,
                                           group_size=T, device="cuda", gather_reports=False)

    for _ in range(warmup):
        call()
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        call()
    torch.cuda.synchronize()
    el = dist.max((time.perf_counter() - t0) / steps)
    return {"ms": round(el * 1e3, 4), "global_batch": global_b,
            "call": "shard.run_protected_sharded(device shard, gather_reports=False)" if pg is not None
            else "run_protected(device batch)",
            "collective": "tfft_allreduce_stats (ncclAllReduce int64 SUM + f64 MAX, 48 B)" if pg is not None
            else "none (1 GPU)"}


def c1_config(args, dist):
    """BASELINE configs[0] (the reference's own CPU-runnable case): FP32, N=1024,
    B=4096 (32 MiB in), forward. The batch fits in L2, so a 256 MiB buffer is
    rewritten between timed iterations (L2 flush, outside the events)."""
    import torch

    import paper_2412_05824_b200 as tf
    from paper_2412_05824_b200 import fft_core

    n, b = 1024, 4096
    x = torch.randn(b * n * 2, dtype=torch.float32, device="cuda").view(torch.complex64).view(b, n)
    y = torch.empty_like(x)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    plan = tf.build_plan(tf.select_params(n, b, "single"), "single")
    for _ in range(max(args.warmup, 3)):
        fft_core.device_execute(plan, x, y)
    times = []
    for _ in range(max(args.steps, 5)):
        # flush: write a 256 MB buffer (> L2), then read it back, so the
        # flush's dirty lines are written back here and not during the timed
        # kernel (a write-only flush left ~126 MB of write-back to overlap it)
        flush.fill_(1)
        flush.view(torch.int64).sum()
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fft_core.device_execute(plan, x, y)
        z.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(z) / 1e3)
    t = dist.max(statistics.median(times))
    del x, y, flush
    torch.cuda.empty_cache()
    return {"workload": "C1: FP32 N=1024 B=4096 forward (L2 flushed between iterations: 256 MB written, then read)",
            "ms": round(t * 1e3, 4),
            "gflops": round(FLOP(n) * b / t / 1e9, 1), "gbs": round(2 * n * b * 8 / t / 1e9, 1)}


def e2e(args, dist, sizes, plans, total_elems):
    """Public API with pinned host buffers: H2D + transform + D2H per N."""
    import torch

    import paper_2412_05824_b200 as tf

    host_in = torch.randn(total_elems * 2, dtype=torch.float64).view(torch.complex128).pin_memory()
    host_out = torch.empty(total_elems, dtype=torch.complex128).pin_memory()
    xin, xout = host_in.numpy(), host_out.numpy()

    def step():
        for n in sizes:
            tf.execute_plan(plans[n], tf.SignalBatch(xin.reshape(-1, n)), out=xout.reshape(-1, n))

    steps = max(1, min(args.steps, 3))
    step()  # warm-up (allocator, plan caches)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
    el = dist.max((time.perf_counter() - t0) / steps)
    flops = sum(FLOP(n) * (total_elems // n) for n in sizes) * dist.world
    nbytes = total_elems * 16 * len(sizes)
    return {"value": round(flops / el / 1e9, 2), "unit": "GFLOP/s", "h2d_bytes_per_step": nbytes,
            "d2h_bytes_per_step": nbytes, "steps": steps, "ms_per_step": round(el * 1e3, 2),
            "path": "paper_2412_05824_b200.execute_plan(SignalBatch(pinned numpy), out=pinned numpy)"}


# ---------------------------------------------------------------------------
# the reference's CPU implementation (oracle/_ref compiled kernel, else the port)


def cpu_reference(sizes, fraction, workers, steps=1, warmup=0):
    from oracle import ref_oracle as O

    kind = "reference" if O.use_ref_kernel(True) else "port"
    total = 2 ** 26
    rng = np.random.default_rng(1234)
    batches = {}
    for n in sizes:
        b = max(1, int(total // n * fraction))
        batches[n] = (rng.standard_normal((b, n)) + 1j * rng.standard_normal((b, n))).astype(np.complex128)
    plans = {n: O.select_params(n, batches[n].shape[0], "double") for n in sizes}

    def step():
        for n in sizes:
            O.execute(batches[n], plans[n], workers=workers)

    for _ in range(warmup):
        step()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    flops = sum(FLOP(n) * batches[n].shape[0] for n in sizes)
    sample = (f"C2 sweep N=2^{int(np.log2(sizes[0]))}..2^{int(np.log2(sizes[-1]))}, "
              f"{fraction:g} of each 1 GiB batch (B=2^26/N*{fraction:g}), FP64, forward; "
              f"resilient_fft execute_plan driver restated in oracle/ref_oracle.py")
    return {"value": round(flops / t / 1e9, 3), "unit": "GFLOP/s", "cores": workers, "kind": kind,
            "sample": sample, "seconds": round(t, 2), "cpu": _cpu_model()}


def _cpu_model():
    """The host CPU the baseline ran on (model name, logical CPUs visible)."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return f"{model} ({os.cpu_count()} logical CPUs)"


def run_reference(args, dist):
    if dist.rank != 0:
        return None
    workers = os.cpu_count() or 1
    sizes = sweep_sizes(args.sweep)
    frac = min(args.cpu_fraction, 1.0 / 16)
    cb = cpu_reference(sizes, frac, workers, steps=args.steps, warmup=min(args.warmup, 1))
    return {
        "metric": "FFT GFLOP/s (5 N log2 N per transform), C2 FP64 sweep N=2^8..2^20",
        "value": cb["value"], "unit": "GFLOP/s", "impl": "reference", "n_gpus": max(dist.world, args.gpus),
        "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(cb["seconds"] * 1e3, 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64 (complex128)", "data": "synthetic (numpy normal)",
        "config": {"workload": "C2: FP64 complex 1-D forward FFT, N=2^8..2^20 (bounded CPU sample)",
                   "parallelism": f"host threads x{workers}"},
        "cpu_baseline": cb,
        "e2e": {"value": cb["value"], "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def _spawn_ranks(args):
    """``--gpus N`` without a torchrun environment: re-launch this script
    under torch.distributed.run, one rank per GPU (rank 0 prints the line)."""
    import socket

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        return _spawn_ranks(args)
    dist = Dist()
    if args.impl == "reference":
        out = run_reference(args, dist)
        if out is not None:
            print(json.dumps(out), flush=True)
        return 0
    dist.init()
    if dist.world != args.gpus and dist.rank == 0:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={dist.world}; reporting {dist.world}", file=sys.stderr)
    out = run_ours(args, dist)
    if dist.rank == 0 and not args.no_cpu:
        out["cpu_baseline"] = cpu_reference(sweep_sizes(args.sweep), args.cpu_fraction, 1)
    if dist.rank == 0:
        print(json.dumps(out), flush=True)
    dist.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
