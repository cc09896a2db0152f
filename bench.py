#!/usr/bin/env python
"""bench.py -- throughput of the B200 elementwise primality path (arXiv
2108.04791 "isprime_fast") in Gints/s, one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N

A step is one isprime_device() call over one batch: plan -> sieve -> classify
(trial division + compaction) -> Miller-Rabin base 2 -> remaining bases, every
row of SURVEY.md 8(a).  The headline workload is BASELINE.json configs[4]
("C5": n = 2^28 mixed magnitudes with Chernick and 2^64-59 inserts), the one
configuration that exercises every row in a single step; C1-C4 are reported
under "per_config".  Multi-GPU is weak scaling: rank r classifies generator
indices [r n, (r+1) n) with no collective on the path (NCCL only reduces the
prime count and the max time).  Inputs are 2 GiB per step (> 126 MB L2), so L2
is not flushed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

METRIC = "Gints/sec classified (1/2/4/8 B200) per magnitude class; % of IMAD or HBM roofline"
UNIT = "Gints/s"
# Minimal pipe work of one modular multiplication, in lane-slots of a 16-lane
# pipe: IMAD.WIDE.U32 and IMAD.HI are half rate on the
# FMA-heavy pipe (profiles/r1_imad_peak.json: 25.2 / 31.7 vs 63.2 lanes/clk/SM
# for IMAD), so they count 2 slots.
#   64-bit Montgomery: 4 WIDE (a*b) + 1 WIDE + 2 IMAD (m) + 4 WIDE (hi(m n)) -> 18 FMA-heavy slots
#     (a squaring needs 3 WIDE for a^2 -> 16; the multiply count below does not
#      separate squarings, so 18 is a conservative, i.e. higher, work figure)
#   32-bit Montgomery: 1 WIDE + 1 IMAD + 1 HI -> 5 FMA-heavy slots
#   FP64 (n < 2^51), lazy signed residues: DMUL (h), DFMA (l), DFMA + DADD (q), DFMA + DADD (r)
#     -> 6 FP64 lane-ops (modmath.cuh fmul_lazy)
# The 32-bit class runs on the FP64 pipe too (csrc/kernels.cuh CLS32_FP64 = 1).
SLOTS_MULMOD64 = 18
SLOTS_MULMOD32 = 5
FP64_OPS_MULMOD = 6
CLS32_ON_FP64 = True
LANES_PER_CLK_SM = 64  # FMA-heavy and FP64 pipes: 16 lanes/clk per SMSP x 4 (B300_MICROARCH.md; measured 63.2 / 63.1)
HBM_BYTES_PER_ELEM = 9      # 8-B value read + 1-B result written


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev: int):
        self.dev = dev
        self.samples = []
        self.proc = None
        self.thread = None
        self.marks = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.perf_counter(), line.strip()))

    def mark(self):
        self.marks.append(time.perf_counter())

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        if len(self.marks) >= 2:
            t0, t1 = self.marks[0], self.marks[-1]
            rows = [s for t, s in self.samples if t0 <= t <= t1 + 0.05]
        if not rows:  # timed region shorter than the sampling interval: nearest samples under load
            rows = [s for _, s in self.samples[-5:]]
        sm, smax, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in rows:
            parts = [p.strip() for p in r.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = max(smax, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def load_counts():
    out = {}
    with open(os.path.join(ROOT, "tests", "golden", "config_counts.txt")) as f:
        for line in f:
            line = line.split("#", 1)[0].split()
            if line:
                out[line[0]] = int(line[2])
    out["C4"] = 203280221  # pi(2^32)
    return out


def make_input(cfg, rank, torch, dev):
    """Rank's batch on the device (weak scaling: generator indices [r n, (r+1) n))."""
    n = workloads.CONFIGS[cfg][1]
    if cfg == "C4":
        if rank != 0:
            raise SystemExit("C4 is the fixed range 0..2^32-1; run it at --gpus 1")
        return torch.arange(n, dtype=torch.int64, device=dev), None
    host = workloads.generate(cfg, start=rank * n, count=n)
    ht = torch.from_numpy(host.view(np.int64))
    return ht.to(dev), host


L2_BYTES = 126 * 2**20
_flush_buf = None


def l2_flush_needed(n):
    """Inputs smaller than a few L2s could stay resident between steps."""
    return n * 8 < 4 * L2_BYTES


def time_steps_flushed(isp, torch, dN, dout, n, steps, warmup, stream):
    """Per-step CUDA events with an L2 flush (a 512 MB write on the same
    stream) between steps, outside the events: every step starts cold."""
    global _flush_buf
    if _flush_buf is None:
        _flush_buf = torch.empty(512 * 2**20, dtype=torch.uint8, device=dN.device)
    for _ in range(warmup):
        isp.isprime_device(dN, dout, n, stream)
    torch.cuda.synchronize()
    l0 = isp.get_stats()["kernel_launches"]
    evs = []
    with torch.cuda.stream(stream):
        for _ in range(steps):
            _flush_buf.fill_(1)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            isp.isprime_device(dN, dout, n, stream)
            e1.record(stream)
            evs.append((e0, e1))
    torch.cuda.synchronize()
    launches = isp.get_stats()["kernel_launches"] - l0
    return sum(a.elapsed_time(b) for a, b in evs) / steps, launches


def time_steps(isp, torch, dN, dout, n, steps, warmup, stream, dist, sampler=None):
    for _ in range(warmup):
        isp.isprime_device(dN, dout, n, stream)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    l0 = isp.get_stats()["kernel_launches"]
    if sampler:
        sampler.mark()
    e0.record(stream)
    for _ in range(steps):
        isp.isprime_device(dN, dout, n, stream)
    e1.record(stream)
    torch.cuda.synchronize()
    if sampler:
        sampler.mark()
    if dist is not None:
        dist.barrier()
    launches = isp.get_stats()["kernel_launches"] - l0
    return e0.elapsed_time(e1) / steps, launches


def kernel_profile(isp, torch, dN, dout, n, steps, stream):
    """Instrumented pass (events around every launch + algorithmic work counters)."""
    isp.set_option("kernel_timing", 1)
    isp.reset_kernel_times()
    isp.reset_stats()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        isp.isprime_device(dN, dout, n, stream)
    e1.record(stream)
    torch.cuda.synchronize()
    kt = isp.get_kernel_times()
    st = isp.get_stats()
    isp.set_option("kernel_timing", 0)
    step_ms = e0.elapsed_time(e1) / steps
    per_step = {k: v[1] / steps for k, v in kt.items() if v[0] > 0}
    return per_step, st, step_ms


def roofline(kern_ms, stats, n, steps, peaks, peaks_kind, clocks, cfg=None):
    """Roofline of the dominant kernel (largest share of the step)."""
    if not kern_ms:
        return None
    name = max(kern_ms, key=kern_ms.get)
    ms = kern_ms[name]
    traffic, ncu = None, None
    tpath = os.path.join(ROOT, "profiles", "ncu_kernel_metrics.json")
    if os.path.exists(tpath):
        try:
            allm = json.load(open(tpath))
            # the capture of this kernel on this configuration only
            ncu = allm.get(f"{name}@{cfg}")
            traffic = ncu["dram_bytes_per_launch"] if ncu else None
        except Exception:
            traffic, ncu = None, None
    if name in ("mr1", "mr2"):
        mm, mf = stats["mulmods"], stats["mulmods_fp64"]
        k = 0 if name == "mr1" else 2
        fma_slots = (0 if CLS32_ON_FP64 else mm[k] * SLOTS_MULMOD32) + mm[k + 1] * SLOTS_MULMOD64
        fp64_ops = (mf[0 if name == "mr1" else 1] + (mm[k] if CLS32_ON_FP64 else 0)) * FP64_OPS_MULMOD
        busiest = max(fma_slots, fp64_ops)
        achieved = busiest / steps / (ms * 1e-3) / 1e12
        mhz = peaks.get("sm_max_mhz", 1965.0)
        peak = 148 * LANES_PER_CLK_SM * mhz * 1e6 / 1e12
        per_pipe = {"fmaheavy": round(fma_slots / steps / (ms * 1e-3) / 1e12 / peak, 4),
                    "fp64": round(fp64_ops / steps / (ms * 1e-3) / 1e12 / peak, 4)}
        return {"kernel": name, "bound": "alu", "achieved": round(achieved, 4), "peak": round(peak, 3),
                "unit": "T lane-slots/s (busiest of FMA-heavy / FP64 pipe)", "frac": round(achieved / peak, 4),
                "frac_per_pipe": per_pipe,
                "traffic": traffic, "ncu": ncu,
                "peak_source": f"derived: 148 SMs x {LANES_PER_CLK_SM} lanes/clk x {mhz:.0f} MHz "
                               "(B300_MICROARCH.md pipe rates; MEASURED_PEAKS sm_max_mhz)",
                "work": f"per step: {fma_slots / steps:.4g} FMA-heavy slots ({SLOTS_MULMOD64}/64-bit Montgomery mulmod) "
                        f"and {fp64_ops / steps:.4g} FP64 ops ({FP64_OPS_MULMOD}/mulmod of the FP64 and 32-bit classes); "
                        "mulmods = square-and-multiply count of ModExp",
                "ms_per_step": round(ms, 4)}
    nbytes = HBM_BYTES_PER_ELEM * n
    if name == "dense":   # fused sieve + gather of a dense range: reads N, writes out
        nbytes = HBM_BYTES_PER_ELEM * n
    elif name == "sieve":
        nbytes = stats["sieved_integers"] / steps / 16.0 if stats["sieved_integers"] else 0.0
    elif name not in ("classify", "dense"):
        nbytes = n
    achieved = nbytes / (ms * 1e-3) / 1e9
    peak = float(peaks.get("hbm_gbs", 6650.0))
    return {"kernel": name, "bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic, "ncu": ncu, "peak_source": f"{peaks_kind} hbm_gbs",
            "work": f"{nbytes:.4g} algorithmic bytes per step", "ms_per_step": round(ms, 4)}


def cpu_baseline_run(cfg, host, sample_n):
    import oracle  # test infrastructure: the cpu_baseline leg only
    if host is None:
        sample = np.arange(sample_n, dtype=np.uint64)
    else:
        sample = host[:sample_n]
    threads = os.cpu_count() or 1
    t = time.perf_counter()
    out = oracle.isprime(sample, threads=threads)
    dt = time.perf_counter() - t
    return {"value": round(sample.shape[0] / dt / 1e9, 6), "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"first {sample.shape[0]} elements of {cfg} ({dt:.2f} s wall, {int(out.sum())} primes)"}


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle (this tier's reference arm), rank 0 only."""
    if rank != 0:
        return
    import oracle
    cfg = args.config
    n = workloads.CONFIGS[cfg][1]
    sample_n = min(n, args.ref_sample)
    if cfg == "C4":
        sample = np.arange(sample_n, dtype=np.uint64)
    else:
        sample = workloads.generate(cfg, count=sample_n)
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        oracle.isprime(sample, threads=threads)
    t = time.perf_counter()
    for _ in range(args.steps):
        oracle.isprime(sample, threads=threads)
    dt = (time.perf_counter() - t) / args.steps
    value = sample_n / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": config_block(cfg, world),
        "cpu_baseline": {"value": round(value, 6), "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": f"first {sample_n} elements of {cfg} per step"},
        "e2e": {"value": round(value, 6), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def witness_option(isp, torch, dev, stream, args, counts, mode, cfgs):
    """Another exact witness mode on the same workloads with the same timing;
    the headline above is the paper's Eq 4 method.  mode 1: Baillie-PSW (a
    strong Lucas test replaces the six remaining Eq 4 bases for n >= 2^49, the
    paper's proposed next step); mode 2: reduced witness sets
    by magnitude (base 2 + one hashed base below 2^32,
    Jaeschke's four bases below 1,122,004,669,633)."""
    res = {}
    isp.set_option("witness", mode)
    try:
        for c in cfgs:
            cn = workloads.CONFIGS[c][1]
            cN, _ = make_input(c, 0, torch, dev)
            cout = torch.empty(cn, dtype=torch.uint8, device=dev)
            if l2_flush_needed(cn):
                cms, _ = time_steps_flushed(isp, torch, cN, cout, cn, args.steps, args.warmup, stream)
            else:
                cms, _ = time_steps(isp, torch, cN, cout, cn, args.steps, args.warmup, stream, None)
            dcount = torch.zeros(1, dtype=torch.int64, device=dev)
            isp.isprime_popcount_device(cout, dcount, cn, stream)
            torch.cuda.synchronize()
            res[c] = {"value": round(cn / (cms * 1e-3) / 1e9, 4), "unit": UNIT, "ms_per_step": round(cms, 4),
                      "correct": int(dcount.item()) == counts[c]}
            del cN, cout
            torch.cuda.empty_cache()
    finally:
        isp.set_option("witness", 0)
    return res


def scalar_latency(isp, torch, dev, stream):
    """Per-call latency for one scalar (the paper's Tables 4, 6 and 7 time a
    single 64-bit prime): the device call on a
    resident value (CUDA events) and the host C-ABI isprime() call on a
    one-element host array (wall clock, H2D + D2H included).  Median of 200."""
    vals = {"2^64-59 (prime)": (1 << 64) - 59, "2^52-47 (prime)": (1 << 52) - 47, "2^31-1 (prime)": (1 << 31) - 1}
    res = {}
    for name, v in vals.items():
        host = np.array([v], dtype=np.uint64)
        dN = torch.from_numpy(host.view(np.int64)).to(dev)
        dout = torch.empty(1, dtype=torch.uint8, device=dev)
        ts, tw = [], []
        for k in range(220):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            isp.isprime_device(dN, dout, 1, stream)
            e1.record(stream)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out = isp.isprime(host)
            t1 = time.perf_counter()
            if k >= 20:
                ts.append(e0.elapsed_time(e1) * 1e3)
                tw.append((t1 - t0) * 1e6)
        assert int(out[0]) == 1 and int(dout.item()) == 1
        res[name] = {"device_us": round(float(np.median(ts)), 2), "host_api_us": round(float(np.median(tw)), 2)}
    return res


def config_block(cfg, world):
    n = workloads.CONFIGS[cfg][1]
    return {"workload": f"{cfg}: {workloads.CONFIGS[cfg][2]} (BASELINE.json configs[{int(cfg[1]) - 1}])",
            "n_per_rank": n, "global_n": n * world, "parallelism": f"dp{world} (contiguous shards, no collective)",
            "l2": "no flush: inputs larger than L2 (%.2f GiB per step)" % (n * 8 / 2**30)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5", choices=sorted(workloads.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-per-config", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=1 << 24)
    ap.add_argument("--ref-sample", type=int, default=1 << 22)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local = _env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as tdist
    import paper_2108_04791_b200 as isp

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        tdist.init_process_group("nccl", device_id=dev)
        dist = tdist
    isp.load(build_if_missing=False)
    stream = torch.cuda.current_stream()
    peaks, peaks_kind = measured_peaks()
    counts = load_counts()

    cfg = args.config
    n = workloads.CONFIGS[cfg][1]
    dN, host = make_input(cfg, rank, torch, dev)
    dout = torch.empty(n, dtype=torch.uint8, device=dev)

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.2)
    ms, launches = time_steps(isp, torch, dN, dout, n, args.steps, args.warmup, stream, dist, sampler)
    sampler.stop()
    clocks = sampler.summary()

    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(t, op=tdist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * n / (ms_max * 1e-3) / 1e9

    # validation: count per rank -> NCCL sum
    dcount = torch.zeros(1, dtype=torch.int64, device=dev)
    isp.isprime_popcount_device(dout, dcount, n, stream)
    torch.cuda.synchronize()
    my_count = int(dcount.item())
    tot = dcount.clone()
    if dist:
        dist.all_reduce(tot)
    total_count = int(tot.item())
    correct = (my_count == counts[cfg]) if rank == 0 else None

    kern_ms, st, inst_ms = kernel_profile(isp, torch, dN, dout, n, args.steps, stream)
    roof = roofline(kern_ms, st, n, args.steps, peaks, peaks_kind, clocks, cfg)

    e2e = None
    if not args.no_e2e:
        if host is None:
            hN = torch.arange(n, dtype=torch.int64).pin_memory()
        else:
            hN = torch.from_numpy(host.view(np.int64)).pin_memory()
        hout = torch.empty(n, dtype=torch.uint8).pin_memory()
        for _ in range(1):
            isp.isprime_into(hN, hout)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        esteps = max(1, min(args.steps, 5))
        for _ in range(esteps):
            isp.isprime_into(hN, hout)
        et = torch.tensor([(time.perf_counter() - t0) / esteps], dtype=torch.float64, device=dev)
        if dist:
            dist.all_reduce(et, op=tdist.ReduceOp.MAX)
        e2e = {"value": round(world * n / float(et.item()) / 1e9, 4), "unit": UNIT,
               "h2d_bytes_per_step": int(n * 8), "d2h_bytes_per_step": int(n),
               "ms_per_step": round(float(et.item()) * 1e3, 3),
               "how": "isprime() host C-ABI on pinned host buffers; host wall clock around the synchronous call",
               "matches_device": bool(np.array_equal(hout.numpy(), dout.cpu().numpy()))}
        del hN, hout

    line = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_max, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic (seeded generator, SURVEY.md 8(d))",
        "config": config_block(cfg, world),
        "roofline": roof, "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks,
        "kernels_ms_per_step": {k: round(v, 4) for k, v in kern_ms.items()},
        "instrumented_ms_per_step": round(inst_ms, 4),
        "prime_count": {"rank0": my_count, "total": total_count, "expected_rank0": counts[cfg], "correct": correct},
        "stats_per_step": {k: (v / args.steps if isinstance(v, int) else [x / args.steps for x in v])
                           for k, v in st.items() if k not in ("window_lo", "window_hi", "kernel_launches")},
    }
    del dN, dout
    torch.cuda.empty_cache()

    if rank == 0 and world == 1:
        line["cpu_baseline"] = cpu_baseline_run(cfg, host, min(n, args.cpu_sample))
        if not args.no_per_config:
            per = {}
            for c in ("C1", "C2", "C3", "C4"):
                if c == cfg:
                    continue
                cn = workloads.CONFIGS[c][1]
                cN, _ = make_input(c, 0, torch, dev)
                cout = torch.empty(cn, dtype=torch.uint8, device=dev)
                csteps = args.steps if c != "C1" else max(args.steps, 100)
                flushed = l2_flush_needed(cn)
                if flushed:
                    cms, cl = time_steps_flushed(isp, torch, cN, cout, cn, csteps, args.warmup, stream)
                else:
                    cms, cl = time_steps(isp, torch, cN, cout, cn, csteps, args.warmup, stream, None)
                isp.isprime_popcount_device(cout, dcount, cn, stream)
                torch.cuda.synchronize()
                ckm, cst, _ = kernel_profile(isp, torch, cN, cout, cn, csteps, stream)
                croof = roofline(ckm, cst, cn, csteps, peaks, peaks_kind, clocks, c)
                per[c] = {"value": round(cn / (cms * 1e-3) / 1e9, 4), "unit": UNIT, "ms_per_step": round(cms, 4),
                          "n": cn, "correct": int(dcount.item()) == counts[c], "gpu_launches_per_step": cl / csteps,
                          "l2": ("flushed between steps (512 MB write outside per-step CUDA events)" if flushed
                                 else "no flush: inputs larger than L2"),
                          "kernels_ms_per_step": {k: round(v, 4) for k, v in ckm.items()}, "roofline": croof}
                del cN, cout
                torch.cuda.empty_cache()
            line["per_config"] = per
        line["scalar_latency"] = scalar_latency(isp, torch, dev, stream)
        line["witness_bpsw"] = witness_option(isp, torch, dev, stream, args, counts, 1, ("C5", "C3"))
        line["witness_reduced"] = witness_option(isp, torch, dev, stream, args, counts, 2, ("C5", "C2"))
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
