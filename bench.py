#!/usr/bin/env python
"""bench.py -- throughput of the B200 elementwise primality path (arXiv
2108.04791 "isprime_fast") in Gints/s, one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N

A step is one isprime_device() call over one batch: plan -> sieve -> classify
(trial division + compaction) -> Miller-Rabin base 2 -> remaining bases, every
row of SURVEY.md 8(a).  The headline workload is BASELINE.json configs[4]
("C5": n = 2^28 mixed magnitudes with Chernick and 2^64-59 inserts), the one
configuration that exercises every row in a single step; the others are
reported under "per_config".

Multi-GPU: one process per GPU, no collective on the path
(NCCL only reduces the prime count and the max time, outside the timed
region).  --scaling weak (default): rank r classifies generator indices
[r n, (r+1) n); --scaling strong: the fixed array of n elements is split
contiguously, rank r owning [floor(r n / W), floor((r+1) n / W)).  C4 (the
dense range 0 .. 2^32-1) is always split by value: rank r classifies the
device iota [floor(r 2^32 / W), floor((r+1) 2^32 / W)) and sieves only that
window.  Inputs of C3-C5 are >= 0.5 GiB per step (> 126 MB L2) and are not
flushed; C1 / C2 are timed with an L2 flush between steps.
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
# Roofline of the witness kernels.  DFMA and IMAD.WIDE share
# one multiplier pipe on B200 (tools/mont_bench.cu: FP64-product warps and
# Montgomery warps on the same SMs overlap by ~8 %, profiles/r2/mont_bench.json),
# so the bound is ONE heavy pipe of 64 lane-slots/clk/SM, and each instruction
# costs 64 / (its measured lanes/clk/SM) slots (profiles/r1_imad_peak.json):
LANES_WIDE, LANES_IMAD, LANES_DFMA = 25.12, 63.09, 63.20
SLOT_WIDE, SLOT_IMAD, SLOT_FP64 = 64 / LANES_WIDE, 64 / LANES_IMAD, 64 / LANES_DFMA
# heavy-pipe instructions per unit of work, from the SASS of the kernels'
# arithmetic (tools/sass_counts.py -> profiles/r2/sass_counts.json):
#   Montgomery product (mr2, msqr64_lz_ptx): 8 IMAD.WIDE + 2 IMAD + 1 IMAD.X
#   base-2 ladder step (mr1, msqr64_shl_lz_ptx): 8 IMAD.WIDE + 2 IMAD
#   FP64 lazy product (fmul_lazy; FP64 and 32-bit classes): DMUL + 3 DFMA + 2 DADD
SLOTS_MONT_PRODUCT = 8 * SLOT_WIDE + 3 * SLOT_IMAD      # 23.4 (predicts 7.95e11/s; measured 7.96e11)
SLOTS_MONT_LADDER = 8 * SLOT_WIDE + 2 * SLOT_IMAD       # 22.4
SLOTS_FP64_PRODUCT = 6 * SLOT_FP64                      # 6.1
SURVEY_IMAD_PER_MULMOD64 = 14                           # 14 IMAD per 64-bit mulmod at 64 lanes/clk
CLS32_ON_FP64 = True
LANES_PER_CLK_SM = 64
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


def load_weak_counts():
    """Prime counts of the weak-scaling batches (tests/golden/weak_shard_counts.txt,
    oracle only): {cfg: {rank: count}}."""
    out = {}
    p = os.path.join(ROOT, "tests", "golden", "weak_shard_counts.txt")
    if os.path.exists(p):
        with open(p) as f:
            for line in f:
                line = line.split("#", 1)[0].split()
                if line:
                    out.setdefault(line[0], {})[int(line[1])] = int(line[2])
    return out


def shard_input(cfg, mode, rank, world):
    """(kind, lo, hi) of rank's batch.  kind "iota": the values lo .. hi-1
    (C4, split by value); kind "gen": generator indices [lo, hi) of cfg."""
    from paper_2108_04791_b200 import shard
    n = workloads.CONFIGS[cfg][1]
    if cfg == "C4":
        a, b = shard.value_range_shard(rank, world, 0, n)
        return "iota", a, b
    if mode == "weak":
        a, b = shard.weak_shard(rank, world, n)
    else:
        a, b = shard.strong_shard(rank, world, n)
    return "gen", a, b


def scaling_of(cfg, mode):
    return "strong" if (cfg == "C4" or mode == "strong") else "weak"


def global_units(cfg, mode, world):
    n = workloads.CONFIGS[cfg][1]
    return n * world if scaling_of(cfg, mode) == "weak" else n


def expected_total(cfg, mode, world, counts, weak_counts):
    """Prime count over all ranks' batches (None when no golden value exists)."""
    if scaling_of(cfg, mode) == "strong":
        return counts[cfg]
    wc = weak_counts.get(cfg, {})
    if all(r in wc for r in range(world)):
        return sum(wc[r] for r in range(world))
    return counts[cfg] if world == 1 else None


def make_input(cfg, mode, rank, world, torch, dev):
    """Rank's batch on the device, and its host copy (None for an iota)."""
    kind, a, b = shard_input(cfg, mode, rank, world)
    if kind == "iota":
        return torch.arange(a, b, dtype=torch.int64, device=dev), None, (kind, a, b)
    host = workloads.generate(cfg, start=a, count=b - a)
    return torch.from_numpy(host.view(np.int64)).to(dev), host, (kind, a, b)


L2_BYTES = 126 * 2**20
_flush_buf = None


def l2_flush_needed(n):
    """Inputs smaller than a few L2s could stay resident between steps."""
    return n * 8 < 4 * L2_BYTES


def time_steps(isp, torch, dN, dout, n, steps, warmup, stream, dist, sampler=None, flush=False):
    """Per-step device time of isprime_device (ms), the MAX over ranks, and
    the library's launch count over the timed steps.  W warm-up calls, then
    barrier + synchronize, CUDA events on the launching stream around the K
    timed calls, synchronize + barrier.  flush=True (inputs that fit in L2):
    a 512 MB write on the same stream between steps, outside per-step events,
    so every step starts from a cold L2."""
    global _flush_buf
    if flush and _flush_buf is None:
        _flush_buf = torch.empty(512 * 2**20, dtype=torch.uint8, device=dN.device)
    for _ in range(warmup):
        isp.isprime_device(dN, dout, n, stream)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = isp.get_stats()["kernel_launches"]
    if sampler:
        sampler.mark()
    if flush:
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
        ms = sum(a.elapsed_time(b) for a, b in evs) / steps
    else:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            isp.isprime_device(dN, dout, n, stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
    if sampler:
        sampler.mark()
    launches = isp.get_stats()["kernel_launches"] - l0
    if dist is not None:
        dist.barrier()
        t = torch.tensor([ms], dtype=torch.float64, device=dN.device)
        ms = float(allreduce(dist, t, dist.ReduceOp.MAX).item())
    return ms, launches


def allreduce(dist, t, op):
    """all_reduce through the process group (NCCL on GPU tensors; a gloo group,
    used only by the functional multi-rank check BENCH_DIST_BACKEND=gloo,
    reduces a host copy)."""
    if dist.get_backend() == "gloo":
        h = t.cpu()
        dist.all_reduce(h, op=op)
        return h.to(t.device)
    dist.all_reduce(t, op=op)
    return t


def count_total(isp, torch, dout, n, stream, dist):
    """(this rank's prime count, NCCL sum over ranks) -- validation only."""
    dcount = torch.zeros(1, dtype=torch.int64, device=dout.device)
    isp.isprime_popcount_device(dout, dcount, n, stream)
    torch.cuda.synchronize()
    mine = int(dcount.item())
    if dist is not None:
        dcount = allreduce(dist, dcount, dist.ReduceOp.SUM)
    return mine, int(dcount.item())


def kernel_profile(isp, torch, dN, dout, n, steps, stream):
    """Instrumented passes: events around every launch (per-kernel device
    time), then the algorithmic work counters (option count_work: separate
    kernel instantiations, so they run in a pass of their own, untimed)."""
    isp.set_option("kernel_timing", 1)
    isp.reset_kernel_times()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        isp.isprime_device(dN, dout, n, stream)
    e1.record(stream)
    torch.cuda.synchronize()
    kt = isp.get_kernel_times()
    isp.set_option("kernel_timing", 0)
    isp.set_option("count_work", 1)
    isp.reset_stats()
    for _ in range(steps):
        isp.isprime_device(dN, dout, n, stream)
    torch.cuda.synchronize()
    st = isp.get_stats()
    isp.set_option("count_work", 0)
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
        # units of work: modular multiplications of the method's square-and-multiply
        # ModExp, counted on the device per magnitude class
        mm, mf = stats["mulmods"], stats["mulmods_fp64"]
        k = 0 if name == "mr1" else 2
        mont = mm[k + 1] / steps
        fp = (mf[0 if name == "mr1" else 1] + (mm[k] if CLS32_ON_FP64 else 0)) / steps
        slots = mont * (SLOTS_MONT_LADDER if name == "mr1" else SLOTS_MONT_PRODUCT) + fp * SLOTS_FP64_PRODUCT
        achieved = slots / (ms * 1e-3) / 1e12
        mhz = peaks.get("sm_max_mhz", 1965.0)
        peak = 148 * LANES_PER_CLK_SM * mhz * 1e6 / 1e12
        survey = (mont * SURVEY_IMAD_PER_MULMOD64 + fp * 6) / (ms * 1e-3) / 1e12 / peak
        ncu_sum = None
        if ncu and ncu.get("fmaheavy_pipe_pct") is not None and ncu.get("fp64_pipe_pct") is not None:
            ncu_sum = round((ncu["fmaheavy_pipe_pct"] + ncu["fp64_pipe_pct"]) / 100.0, 4)
        return {"kernel": name, "bound": "alu", "achieved": round(achieved, 4), "peak": round(peak, 3),
                "unit": "T heavy-pipe lane-slots/s (IMAD.WIDE and DFMA share one multiplier pipe)",
                "frac": round(achieved / peak, 4),
                "ncu_fmaheavy_plus_fp64": ncu_sum,
                "survey_model_frac": round(survey, 4),
                "traffic": traffic, "ncu": ncu,
                "peak_source": f"148 SMs x {LANES_PER_CLK_SM} lane-slots/clk x {mhz:.0f} MHz (MEASURED_PEAKS "
                               f"sm_max_mhz); per-instruction slots 64/measured lanes/clk/SM: IMAD.WIDE "
                               f"{SLOT_WIDE:.2f}, IMAD {SLOT_IMAD:.2f}, DFMA {SLOT_FP64:.2f} (profiles/r1_imad_peak.json)",
                "work": f"per step: {mont:.4g} Montgomery {'ladder steps' if name == 'mr1' else 'products'} x "
                        f"{SLOTS_MONT_LADDER if name == 'mr1' else SLOTS_MONT_PRODUCT:.1f} slots + {fp:.4g} FP64 "
                        f"products x {SLOTS_FP64_PRODUCT:.1f} slots (SASS: profiles/r2/sass_counts.json); "
                        f"survey_model_frac: {SURVEY_IMAD_PER_MULMOD64} slots per 64-bit mulmod",
                "ms_per_step": round(ms, 4)}
    fused = stats.get("mulmods_fused", [0, 0])
    if name == "classify" and sum(fused) > 0:
        # classify with the fused witness tests (option fuse_bits): the strong
        # tests of the 32-bit class run on the FP64 pipe inside the streaming
        # pass, so the multiplier pipe is its roofline; the HBM side is reported
        # beside it
        fp = sum(fused) / steps
        slots = fp * SLOTS_FP64_PRODUCT
        achieved = slots / (ms * 1e-3) / 1e12
        mhz = peaks.get("sm_max_mhz", 1965.0)
        peak = 148 * LANES_PER_CLK_SM * mhz * 1e6 / 1e12
        hbm = HBM_BYTES_PER_ELEM * n / (ms * 1e-3) / 1e9
        ncu_sum = None
        if ncu and ncu.get("fmaheavy_pipe_pct") is not None and ncu.get("fp64_pipe_pct") is not None:
            ncu_sum = round((ncu["fmaheavy_pipe_pct"] + ncu["fp64_pipe_pct"]) / 100.0, 4)
        return {"kernel": name, "bound": "alu", "achieved": round(achieved, 4), "peak": round(peak, 3),
                "unit": "T heavy-pipe lane-slots/s (IMAD.WIDE and DFMA share one multiplier pipe)",
                "frac": round(achieved / peak, 4), "ncu_fmaheavy_plus_fp64": ncu_sum,
                "hbm_gbs": round(hbm, 1), "hbm_frac": round(hbm / float(peaks.get("hbm_gbs", 6650.0)), 4),
                "traffic": traffic, "ncu": ncu,
                "work": f"per step: {fused[0] / steps:.4g} base-2 + {fused[1] / steps:.4g} remaining-base FP64 "
                        f"products x {SLOTS_FP64_PRODUCT:.1f} slots in the streaming pass (trial division, "
                        f"classification and {HBM_BYTES_PER_ELEM} B/element of traffic besides: issue-bound)",
                "ms_per_step": round(ms, 4)}
    if name == "small":
        return {"kernel": name, "bound": "latency", "achieved": None, "peak": None, "unit": None, "frac": None,
                "traffic": traffic, "ncu": ncu,
                "work": f"{n} elements in one fused launch ({ms * 1e3:.1f} us): launch- and latency-bound "
                        f"({9 * n / 1e6:.2f} MB of traffic = {9 * n / (peaks.get('hbm_gbs', 6541.1) * 1e9) * 1e6:.2f} "
                        "us at HBM peak), SURVEY.md 8(d)",
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


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline_run(cfg, host, sample_n, sample1_n):
    """The oracle as it stands on this host's cores: all threads on the first
    sample_n elements, and one thread on the first sample1_n."""
    import oracle  # test infrastructure: the cpu_baseline leg only
    sample = np.arange(sample_n, dtype=np.uint64) if host is None else host[:sample_n]
    threads = os.cpu_count() or 1
    t = time.perf_counter()
    out = oracle.isprime(sample, threads=threads)
    dt = time.perf_counter() - t
    s1 = sample[:sample1_n]
    t = time.perf_counter()
    oracle.isprime(s1, threads=1)
    dt1 = time.perf_counter() - t
    return {"value": round(sample.shape[0] / dt / 1e9, 6), "unit": UNIT, "cores": threads, "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"first {sample.shape[0]} elements of {cfg} ({dt:.2f} s wall on {threads} threads, "
                      f"{int(out.sum())} primes)",
            "one_thread": {"value": round(s1.shape[0] / dt1 / 1e9, 6), "unit": UNIT,
                           "sample": f"first {s1.shape[0]} elements of {cfg} ({dt1:.2f} s wall, 1 thread)",
                           "ns_per_element": round(dt1 / s1.shape[0] * 1e9, 1)}}


def config_block(cfg, mode, world):
    n = workloads.CONFIGS[cfg][1]
    sc = scaling_of(cfg, mode)
    if cfg == "C4":
        par = f"dp{world}: value-range split, rank r classifies the iota [floor(r 2^32/W), floor((r+1) 2^32/W))"
    elif sc == "weak":
        par = f"dp{world}: weak, rank r classifies generator indices [r n, (r+1) n), no collective"
    else:
        par = f"dp{world}: strong, contiguous split [floor(r n/W), floor((r+1) n/W)) of the fixed array"
    return {"workload": f"{cfg}: {workloads.CONFIGS[cfg][2]} (BASELINE.json configs[{int(cfg[1]) - 1}])",
            "n_per_rank": n if sc == "weak" else n // world, "global_n": global_units(cfg, mode, world),
            "parallelism": par,
            "l2": ("flushed between steps (512 MB write outside per-step CUDA events)" if l2_flush_needed(n // world)
                   else "no flush: inputs larger than L2 (%.2f GiB per rank per step)" % (n * 8 / world / 2**30))}


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
        "scaling": scaling_of(cfg, args.scaling), "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": config_block(cfg, args.scaling, 1),
        "cpu_baseline": {"value": round(value, 6), "unit": UNIT, "cores": threads, "kind": "oracle",
                         "cpu_model": cpu_model(),
                         "sample": f"first {sample_n} elements of {cfg} per step, on rank 0's host only"},
        "e2e": {"value": round(value, 6), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def measure_config(isp, torch, dev, stream, dist, rank, world, cfg, mode, steps, warmup, counts, weak_counts,
                   profile=True, peaks=None, peaks_kind=None, clocks=None):
    """One configuration in one scaling mode across all ranks: value (max over
    ranks), correctness of the NCCL-summed count, and (optionally) the
    instrumented pass with the roofline of the dominant kernel (rank-local)."""
    dN, _, (kind, a, b) = make_input(cfg, mode, rank, world, torch, dev)
    n = b - a
    dout = torch.empty(n, dtype=torch.uint8, device=dev)
    flush = l2_flush_needed(n)
    csteps = max(steps, 100) if cfg == "C1" else steps
    ms, launches = time_steps(isp, torch, dN, dout, n, csteps, warmup, stream, dist, flush=flush)
    mine, total = count_total(isp, torch, dout, n, stream, dist)
    exp = expected_total(cfg, mode, world, counts, weak_counts)
    units = global_units(cfg, mode, world)
    res = {"value": round(units / (ms * 1e-3) / 1e9, 4), "unit": UNIT, "ms_per_step": round(ms, 4),
           "scaling": scaling_of(cfg, mode), "n_per_rank": n, "global_n": units,
           "correct": (total == exp) if exp is not None else None, "prime_count_total": total,
           "gpu_launches_per_step": launches / csteps,
           "l2": "flushed between steps" if flush else "no flush: inputs larger than L2"}
    if profile:
        ckm, cst, _ = kernel_profile(isp, torch, dN, dout, n, csteps, stream)
        res["kernels_ms_per_step"] = {k: round(v, 4) for k, v in ckm.items()}
        res["roofline"] = roofline(ckm, cst, n, csteps, peaks, peaks_kind, clocks, cfg)
    del dN, dout
    torch.cuda.empty_cache()
    return res


def witness_option(isp, torch, dev, stream, args, counts, mode, cfgs):
    """Another exact witness mode on the same workloads with the same timing;
    the headline above is the paper's Eq 4 method.  mode 1: Baillie-PSW (a
    strong Lucas test replaces the six remaining Eq 4 bases for n >= 2^51, the
    paper's proposed next step); mode 2: reduced witness sets
    by magnitude (base 2 + one hashed base below 2^32,
    Jaeschke's four bases below 1,122,004,669,633)."""
    res = {}
    isp.set_option("witness", mode)
    try:
        for c in cfgs:
            r = measure_config(isp, torch, dev, stream, None, 0, 1, c, "weak", args.steps, args.warmup, counts, {},
                               profile=False)
            res[c] = {k: r[k] for k in ("value", "unit", "ms_per_step", "correct")}
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


def stride2_run(isp, torch, dev, stream, args, peaks, clocks):
    """odd numbers in a restricted range, N[i]
    = N0 + 2 i, 2^28 elements below 2^32 -- the fused streaming sieve
    (dense2_kernel, no global bitmap).  Device time per call and the achieved
    fraction of HBM at 9 algorithmic bytes per element."""
    res = {}
    for lo in (1, (1 << 32) - (1 << 29) + 1):
        n = 1 << 28
        dN = torch.arange(lo, lo + 2 * n, 2, dtype=torch.int64, device=dev)
        dout = torch.empty(n, dtype=torch.uint8, device=dev)
        ms, _ = time_steps(isp, torch, dN, dout, n, args.steps, args.warmup, stream, None)
        km, st, _ = kernel_profile(isp, torch, dN, dout, n, args.steps, stream)
        gbs = 9 * n / (ms * 1e-3) / 1e9
        res[f"N0={lo}"] = {"value": round(n / (ms * 1e-3) / 1e9, 4), "unit": UNIT, "ms_per_step": round(ms, 4),
                           "hbm_GBps_algorithmic": round(gbs, 1),
                           "hbm_frac": round(gbs / float(peaks.get("hbm_gbs", 6541.1)), 4),
                           "queued_for_witness_kernels": st["queued32"] + st["queued64"],
                           "kernels_ms_per_step": {k: round(v, 4) for k, v in km.items()}}
        del dN, dout
        torch.cuda.empty_cache()
    return res


def e2e_run(isp, torch, dev, dist, host, shard, dout, steps):
    """The same metric through the host C-ABI isprime() on pinned buffers:
    H2D of the batch and D2H of the result inside the timed region (host wall
    clock around the synchronous call), max over ranks."""
    kind, a, b = shard
    n = b - a
    if host is None:
        hN = torch.arange(a, b, dtype=torch.int64).pin_memory()
    else:
        hN = torch.from_numpy(host.view(np.int64)).pin_memory()
    hout = torch.empty(n, dtype=torch.uint8).pin_memory()
    isp.isprime_into(hN, hout)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    esteps = max(1, min(steps, 5))
    for _ in range(esteps):
        isp.isprime_into(hN, hout)
    et = torch.tensor([(time.perf_counter() - t0) / esteps], dtype=torch.float64, device=dev)
    if dist:
        et = allreduce(dist, et, dist.ReduceOp.MAX)
    matches = bool(np.array_equal(hout.numpy(), dout.cpu().numpy()))
    del hN, hout
    return float(et.item()), matches, n


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5", choices=sorted(workloads.CONFIGS))
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: every rank a full batch; strong: the fixed array split across ranks "
                         "(C4 is always split by value range)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-per-config", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip scalar latency and witness-option lines")
    ap.add_argument("--cpu-sample", type=int, default=1 << 24)
    ap.add_argument("--cpu-sample1", type=int, default=1 << 20)
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

    # BENCH_SAME_DEVICE=1 + BENCH_DIST_BACKEND=gloo: every rank on cuda:0 -- a
    # functional check of the multi-rank code path on a one-GPU box, never a
    # measurement (the ranks' kernels then share one GPU)
    if os.environ.get("BENCH_SAME_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            tdist.init_process_group("nccl", device_id=dev)
        else:
            tdist.init_process_group(backend)
        dist = tdist
    isp.load(build_if_missing=False)
    stream = torch.cuda.current_stream()
    peaks, peaks_kind = measured_peaks()
    counts = load_counts()
    weak_counts = load_weak_counts()

    cfg, mode = args.config, args.scaling
    dN, host, shard = make_input(cfg, mode, rank, world, torch, dev)
    n = shard[2] - shard[1]
    dout = torch.empty(n, dtype=torch.uint8, device=dev)
    units = global_units(cfg, mode, world)

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.2)
    ms_max, launches = time_steps(isp, torch, dN, dout, n, args.steps, args.warmup, stream, dist, sampler,
                                  flush=l2_flush_needed(n))
    sampler.stop()
    clocks = sampler.summary()
    value = units / (ms_max * 1e-3) / 1e9

    # validation: count per rank -> NCCL sum, against the oracle's golden counts
    my_count, total_count = count_total(isp, torch, dout, n, stream, dist)
    exp_total = expected_total(cfg, mode, world, counts, weak_counts)
    # rank 0's own batch has a golden count at W = 1 and in weak scaling (indices [0, n))
    exp_rank0 = counts[cfg] if (world == 1 or scaling_of(cfg, mode) == "weak") else None

    kern_ms, st, inst_ms = kernel_profile(isp, torch, dN, dout, n, args.steps, stream)
    roof = roofline(kern_ms, st, n, args.steps, peaks, peaks_kind, clocks, cfg)

    e2e = None
    if not args.no_e2e:
        et, matches, _ = e2e_run(isp, torch, dev, dist, host, shard, dout, args.steps)
        e2e = {"value": round(units / et / 1e9, 4), "unit": UNIT,
               "h2d_bytes_per_step": int(n * 8), "d2h_bytes_per_step": int(n),
               "ms_per_step": round(et * 1e3, 3),
               "how": "isprime() host C-ABI on pinned host buffers; host wall clock around the synchronous call, "
                      "max over ranks; bytes are per rank",
               "matches_device": matches}

    line = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_max, 4), "higher_is_better": True,
        "scaling": scaling_of(cfg, mode), "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (seeded generator, SURVEY.md 8(d))",
        "config": config_block(cfg, mode, world),
        "roofline": roof, "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks,
        "kernels_ms_per_step": {k: round(v, 4) for k, v in kern_ms.items()},
        "instrumented_ms_per_step": round(inst_ms, 4),
        "prime_count": {"rank0": my_count, "total": total_count, "expected_total": exp_total,
                        "correct": (total_count == exp_total) if exp_total is not None else None,
                        "rank0_correct": (my_count == exp_rank0) if exp_rank0 is not None else None},
        "stats_per_step": {k: (v / args.steps if isinstance(v, int) else [x / args.steps for x in v])
                           for k, v in st.items() if k not in ("window_lo", "window_hi", "kernel_launches")},
    }
    del dN, dout
    torch.cuda.empty_cache()

    if not args.no_per_config:
        per = {}
        for c in ("C1", "C2", "C3", "C4", "C5"):
            if c == cfg:
                continue
            per[c] = measure_config(isp, torch, dev, stream, dist, rank, world, c, mode, args.steps, args.warmup,
                                    counts, weak_counts, True, peaks, peaks_kind, clocks)
        line["per_config"] = per
        if world > 1:
            other = "strong" if mode == "weak" else "weak"
            line[f"per_config_{other}"] = {
                c: measure_config(isp, torch, dev, stream, dist, rank, world, c, other, args.steps, args.warmup,
                                  counts, weak_counts, False)
                for c in ("C1", "C2", "C3", "C5")}
    if rank == 0 and world == 1:
        line["cpu_baseline"] = cpu_baseline_run(cfg, host, min(n, args.cpu_sample), min(n, args.cpu_sample1))
        if not args.no_extras:
            line["scalar_latency"] = scalar_latency(isp, torch, dev, stream)
            line["stride2_odd_range"] = stride2_run(isp, torch, dev, stream, args, peaks, clocks)
            line["witness_bpsw"] = witness_option(isp, torch, dev, stream, args, counts, 1, ("C5", "C3"))
            line["witness_reduced"] = witness_option(isp, torch, dev, stream, args, counts, 2, ("C5", "C2"))
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
