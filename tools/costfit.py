"""Re-fit the plan's path cost model on this GPU (the
analogue of the paper's Fig BestFit: its Eq 7/8 choose the
sieve or the per-element path from numElements and max M, with constants
fitted on an i7 that "can readily be adjusted").

The plan kernel (csrc/kernels.cuh plan_kernel) sieves a window [wlo, whi) when
    sieve_fixed + span * sieve_per_int  <  (MR cost of the sampled elements in it),
MR cost = mr32_per_bit * (odd elements) * (bit length).  This script measures
the three constants with the library's own kernel timers, then checks the
choice: for a grid of (n, M) it times the sieve path (sieve costs set to 0, so
the plan always sieves its sampled range), the MR path (force_path = 2) and
the automatic plan, and reports how far auto is from the faster of the two.

    python tools/costfit.py [--apply] [--out gpurun_out/costfit.json]

--apply sets the fitted constants (option keys sieve_fs_per_int,
sieve_fixed_ns, mr32_fs_per_bit, mr_fixed_ns) before the validation grid.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_04791_b200 as isp  # noqa: E402

DEV = torch.device("cuda:0")


def uniform(n, lo, hi, seed):
    rng = np.random.default_rng(seed)
    return torch.from_numpy(rng.integers(lo, hi, size=n, dtype=np.uint64).view(np.int64)).to(DEV)


SIEVE_ALWAYS = {"sieve_fs_per_int": 0, "sieve_fixed_ns": 0}   # auto plan sieves its whole sampled window
MR_ALWAYS = {"force_path": 2}


def run(dN, opts, steps=5):
    """Kernel times (ms per call), the event-timed total and the plan's window
    for one option set (restored afterwards)."""
    n = dN.shape[0]
    dout = torch.empty(n, dtype=torch.uint8, device=DEV)
    saved = {k: isp.get_option(k) for k in opts}
    for k, v in opts.items():
        isp.set_option(k, v)
    for _ in range(2):
        isp.isprime_device(dN, dout)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        isp.isprime_device(dN, dout)
    e1.record()
    torch.cuda.synchronize()
    total = e0.elapsed_time(e1) / steps
    isp.set_option("kernel_timing", 1)
    isp.reset_kernel_times()
    isp.reset_stats()
    for _ in range(steps):
        isp.isprime_device(dN, dout)
    torch.cuda.synchronize()
    kt = {k: v[1] / steps for k, v in isp.get_kernel_times().items() if v[0]}
    st = isp.get_stats()
    isp.set_option("kernel_timing", 0)
    for k, v in saved.items():
        isp.set_option(k, v)
    return total, kt, (st["window_lo"], st["window_hi"])


def fit_line(x, y):
    A = np.vstack([np.ones_like(x), x]).T
    (a, b), *_ = np.linalg.lstsq(A, y, rcond=None)
    return float(a), float(b)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--apply", action="store_true")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    isp.set_option("small_max", 0)
    isp.set_option("sieve_cache", 0)
    keys = ("sieve_fs_per_int", "sieve_fixed_ns", "mr32_fs_per_bit", "mr_fixed_ns")
    res = {"defaults": {k: isp.get_option(k) for k in keys}}

    # 1. sieve: time of sieve_kernel against the window span (sieve costs set to
    #    zero, so the plan sieves the sampled range of values uniform in [0, W))
    spans, st = [], []
    for lw in range(20, 33, 2):
        W = 1 << lw
        dN = uniform(1 << 22, 0, W, lw)
        _, kt, (wlo, whi) = run(dN, SIEVE_ALWAYS)
        spans.append(int(whi - wlo))
        st.append(kt.get("sieve", 0.0))
    a, b = fit_line(np.array(spans, dtype=np.float64), np.array(st, dtype=np.float64))
    res["sieve"] = {"span": spans, "ms": [round(x, 5) for x in st], "fixed_ns": round(a * 1e6, 1),
                    "fs_per_int": round(b * 1e12, 1)}

    # 2. trial division + MR per odd element per bit (force_path = MR): the
    #    pipeline's time beyond the streaming classify pass it shares with the
    #    sieve path, over uniform odd values of bit length L
    per_bit = []
    for L in (21, 24, 28, 32):
        n = 1 << 22
        dN = uniform(n, 1 << (L - 1), 1 << L, 100 + L)
        _, k_mr, _ = run(dN, MR_ALWAYS)
        _, k_sv, _ = run(dN, {"force_path": 1})
        extra = sum(k_mr.get(k, 0.0) for k in ("classify", "sort", "mr1", "mr2")) - k_sv.get("classify", 0.0)
        odd = int((dN.remainder(2) != 0).sum().item())
        per_bit.append({"L": L, "ms_mr_extra": round(extra, 5), "fs_per_odd_bit": round(extra * 1e12 / (odd * L), 1)})
    res["mr32"] = {"points": per_bit, "fs_per_bit": round(float(np.median([p["fs_per_odd_bit"] for p in per_bit])), 1)}

    # 3. the witness kernels' latency floor: a short array (2^16 values below
    #    2^20) through the MR path against the sieve path, witness kernels only
    dN = uniform(1 << 16, 1 << 19, 1 << 20, 7)
    _, k_mr, _ = run(dN, MR_ALWAYS)
    _, k_sv, _ = run(dN, SIEVE_ALWAYS)
    wk = ("sort", "mr1", "mr2")
    res["mr_fixed_ns"] = round((sum(k_mr.get(k, 0.0) for k in wk) - sum(k_sv.get(k, 0.0) for k in wk)) * 1e6, 1)

    fitted = {"sieve_fs_per_int": int(round(res["sieve"]["fs_per_int"])),
              "sieve_fixed_ns": int(round(max(res["sieve"]["fixed_ns"], 0.0))),
              "mr32_fs_per_bit": int(round(res["mr32"]["fs_per_bit"])),
              "mr_fixed_ns": int(round(max(res["mr_fixed_ns"], 0.0)))}
    res["fitted"] = fitted
    if args.apply:
        for k, v in fitted.items():
            isp.set_option(k, v)
    res["applied"] = bool(args.apply)

    # 4. the crossover (Fig BestFit analogue): n elements uniform in [0, M)
    grid = []
    for lm in (20, 24, 28, 32):
        for ln in (16, 20, 24):
            dN = uniform(1 << ln, 0, 1 << lm, lm * 100 + ln)
            t_s, _, _ = run(dN, SIEVE_ALWAYS)
            t_m, _, _ = run(dN, MR_ALWAYS)
            t_a, _, w = run(dN, {})
            best = min(t_s, t_m)
            grid.append({"log2_M": lm, "log2_n": ln, "ms_sieve": round(t_s, 4), "ms_mr": round(t_m, 4),
                         "ms_auto": round(t_a, 4), "auto_window": [int(w[0]), int(w[1])],
                         "auto_over_best": round(t_a / best, 3),
                         "faster": "sieve" if t_s < t_m else "mr"})
    res["crossover"] = grid
    res["auto_within_10pct"] = sum(g["auto_over_best"] <= 1.10 for g in grid)
    res["grid_points"] = len(grid)
    line = json.dumps(res)
    print(line)
    if args.out:
        with open(args.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
