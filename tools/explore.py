"""Quick GPU timing sweeps of library options per config (device-resident
inputs, CUDA events).  Prints one JSON line per (config, option set).
    python tools/explore.py C3 win64=1,2,3 td_primes64=8,16,24,32"""
import itertools
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_04791_b200 as isp  # noqa: E402
import workloads  # noqa: E402


def run(cfg, opts, steps=10, count=None):
    n = workloads.CONFIGS[cfg][1] if count is None else count
    if cfg == "C4":
        dN = torch.arange(n, dtype=torch.int64, device="cuda")
    else:
        dN = torch.from_numpy(workloads.generate(cfg, count=n).view(np.int64)).cuda()
    dout = torch.empty(n, dtype=torch.uint8, device="cuda")
    saved = {k: isp.get_option(k) for k in opts}
    for k, v in opts.items():
        isp.set_option(k, v)
    for _ in range(3):
        isp.isprime_device(dN, dout)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        isp.isprime_device(dN, dout)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    isp.set_option("kernel_timing", 1)
    isp.reset_kernel_times()
    isp.reset_stats()
    for _ in range(steps):
        isp.isprime_device(dN, dout)
    torch.cuda.synchronize()
    kt = {k: round(v[1] / steps, 4) for k, v in isp.get_kernel_times().items() if v[0]}
    st = isp.get_stats()
    isp.set_option("kernel_timing", 0)
    count_p = int(dout.sum(dtype=torch.int64).item())
    for k, v in saved.items():
        isp.set_option(k, v)
    print(json.dumps({"cfg": cfg, "n": n, "opts": opts, "ms": round(ms, 4), "gints": round(n / ms / 1e6, 3),
                      "primes": count_p, "kernels": kt,
                      "stats": {k: st[k] for k in ("window_lo", "window_hi", "queued32", "queued64", "passed32",
                                                   "passed64", "sieved_integers")}}), flush=True)
    del dN, dout
    torch.cuda.empty_cache()


def main():
    cfg = sys.argv[1]
    grid = {}
    count = None
    for a in sys.argv[2:]:
        k, v = a.split("=")
        if k == "count":
            count = int(v)
            continue
        grid[k] = [int(x) for x in v.split(",")]
    keys = list(grid)
    for combo in itertools.product(*[grid[k] for k in keys]) if keys else [()]:
        run(cfg, dict(zip(keys, combo)), count=count)


if __name__ == "__main__":
    main()
