"""Workloads for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck) over the pipeline kernels at multi-segment sizes.

    compute-sanitizer --tool racecheck python tools/sanitize.py dense

Each workload runs one isprime_device() call and checks the result against
the CPU oracle (test infrastructure, allowed in tools), so a sanitizer run
that reports 0 hazards also shows the output it watched was correct.

  dense    N = 1 .. 2^26 (odd start; 342 segments: 2-3 per block of the
           148-block dense_kernel, both shared buffers and the k >= 2
           "buffer empty" hand-over), then 3 .. 3 + 2^21 + 1
  pipeline C5 prefix of 2^21 elements: plan, sieve, classify (several tiles
           per block), qscatter, mr1, mr2
  c3       C3 prefix of 2^20 (Montgomery class only)
  small    short-array path (small_kernel, small_warp_kernel)
  chunks   several device chunks per call, every witness mode, inputs where
           every element survives to phase 2 (queues at their worst case)
  full     C2, C3, C5 at full size
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import workloads  # noqa: E402


def run(isp, torch, N, **opts):
    saved = {k: isp.get_option(k) for k in opts}
    for k, v in opts.items():
        isp.set_option(k, v)
    try:
        dN = torch.from_numpy(np.ascontiguousarray(N).view(np.int64)).cuda()
        dout = torch.full((N.shape[0],), 7, dtype=torch.uint8, device="cuda")
        isp.isprime_device(dN, dout)
        torch.cuda.synchronize()
        got = dout.cpu().numpy()
    finally:
        for k, v in saved.items():
            isp.set_option(k, v)
    exp = oracle.isprime(N)
    bad = int((got != exp).sum())
    print(f"{N.shape[0]} elements, {int(exp.sum())} primes, {bad} mismatches", flush=True)
    assert bad == 0


def main():
    import torch
    import paper_2108_04791_b200 as isp
    what = sys.argv[1] if len(sys.argv) > 1 else "pipeline"
    if what == "dense":
        run(isp, torch, np.arange(1, 1 + (1 << 26), dtype=np.uint64), small_max=0)
        run(isp, torch, np.arange(3, 3 + (1 << 21) + 1, dtype=np.uint64), small_max=0)
    elif what == "pipeline":
        run(isp, torch, workloads.generate("C5", count=1 << 21), small_max=0)
    elif what == "c3":
        run(isp, torch, workloads.generate("C3", count=1 << 20), small_max=0)
    elif what == "small":
        run(isp, torch, workloads.generate("C5", count=3000))
        run(isp, torch, workloads.generate("C5", count=100_000))
    elif what == "chunks":  # several device chunks per call, every witness mode, all-prime input
        N = workloads.generate("C5", count=(1 << 22) + 5)
        for w in (0, 1, 2):
            run(isp, torch, N, small_max=0, chunk_log2=20, witness=w)
        cs = np.array(workloads.chernick_numbers(), dtype=np.uint64)
        primes = np.array([(1 << 64) - 59, (1 << 61) - 1, 4294967291, (1 << 49) - 81], dtype=np.uint64)
        run(isp, torch, np.tile(np.concatenate([primes, cs]), 300), small_max=0)
        run(isp, torch, np.tile(primes, 1 << 18), small_max=0)  # every element survives to phase 2
    elif what == "full":  # the full-size configurations in the bench's launch configuration
        for cfg in ("C2", "C3", "C5"):
            run(isp, torch, workloads.generate(cfg))
    else:
        raise SystemExit(f"unknown workload {what}")
    print("sanitize workload ok", what)


if __name__ == "__main__":
    main()
