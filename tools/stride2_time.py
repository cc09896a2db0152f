"""Device time of isprime_device on stride-2 ranges N[i] = lo + 2 i (odd
numbers in a restricted range): 2^28 elements, CUDA events."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_04791_b200 as isp  # noqa: E402

for lo, n in ((1, 1 << 28), ((1 << 31) | 1, 1 << 28), ((1 << 32) - (1 << 29) + 1, 1 << 28)):
    dN = torch.arange(lo, lo + 2 * n, 2, dtype=torch.int64, device="cuda")
    dout = torch.empty(n, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        isp.isprime_device(dN, dout)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        isp.isprime_device(dN, dout)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(json.dumps({"stride2_lo": lo, "n": n, "ms": round(ms, 4), "gints": round(n / ms / 1e6, 2),
                      "GBps_9B": round(9 * n / ms / 1e6, 1), "primes": int(dout.sum(dtype=torch.int64).item())}))
    del dN, dout
    torch.cuda.empty_cache()
