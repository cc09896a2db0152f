"""Host enqueue time of isprime_device (the call returns before the GPU work
ends) against the GPU time per call, for mid-size arrays: when the first is
below the second the pipeline is GPU-bound back to back, and capturing it in a
CUDA graph could not speed it up."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_04791_b200 as isp  # noqa: E402
import workloads  # noqa: E402

res = []
for lg in (18, 20, 22):
    n = 1 << lg
    dN = torch.from_numpy(workloads.generate("C5", count=n).view(np.int64)).cuda()
    dout = torch.empty(n, dtype=torch.uint8, device="cuda")
    for _ in range(5):
        isp.isprime_device(dN, dout)
    torch.cuda.synchronize()
    steps = 200
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    for _ in range(steps):
        isp.isprime_device(dN, dout)
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    res.append({"n": n, "host_enqueue_us_per_call": round((t1 - t0) / steps * 1e6, 2),
                "gpu_us_per_call": round(e0.elapsed_time(e1) / steps * 1e3, 2)})
print(json.dumps(res))
