"""How an L2 flush between steps changes the C2 step (device time, CUDA events):
no flush; bench.py's flush (a 512 MB fill: leaves L2 full of dirty lines);
a read-only flush (a 512 MB reduction: leaves L2 clean)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_04791_b200 as isp  # noqa: E402
import workloads  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
n = workloads.CONFIGS[cfg][1]
dN = torch.from_numpy(workloads.generate(cfg, count=n).view(np.int64)).cuda()
dout = torch.empty(n, dtype=torch.uint8, device="cuda")
buf = torch.empty(512 * 2**20, dtype=torch.uint8, device="cuda")
acc = torch.zeros(1, dtype=torch.int64, device="cuda")
for _ in range(3):
    isp.isprime_device(dN, dout)
torch.cuda.synchronize()


def timed(flush, steps=20):
    evs = []
    for _ in range(steps):
        if flush == "fill":
            buf.fill_(1)
        elif flush == "read":
            acc.copy_(buf.view(torch.int64).sum())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        isp.isprime_device(dN, dout)
        e1.record()
        evs.append((e0, e1))
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in evs) / steps


res = {"cfg": cfg}
for f in ("none", "fill", "read", "none", "fill"):
    res.setdefault(f, []).append(round(timed(f), 4))
print(json.dumps(res))
