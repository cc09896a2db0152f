"""Does the phase-2 kernel overlap its FP64-pipe and FMA-heavy-pipe classes?
C5 split by magnitude: phase-2 time of the values below 2^51 alone, of the
values above alone, and of both together (same elements)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_04791_b200 as isp  # noqa: E402
import workloads  # noqa: E402


def kernels(N, steps=5):
    dN = torch.from_numpy(N.view(np.int64)).cuda()
    dout = torch.empty(N.shape[0], dtype=torch.uint8, device="cuda")
    for _ in range(2):
        isp.isprime_device(dN, dout)
    isp.set_option("kernel_timing", 1)
    isp.reset_kernel_times()
    for _ in range(steps):
        isp.isprime_device(dN, dout)
    torch.cuda.synchronize()
    kt = {k: round(v[1] / steps, 4) for k, v in isp.get_kernel_times().items() if v[0]}
    isp.set_option("kernel_timing", 0)
    return kt


N = workloads.generate("C5")
big = N >= np.uint64(1 << 51)
mid = (N >= np.uint64(1 << 32)) & ~big
res = {"all": kernels(N), "fp64_class_only": kernels(N[mid]), "montgomery_only": kernels(N[big]),
       "fp64_and_montgomery": kernels(N[mid | big])}
print(json.dumps(res))
