"""Probe: arrays of more than 2^31 / 2^32 elements (chunk loop, 64-bit offsets).
The input is filled piecewise (one torch kernel per 2^30 elements)."""
import sys; sys.path.insert(0, '/root/repo')
import torch
import paper_2108_04791_b200 as isp


def arange_mod32(total):
    dN = torch.empty(total, dtype=torch.int64, device='cuda')
    step = 1 << 30
    for s0 in range(0, total, step):
        m = min(step, total - s0)
        torch.arange(s0, s0 + m, dtype=torch.int64, device='cuda', out=dN[s0:s0 + m])
        dN[s0:s0 + m].bitwise_and_(0xFFFFFFFF)
    return dN


for total in ((1 << 32) + (1 << 20),):
    base = total - (1 << 20)
    dN = arange_mod32(total)
    print("vals", dN[base:base + 4].tolist(), dN[base - 2:base + 2].tolist(), flush=True)
    dout = torch.full((total,), 7, dtype=torch.uint8, device='cuda')
    isp.isprime_device(dN, dout); torch.cuda.synchronize()
    print(total, "tail sum", int(dout[base:].sum(dtype=torch.int64).item()),
          "head sum", int(dout[:base].sum(dtype=torch.int64).item()), flush=True)
