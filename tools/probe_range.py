import sys, os, json
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2108_04791_b200 as isp
rng = np.random.default_rng(1)
for lo, hi in ((1 << 40, 1 << 48), (1 << 56, 1 << 62), (1 << 20, 1 << 32)):
    n = 1 << 24
    N = (rng.integers(lo, hi, size=n, dtype=np.uint64) | np.uint64(1))
    dN = torch.from_numpy(N.view(np.int64)).cuda(); dout = torch.empty(n, dtype=torch.uint8, device='cuda')
    for _ in range(3): isp.isprime_device(dN, dout)
    isp.set_option("kernel_timing", 1); isp.reset_kernel_times(); isp.reset_stats()
    for _ in range(5): isp.isprime_device(dN, dout)
    torch.cuda.synchronize()
    kt = {k: round(v[1] / 5, 4) for k, v in isp.get_kernel_times().items() if v[0]}
    st = isp.get_stats()
    print(json.dumps({"range": [lo.bit_length()-1, hi.bit_length()-1], "kernels": kt, "q64": st["queued64"]/5, "p64": st["passed64"]/5}))
    isp.set_option("kernel_timing", 0)
