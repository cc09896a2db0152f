"""Randomized structured stress of the CUDA path against the CPU oracle (test
infrastructure: calls oracle/, never part of the product path).

    python tools/fuzz_gpu.py [cases] [seed] [log2 min size] [log2 max size] > gpurun_out/fuzz.jsonl

Each case draws a size, a mixture of structured pieces (log-uniform bit
lengths, narrow windows, arithmetic progressions of stride 1 / 2 / other,
values hugging 2^32 / 2^51 / 2^63 / 2^64, all-even runs, constant runs,
repeated primes), an element misalignment of both buffers and a random set of
options, runs isprime_device into a poisoned buffer (and, for a third of the
cases up to 2^22 elements, the host call isprime) and compares every byte
with oracle.isprime (out[i] = 1 iff N[i] is prime).  One JSON
line per case, a summary line at the end; exit code 1 on any mismatch.
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2108_04791_b200 as isp  # noqa: E402

U64 = np.uint64
OPTS = {
    "force_path": (0, 0, 0, 1, 2),
    "witness": (0, 0, 1, 2),
    "bases32": (3, 7),
    "fuse_bits": (32, 32, 0, 51),
    "chunk_log2": (30, 30, 16, 20, 24),
    "td_primes32": (24, 0, 7, 64),
    "td_primes64": (32, 0, 5, 64),
    "win64": (3, 1, 2),
    "sched": (0, 1, 2),
    "small_max": (1 << 17, 0),
    "warp_max": (4096, 0),
    "sieve_cache": (0, 1),
    "graph": (0, 0, 1),
}


def piece(rng, m):
    kind = int(rng.integers(0, 11))
    if kind == 0:  # log-uniform bit length
        bits = rng.integers(1, 65, size=m)
        v = rng.integers(0, 1 << 63, size=m, dtype=np.uint64) * U64(2) + rng.integers(0, 2, size=m, dtype=np.uint64)
        v = v >> (U64(64) - bits.astype(np.uint64))
        return kind, v | (U64(1) << (bits.astype(np.uint64) - U64(1)))
    if kind == 1:  # narrow window below 2^32
        lo = int(rng.integers(0, (1 << 32) - (1 << 22)))
        return kind, rng.integers(lo, lo + (1 << int(rng.integers(4, 22))), size=m, dtype=np.uint64)
    if kind in (2, 3, 4):  # arithmetic progression: stride 1, 2, other
        d = (1, 2, int(rng.integers(3, 1000)))[kind - 2]
        top = (1 << 32) if rng.integers(0, 4) else (1 << 64)
        hi = top - d * m - 1
        lo = int(rng.integers(0, max(hi, 1), dtype=np.uint64)) if hi > 0 else 0
        t = int(rng.integers(0, 6))
        if t < 2:
            lo = max(0, min(lo, 5))  # ranges that start at 0 .. 5
        elif t == 2 and d * m < (1 << 32):
            lo = (1 << 32) - d * m + int(rng.integers(-3, 4)) * d  # ending at / crossing 2^32
            lo = max(lo, 0)
        return kind, U64(lo) + U64(d) * np.arange(m, dtype=np.uint64)
    if kind == 5:  # hugging a class boundary
        b = (1 << int(rng.choice([16, 20, 31, 32, 33, 50, 51, 52, 53, 55, 59, 62, 63, 64])))
        off = rng.integers(-(1 << 12), 1 << 12, size=m)
        v = (b + off.astype(object)) % (1 << 64)
        return kind, np.array(v, dtype=np.uint64)
    if kind == 6:  # even run
        return kind, rng.integers(0, 1 << 63, size=m, dtype=np.uint64) * U64(2)
    if kind == 7:  # one value repeated
        pool = [0, 1, 2, 3, 2047, (1 << 31) - 1, (1 << 32) + 15, (1 << 61) - 1, (1 << 64) - 59, (1 << 64) - 1,
                3215031751, 3825123056546413051, 18446744030759878681]
        c = np.uint64(pool[int(rng.integers(0, len(pool)))])
        return kind, np.full(m, c, dtype=np.uint64)
    if kind == 8:  # uniform 64-bit odd
        return kind, rng.integers(0, 1 << 63, size=m, dtype=np.uint64) * U64(2) + U64(1)
    if kind == 9:  # uniform 32-bit
        return kind, rng.integers(0, 1 << 32, size=m, dtype=np.uint64)
    # squares and products of two nearby primes-ish odd numbers (hard composites for trial division)
    a = rng.integers(1 << 10, 1 << 32, size=m, dtype=np.uint64) | U64(1)
    return kind, a * (a + U64(2) * rng.integers(0, 3, size=m, dtype=np.uint64))


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 20211
    # optional size range (log2): python tools/fuzz_gpu.py 24 5 25.5 27.5 for multi-chunk sizes
    lg_lo = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
    lg_hi = float(sys.argv[4]) if len(sys.argv) > 4 else 23.5
    big_ok = len(sys.argv) <= 3
    rng = np.random.default_rng(seed)
    dev = torch.device("cuda:0")
    defaults = {k: isp.get_option(k) for k in OPTS}
    bad_cases = 0
    total = 0
    t0 = time.time()
    for c in range(cases):
        n = int(2 ** rng.uniform(lg_lo, lg_hi))
        if big_ok and rng.integers(0, 12) == 0:
            n = int(rng.integers((1 << 24), (1 << 25)))
        if big_ok and rng.integers(0, 4) == 0:  # sizes at the paths' thresholds (short-array limits, tiles, dense minimum, chunks)
            t = (4096, 8192, 1 << 16, 1 << 17, 1 << 20, 1 << 21, (1 << 20) + 8192, 1 << 24)
            n = max(1, int(t[int(rng.integers(0, len(t)))]) + int(rng.integers(-2, 3)))
        parts, kinds, left = [], [], n
        while left > 0:
            m = left if rng.integers(0, 3) == 0 else int(rng.integers(1, left + 1))
            k, v = piece(rng, m)
            kinds.append(k)
            parts.append(v)
            left -= m
        N = np.concatenate(parts)
        r = int(rng.integers(0, 8))
        if r < 2:
            rng.shuffle(N)
        elif r == 2:
            N = np.sort(N)
        if rng.integers(0, 4) == 0:  # a few foreign elements where the plan's samples may miss them
            k = int(rng.integers(1, 5))
            pos = rng.integers(0, n, size=k)
            N = N.copy()
            N[pos] = piece(rng, k)[1]
        opts = {}
        for k, vals in OPTS.items():
            if rng.integers(0, 3) == 0:
                opts[k] = int(vals[int(rng.integers(0, len(vals)))])
        for k, v in defaults.items():
            isp.set_option(k, opts.get(k, v))
        off_in, off_out = int(rng.integers(0, 2)), int(rng.integers(0, 8))
        exp = oracle.isprime(N)
        dbuf = torch.zeros(n + 2, dtype=torch.int64, device=dev)
        dbuf[off_in:off_in + n] = torch.from_numpy(N.view(np.int64)).to(dev)
        dout = torch.full((n + 16,), 7, dtype=torch.uint8, device=dev)
        isp.isprime_device(dbuf.data_ptr() + 8 * off_in, dout.data_ptr() + off_out, n)
        torch.cuda.synchronize()
        full = dout.cpu().numpy()
        got = full[off_out:off_out + n]
        bad = np.nonzero(got != exp)[0]
        guard = bool((full[:off_out] == 7).all() and (full[off_out + n:] == 7).all())
        rec = {"case": c, "n": n, "kinds": kinds[:12], "opts": opts, "off": [off_in, off_out],
               "primes": int(exp.sum()), "mismatches": int(bad.size), "guard_intact": guard}
        if bad.size:
            rec["first"] = [[int(i), int(N[i]), int(got[i]), int(exp[i])] for i in bad[:8]]
        if n <= (1 << 22) and rng.integers(0, 3) == 0:  # the host C-ABI call on the same input
            hbad = int(np.count_nonzero(isp.isprime(N) != exp))
            rec["host_mismatches"] = hbad
            if hbad:
                bad_cases += 1
        if bad.size or not guard:
            bad_cases += 1
        total += n
        print(json.dumps(rec), flush=True)
    for k, v in defaults.items():
        isp.set_option(k, v)
    print(json.dumps({"summary": True, "cases": cases, "seed": seed, "elements": total, "bad_cases": bad_cases,
                      "wall_s": round(time.time() - t0, 1)}))
    sys.exit(1 if bad_cases else 0)


if __name__ == "__main__":
    main()
