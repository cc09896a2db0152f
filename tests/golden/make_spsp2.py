"""Write tests/golden/spsp2_below_2p32.txt: every odd composite n < 2^32 that
is a strong probable prime to base 2 (Eq 1-3 with reading G2),
computed by calling oracle/ only: the plain sieve (oracle.sieve) decides
"composite", the oracle's strong test (oracle.sprp_array) decides "passes
base 2".  The list pins the reduced witness sets of option witness = 2
(SURVEY.md 8(f) f1): below 2^32 a second base that rejects every listed n
makes base 2 + that base exact.  Checked against the survey's independent
count (2314) and its first entries (2047, 3277, 4033,
4681, 8321).

    python tests/golden/make_spsp2.py     (several minutes on 8 cores, ~4.5 GB RAM)
"""
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "spsp2_below_2p32.txt")
SEG = 1 << 24


def main():
    t0 = time.time()
    limit = 1 << 32
    is_prime = oracle.sieve(limit)
    print(f"sieve pi(2^32 - 1) = {int(is_prime.sum())}  {time.time() - t0:.0f}s", flush=True)
    found = []
    lock = threading.Lock()
    nseg = limit // SEG
    next_seg = [0]

    def work():
        while True:
            with lock:
                k = next_seg[0]
                next_seg[0] += 1
            if k >= nseg:
                return
            lo = k * SEG
            seg = is_prime[lo:lo + SEG]
            cand = np.nonzero(seg[1::2] == 0)[0].astype(np.uint64) * 2 + 1 + lo  # odd composites (and 1)
            cand = cand[cand >= 3]
            if cand.shape[0] == 0:
                continue
            ok = oracle.sprp_array(cand, np.full(cand.shape[0], 2, dtype=np.uint64))
            hit = cand[ok != 0]
            if hit.shape[0]:
                with lock:
                    found.extend(int(x) for x in hit)

    threads = [threading.Thread(target=work) for _ in range(oracle.default_threads())]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    found.sort()
    print(f"{len(found)} strong base-2 pseudoprimes below 2^32  {time.time() - t0:.0f}s", flush=True)
    assert len(found) == 2314, len(found)
    assert found[:5] == [2047, 3277, 4033, 4681, 8321], found[:5]
    with open(OUT, "w") as f:
        f.write("# Odd composite n < 2^32 that are strong probable primes to base 2, ascending.\n")
        f.write("# Written by tests/golden/make_spsp2.py (oracle/ only: plain sieve + oracle strong test).\n")
        f.write("# Count 2314 = SURVEY.md Appendix A (independent run); first entries SPEC.md:492.\n")
        for x in found:
            f.write(f"{x}\n")


if __name__ == "__main__":
    main()
