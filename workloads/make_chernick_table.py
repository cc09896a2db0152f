"""Write workloads/chernick_k.txt: every k in [1, 242347] for which 6k+1,
12k+1 and 18k+1 are all prime (Chernick's form of Carmichael numbers; 242347
is the largest k with (6k+1)(12k+1)(18k+1) < 2^64).  Calls oracle/ only.

    python workloads/make_chernick_table.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402

KMAX = 242347


def main():
    k = np.arange(1, KMAX + 1, dtype=np.uint64)
    a = oracle.isprime(6 * k + 1)
    b = oracle.isprime(12 * k + 1)
    c = oracle.isprime(18 * k + 1)
    ks = k[(a & b & c).astype(bool)]
    assert (6 * KMAX + 1) * (12 * KMAX + 1) * (18 * KMAX + 1) < 2**64
    assert (6 * (KMAX + 1) + 1) * (12 * (KMAX + 1) + 1) * (18 * (KMAX + 1) + 1) >= 2**64
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "chernick_k.txt")
    with open(path, "w") as f:
        f.write("# k in [1, 242347] with 6k+1, 12k+1, 18k+1 all prime "
                "(written by workloads/make_chernick_table.py via oracle/)\n")
        for v in ks.tolist():
            f.write(f"{v}\n")
    print(f"{len(ks)} values -> {path}")


if __name__ == "__main__":
    main()
