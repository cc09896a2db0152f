"""Write tests/golden/config_counts.txt: the prime count of every BASELINE.json
configuration, computed by calling oracle/ only (C4 through the plain sieve).
Also checks them against the independent survey values in generator.txt.

    python tests/golden/make_golden.py          (C1, C2, C3, C5: about a minute on 8 cores)
    python tests/golden/make_golden.py --c4     (adds pi(2^32) via the plain sieve)
    python tests/golden/make_golden.py --weak   (writes weak_shard_counts.txt instead: the
        prime count of generator indices [r n, (r+1) n) for r < 8, the batch rank r of a
        weak-scaling bench run classifies; a few minutes on 8 cores)
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import workloads  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def weak():
    with open(os.path.join(HERE, "weak_shard_counts.txt"), "w") as f:
        f.write("# Prime count of generator indices [r n, (r+1) n) per config and rank r < 8 (weak scaling:\n")
        f.write("# every rank classifies a full batch).  Written by tests/golden/make_golden.py --weak\n")
        f.write("# (oracle/ only).  Columns: config rank count\n")
        for cfg in ("C1", "C2", "C3", "C5"):
            n = workloads.CONFIGS[cfg][1]
            for r in range(8):
                t = time.time()
                c = int(oracle.isprime(workloads.generate(cfg, start=r * n, count=n)).sum())
                print(cfg, r, c, f"{time.time() - t:.1f}s", flush=True)
                f.write(f"{cfg} {r} {c}\n")
                f.flush()


def main():
    if "--weak" in sys.argv:
        weak()
        return
    rows = []
    for cfg in ("C1", "C2", "C3", "C5"):
        t = time.time()
        c = int(oracle.isprime(workloads.generate(cfg)).sum())
        rows.append((cfg, c))
        print(cfg, c, f"{time.time() - t:.1f}s", flush=True)
    if "--c4" in sys.argv:
        t = time.time()
        c = int(oracle.dense_range(0, 1 << 32).sum())
        rows.append(("C4", c))
        print("C4", c, f"{time.time() - t:.1f}s", flush=True)
    survey = {}
    with open(os.path.join(HERE, "generator.txt")) as f:
        for line in f:
            line = line.split("#", 1)[0].split()
            if line and line[0].startswith("C"):
                survey[line[0]] = int(line[3])
    for cfg, c in rows:
        assert survey[cfg] == c, (cfg, c, survey[cfg])
    with open(os.path.join(HERE, "config_counts.txt"), "w") as f:
        f.write("# Prime count per BASELINE.json config, written by tests/golden/make_golden.py\n")
        f.write("# (oracle/ only; equals the survey's independent counts in generator.txt)\n")
        for cfg, c in rows:
            f.write(f"{cfg} {workloads.CONFIGS[cfg][1]} {c}\n")


if __name__ == "__main__":
    main()
