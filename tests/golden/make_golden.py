"""Write tests/golden/config_counts.txt: the prime count of every BASELINE.json
configuration, computed by calling oracle/ only (C4 through the plain sieve).
Also checks them against the independent survey values in generator.txt.

    python tests/golden/make_golden.py          (C1, C2, C3, C5: about a minute on 8 cores)
    python tests/golden/make_golden.py --c4     (adds pi(2^32) via the plain sieve)
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import workloads  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
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
