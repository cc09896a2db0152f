"""SASS instruction counts of the arithmetic the witness kernels are built
from, per operation, from the inner loops of tools/mont_bench.cu (compiled
here for sm_100a; cuobjdump -sass).  Writes profiles/r2/sass_counts.json.

  k_sqr<2, 4>    4 chains of the lazy Montgomery square (msqr64_lz_ptx, mr2's
                 main loop for n < 2^62)
  k_sqr<0, 4>    4 chains of the subtraction-REDC square (msqr64_ptx, n >= 2^62)
  k_ladder<1,*>  the base-2 ladder step of mr1 (msqr64_shl_lz_ptx)
  k_mixed        FP64 lazy product (fmul_lazy) loop and Montgomery loop

    python tools/sass_counts.py
"""
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tools", "mont_bench.cu")
BIN = os.path.join(ROOT, "build", "mont_bench_sass")
HEAVY = ("IMAD.WIDE", "IMAD.HI", "IMAD", "IMAD.X", "IMAD.MOV", "IMAD.IADD", "IMAD.SHL", "DFMA", "DADD", "DMUL")


def loops(sass_fn):
    lines = [l for l in sass_fn.split("\n") if re.search(r"/\*[0-9a-f]{4}\*/", l)]
    addr = lambda l: int(re.search(r"/\*([0-9a-f]{4})\*/", l).group(1), 16)
    out = []
    for l in lines:
        m = re.search(r"BRA.*?(0x[0-9a-f]+)", l)
        if m and int(m.group(1), 16) < addr(l):
            lo = int(m.group(1), 16)
            body = [x for x in lines if lo <= addr(x) <= addr(l)]
            hist = {}
            for x in body:
                mm = re.search(r"\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", x)
                if mm:
                    op = mm.group(2)
                    hist[op] = hist.get(op, 0) + 1
            out.append(hist)
    return out


def main():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-o", BIN, SRC],
                   check=True)
    sass = subprocess.run(["cuobjdump", "-sass", BIN], capture_output=True, text=True, check=True).stdout
    res = {}
    for f in re.split(r"\n\s+Function : ", sass)[1:]:
        name = f.split("\n")[0].strip()
        want = {"_Z5k_sqrILi2ELi4EEvPyy": ("lazy Montgomery square (msqr64_lz_ptx)", 4),
                "_Z5k_sqrILi0ELi4EEvPyy": ("subtraction-REDC Montgomery square (msqr64_ptx)", 4),
                "_Z8k_ladderILi1ELi256EEvPyy": ("base-2 ladder step (msqr64_shl_lz_ptx)", 1)}
        if name in want:
            what, per = want[name]
            h = loops(f)[0]
            res[what] = {"kernel": name, "ops_per_unit": {k: round(v / per, 2) for k, v in sorted(h.items())},
                         "instructions_per_unit": round(sum(h.values()) / per, 2),
                         "note": f"inner loop / {per} (loop control included)"}
        if name.startswith("_Z7k_mixedILi2ELi1ELi3EE"):
            ls = loops(f)
            for h in ls:
                if any(k.startswith("DFMA") for k in h):
                    res["FP64 lazy product (fmul_lazy)"] = {
                        "kernel": name, "ops_per_unit": {k: round(v / 3, 2) for k, v in sorted(h.items())},
                        "instructions_per_unit": round(sum(h.values()) / 3, 2), "note": "inner loop / 3 chains"}
    out = os.path.join(ROOT, "profiles", "r2", "sass_counts.json")
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
