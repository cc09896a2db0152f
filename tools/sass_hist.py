"""Opcode histogram per kernel from cuobjdump -sass (IMAD-pipe vs ALU counts).
    python tools/sass_hist.py paper_2108_04791_b200/libisprime.so [kernel-substring]"""
import collections
import re
import subprocess
import sys

IMAD_PIPE = ("IMAD", "IMUL")


def functions(path):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    cur, body = None, []
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m and cur:
            body.append(m.group(1))
    if cur:
        yield cur, body


def main():
    path = sys.argv[1]
    filt = sys.argv[2] if len(sys.argv) > 2 else ""
    for name, ops in functions(path):
        if filt not in name:
            continue
        c = collections.Counter(op.split(".")[0] for op in ops)
        imad = sum(v for k, v in c.items() if k.startswith(IMAD_PIPE))
        print(f"{name[:90]}: {len(ops)} instrs, IMAD-pipe {imad}")
        print("   ", ", ".join(f"{k}:{v}" for k, v in c.most_common(14)))


if __name__ == "__main__":
    main()
