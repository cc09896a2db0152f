"""Per-source-line view of one kernel in an ncu report (needs -lineinfo and
--import-source on): share of executed warp instructions and of stall samples
per CUDA line, hottest first.

    python tools/ncu_lines.py gpurun_out/prof_C5.ncu-rep classify [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    lines, hdr, fname = [], None, None
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        elif r and r[0] == "Line No":
            hdr = r
        elif hdr and r and r[0].isdigit():
            iS = hdr.index("Warp Stall Sampling (All Samples)")
            iE = hdr.index("Instructions Executed")
            try:
                lines.append((fname, int(r[0]), r[1].strip(), int(r[iS] or 0), int(r[iE] or 0)))
            except ValueError:
                pass
    ts = sum(x[3] for x in lines) or 1
    te = sum(x[4] for x in lines) or 1
    print(f"{'file:line':28s} {'inst%':>6s} {'stall%':>6s}  source")
    for f, ln, src, s, e in sorted(lines, key=lambda x: -x[4])[:top]:
        print(f"{f + ':' + str(ln):28s} {100 * e / te:6.2f} {100 * s / ts:6.2f}  {src[:90]}")


if __name__ == "__main__":
    main()
