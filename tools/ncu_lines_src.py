"""Per-source-line instruction and stall-sample totals of one kernel in an ncu
report (--import-source on, -lineinfo):
    python tools/ncu_lines_src.py report.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = None
agg = []
fname = ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[2] != "-":
        continue
    try:
        inst = float(r[hdr.index("Instructions Executed")])
        samp = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except ValueError:
        continue
    agg.append((inst, samp, fname, r[0], r[1].strip()[:90]))
ti = sum(a[0] for a in agg) or 1
ts = sum(a[1] for a in agg) or 1
print(f"total inst {ti:.4g}  samples {ts:.4g}")
for a in sorted(agg, key=lambda a: -a[1])[:top]:
    print(f"{100*a[0]/ti:5.1f}% inst {100*a[1]/ts:5.1f}% samp  {a[2]}:{a[3]}  {a[4]}")
