"""Summarise gpurun_out/ab.jsonl (tools/ab.sh): median step and kernel times per library and config."""
import json
import statistics
import sys
from collections import defaultdict

rows = defaultdict(list)
lib = None
for line in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ab.jsonl"):
    try:
        d = json.loads(line)
    except ValueError:
        continue
    if "lib" in d:
        lib = d["lib"].split("/")[-1]
        continue
    rows[(d["cfg"], lib)].append(d)
for (cfg, lib), ds in sorted(rows.items()):
    ks = sorted({k for d in ds for k in d["kernels"]})
    med = {k: round(statistics.median(d["kernels"].get(k, 0) for d in ds), 4) for k in ks}
    print(cfg, lib, "ms", round(statistics.median(d["ms"] for d in ds), 4), med)
