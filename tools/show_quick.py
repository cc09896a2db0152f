"""Print gpurun_out/quick.jsonl (tools/gpu_quick.sh) one line per run."""
import json
import sys

for line in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/quick.jsonl"):
    try:
        d = json.loads(line)
    except ValueError:
        print(line.rstrip()[:200])
        continue
    print(d["cfg"], d["opts"], d["ms"], d["gints"], d["kernels"])
