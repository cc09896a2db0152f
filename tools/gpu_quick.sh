#!/bin/bash
# Quick GPU check of a change: device timings of the configurations (CFGS,
# explore.py option grid OPTS) and a parity subset (PYK: pytest -k expression).
#   CFGS="C2 C3 C5" OPTS="" PYK="random_all or config_full" bash tools/gpu_quick.sh
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in ${CFGS:-C2 C3 C5}; do python tools/explore.py $c ${OPTS:-} >> gpurun_out/quick.jsonl 2>&1; done
if [ -n "${PYK:-}" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$PYK" > gpurun_out/pytest_quick.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
fi
