#!/bin/bash
# A/B of library builds: LIBS="base e1" CFGS="C2 C5" REPS=2 bash tools/gpu_ab.sh
# (build/lib_<name>.so; tools/explore.py device timings into gpurun_out/ab.jsonl)
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/ab.jsonl
for rep in $(seq ${REPS:-2}); do
  for c in ${CFGS:-C2 C5}; do
    for L in ${LIBS}; do
      echo "{\"lib\": \"$L\", \"rep\": $rep}" >> gpurun_out/ab.jsonl
      ISPRIME_LIB=build/lib_$L.so timeout 300 python tools/explore.py $c >> gpurun_out/ab.jsonl 2>&1
    done
  done
done
if [ -n "${PYK:-}" ]; then
  ISPRIME_LIB=build/lib_${PYLIB}.so timeout 900 python -m pytest tests -m gpu -x -q -k "$PYK" > gpurun_out/pytest_ab.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_ab.log
fi
