#!/bin/bash
# A/B device timing of builds of libisprime.so on the same box:
#   bash tools/ab.sh "build/lib_a.so build/lib_b.so ..." C4 C5 ...
# alternates the libraries three times per config (tools/explore.py lines,
# one per run, tagged with the library) into gpurun_out/ab.jsonl
set -u
LIBS=$1; shift 1
mkdir -p gpurun_out
for c in "$@"; do
  for rep in 1 2 3; do
    for L in $LIBS; do
      echo "{\"lib\": \"$L\", \"rep\": $rep}" >> gpurun_out/ab.jsonl
      ISPRIME_LIB=$L timeout 600 python tools/explore.py $c >> gpurun_out/ab.jsonl 2>&1
    done
  done
done
