#!/bin/bash
# compute-sanitizer over the pipeline kernels (tools/sanitize.py workloads);
# logs to gpurun_out/sanitize_<tool>_<workload>.log, summary in gpurun_out/sanitize_status.txt
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for w in ${SAN_WORKLOADS:-dense pipeline c3 small}; do
    extra=""
    [ "$tool" = "memcheck" ] && extra="--leak-check full"
    [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
    timeout ${SAN_TIMEOUT:-900} $CS --tool $tool $extra --error-exitcode 9 python tools/sanitize.py $w \
      > gpurun_out/sanitize_${tool}_${w}.log 2>&1
    echo "$tool $w rc=$?" >> gpurun_out/sanitize_status.txt
  done
done
