#!/bin/bash
# One source-level ncu capture: KERN regex, CFG, OPTS (explore.py option grid, one value each)
#   KERN=classify_kernel CFG=C5 OPTS="fuse=1" TAG=f1 bash tools/gpu_srcprof1.sh
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFG=${CFG:-C5}; KERN=${KERN:-classify_kernel}; TAG=${TAG:-x}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KERN" -s ${SKIP:-3} -c ${COUNT:-1} \
  -o gpurun_out/src_${CFG}_$TAG python tools/explore.py $CFG ${OPTS:-} > gpurun_out/src_ncu_${CFG}_$TAG.log 2>&1
echo "src $CFG $TAG rc=$?" >> gpurun_out/src_status.txt
