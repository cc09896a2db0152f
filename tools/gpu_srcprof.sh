#!/bin/bash
# Source-level ncu capture of selected kernels on one configuration:
#   KERN="classify_kernel" CFG=C5 bash tools/gpu_srcprof.sh
# -> gpurun_out/src_<CFG>.ncu-rep (read here with ncu -i ... --page source --csv)
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/src_build.log 2>&1
CFG=${CFG:-C5}; KERN=${KERN:-classify_kernel}
python tools/explore.py $CFG > gpurun_out/src_plain_$CFG.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KERN" -s ${SKIP:-3} -c ${COUNT:-1} \
  -o gpurun_out/src_$CFG python tools/explore.py $CFG > gpurun_out/src_ncu_$CFG.log 2>&1
echo "src $CFG rc=$?" >> gpurun_out/src_status.txt
