#!/bin/bash
# ncu evidence for one configuration (default C5): launch list of the bench
# command and full-set captures of the witness / classify kernels.
# Every profiled command first runs once without ncu and must exit 0.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFG=${NCU_CFG:-C5}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ncu_build.log 2>&1
BENCH="python bench.py --config $CFG --steps 2 --warmup 3 --no-per-config --no-e2e"
$BENCH > gpurun_out/ncu_plain_bench.json 2> gpurun_out/ncu_plain_bench.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv $BENCH > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?" >> gpurun_out/ncu_status.txt
EXP="python tools/explore.py $CFG"
$EXP > gpurun_out/ncu_plain_explore.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"mr1_kernel|mr2_kernel|classify_kernel|qscatter|sieve_kernel" -s 15 -c 5 -o gpurun_out/prof_$CFG $EXP > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_status.txt
