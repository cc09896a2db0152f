#!/bin/bash
# One GPU call that produces the round's measurement evidence:
#   gpurun_out/bench.json          default bench.py line (no profiler attached)
#   gpurun_out/launches_C5.csv     ncu launch list of the same bench command (gpu__time_duration per launch)
#   gpurun_out/prof_C5.ncu-rep     ncu --set full of plan/sieve/classify/sort/mr1/mr2 on C5
#   gpurun_out/prof_C4.ncu-rep     ncu --set full of dense + classify + sieve on a C4 chunk
#   gpurun_out/prof_C3.ncu-rep, prof_C2.ncu-rep   the witness kernels and classify on C3 / C2
# Every profiled command first exits 0 without ncu.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/prof_build.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" > gpurun_out/prof_status.txt
BENCH="python bench.py --config C5 --steps 2 --warmup 3 --no-per-config --no-e2e"
$BENCH > gpurun_out/ncu_plain_bench.json 2> gpurun_out/ncu_plain_bench.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C5.csv $BENCH > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?" >> gpurun_out/prof_status.txt
python tools/explore.py C5 > gpurun_out/ncu_plain_c5.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"plan_kernel|sieve_kernel|classify_kernel|qscatter|mr1_kernel|mr2_kernel" -s 18 -c 6 -o gpurun_out/prof_C5 python tools/explore.py C5 > gpurun_out/ncu_full_c5.log 2>&1
echo "full C5 rc=$?" >> gpurun_out/prof_status.txt
python tools/explore.py C4 > gpurun_out/ncu_plain_c4.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dense_kernel|classify_kernel|sieve_kernel" -s 9 -c 3 -o gpurun_out/prof_C4 python tools/explore.py C4 > gpurun_out/ncu_full_c4.log 2>&1
echo "full C4 rc=$?" >> gpurun_out/prof_status.txt
python tools/explore.py C3 > gpurun_out/ncu_plain_c3.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"classify_kernel|mr1_kernel|mr2_kernel" -s 9 -c 3 -o gpurun_out/prof_C3 python tools/explore.py C3 > gpurun_out/ncu_full_c3.log 2>&1
echo "full C3 rc=$?" >> gpurun_out/prof_status.txt
python tools/explore.py C2 > gpurun_out/ncu_plain_c2.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"classify_kernel|mr1_kernel|mr2_kernel" -s 9 -c 3 -o gpurun_out/prof_C2 python tools/explore.py C2 > gpurun_out/ncu_full_c2.log 2>&1
echo "full C2 rc=$?" >> gpurun_out/prof_status.txt
# summaries on the box (gpurun copies back at most 64 MiB of gpurun_out/):
# per-config full_summary.json + the refreshed ncu_kernel_metrics.json; only
# the C5 report itself is kept for per-line analysis
TAG=${PROFILE_TAG:-latest}
for c in C5 C4 C3 C2; do
  [ -f gpurun_out/prof_$c.ncu-rep ] && python tools/ncu_summary.py gpurun_out/prof_$c.ncu-rep gpurun_out/${PROFILE_PREFIX:-r2}_ncu_${c}_$TAG > /dev/null
done
cp profiles/ncu_kernel_metrics.json gpurun_out/ 2>/dev/null
rm -f gpurun_out/prof_C4.ncu-rep gpurun_out/prof_C3.ncu-rep gpurun_out/prof_C2.ncu-rep
