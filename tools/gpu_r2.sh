#!/bin/bash
# Round-2 GPU session: build, smoke, GPU tests, sanitizer, bench.  Logs to gpurun_out/.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/status.txt
if [ "${RUN_TESTS:-1}" = 1 ]; then
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
fi
if [ "${RUN_SAN:-0}" = 1 ]; then bash tools/gpu_sanitize.sh; echo "sanitize done" >> gpurun_out/status.txt; fi
if [ "${RUN_BENCH:-1}" = 1 ]; then
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/status.txt
fi
