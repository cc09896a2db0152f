#!/bin/bash
# One GPU session: build, smoke, micro-benchmark, GPU tests, bench.  Logs to gpurun_out/.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu | head -20 > gpurun_out/lscpu.txt; nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/status.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/imad_peak tools/imad_peak.cu && timeout 60 tools/imad_peak > gpurun_out/imad_peak.json 2>&1; echo "imad rc=$?" >> gpurun_out/status.txt
timeout ${TEST_TIMEOUT:-900} python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 600 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/status.txt
