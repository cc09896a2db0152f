python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" > gpurun_out/status.txt
EXPLORE_CONFIGS="C3 C5" EXPLORE_ARGS="td_primes64=16,24,32" bash tools/gpu_explore.sh
