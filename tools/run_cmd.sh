python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" > gpurun_out/status.txt
EXPLORE_CONFIGS="C3 C5" EXPLORE_ARGS="win64=1,2,3 mr2_group=3,6" bash tools/gpu_explore.sh
