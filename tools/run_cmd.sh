nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mr_step_bench tools/mr_step_bench.cu && timeout 120 tools/mr_step_bench > gpurun_out/mr_step.json 2>&1
