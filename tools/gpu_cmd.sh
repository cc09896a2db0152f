set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "prefix or random_all or witness_option or short_array or edge or chernick" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
for c in C5 C3 C2; do timeout 600 python tools/explore.py $c >> gpurun_out/exp.jsonl 2>&1; done
