set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/status.txt
BENCH_SAME_DEVICE=1 BENCH_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench2_func.json 2> gpurun_out/bench2_func.err; echo "bench2 rc=$?" >> gpurun_out/status.txt
BENCH_SAME_DEVICE=1 BENCH_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 3 --warmup 3 --config C4 --scaling strong --no-per-config > gpurun_out/bench2_c4_func.json 2> gpurun_out/bench2_c4_func.err; echo "bench2 c4 rc=$?" >> gpurun_out/status.txt
timeout 600 python tools/explore.py C5 chunk_log2=26,27,28 > gpurun_out/exp_chunk.jsonl 2>&1
timeout 600 python tools/explore.py C3 chunk_log2=24,25,26 >> gpurun_out/exp_chunk.jsonl 2>&1
timeout 600 python tools/explore.py C4 chunk_log2=27,28,29,30 >> gpurun_out/exp_chunk.jsonl 2>&1
timeout 600 python tools/explore.py C2 chunk_log2=22,23,24 >> gpurun_out/exp_chunk.jsonl 2>&1
