#!/bin/bash
# Option sweeps on the GPU; output gpurun_out/explore.jsonl
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
{
python tools/explore.py C1 force_path=0,1,2
python tools/explore.py C2 force_path=0,2 td_primes32=0,8,16,24,32
python tools/explore.py C3 win64=1,2,3 td_primes64=8,16,24,32
python tools/explore.py C4 force_path=0,1
python tools/explore.py C5 td_primes64=8,24
} > gpurun_out/explore.jsonl 2> gpurun_out/explore.err
