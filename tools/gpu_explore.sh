#!/bin/bash
# Option sweeps on the GPU; output gpurun_out/explore.jsonl
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
{
for c in ${EXPLORE_CONFIGS:-C1 C2 C3 C4 C5}; do python tools/explore.py $c ${EXPLORE_ARGS:-}; done
} > gpurun_out/explore.jsonl 2> gpurun_out/explore.err
