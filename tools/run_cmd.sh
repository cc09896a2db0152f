python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
{
python tools/explore.py C5 td_primes64=8,16,24,32 td_primes32=8,16,24
python tools/explore.py C3 td_primes64=8,16,24,32
python tools/explore.py C2 td_primes32=8,16,24,32
} > gpurun_out/explore.jsonl 2> gpurun_out/explore.err
