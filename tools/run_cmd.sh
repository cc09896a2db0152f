python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for CFG in C5 C4; do
EXP="python tools/explore.py $CFG"
$EXP > gpurun_out/ncu_plain_$CFG.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"classify_kernel|sieve_kernel|qscatter" -s 6 -c 3 -o gpurun_out/prof2_$CFG $EXP > gpurun_out/ncu2_$CFG.log 2>&1
echo "$CFG rc=$?" >> gpurun_out/ncu_status.txt
done
