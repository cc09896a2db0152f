set -u
bash tools/ab.sh build/lib_base.so build/lib_new.so C4 C2
python tools/stride2_time.py >> gpurun_out/exp.jsonl 2>&1
