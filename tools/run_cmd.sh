NCU_CFG=C5 bash tools/gpu_ncu.sh
