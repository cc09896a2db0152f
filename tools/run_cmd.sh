bash tools/gpu_session.sh
EXPLORE_CONFIGS="C3 C5" bash tools/gpu_explore.sh
