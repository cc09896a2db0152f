bash tools/gpu_session.sh
