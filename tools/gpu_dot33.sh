set -x
mkdir -p gpurun_out
timeout 600 python tools/bench_dot33.py > gpurun_out/dot33.log 2>&1
nvidia-smi --query-gpu=memory.used --format=csv >> gpurun_out/dot33.log
