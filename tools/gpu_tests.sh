set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --maxfail=40 --durations=5 > gpurun_out/pytest_gpu.log 2>&1
