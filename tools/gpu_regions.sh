set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_regions_gpu.py tests/test_forge_bridge.py -m gpu -q -p no:cacheprovider -x --durations=10 > gpurun_out/pytest_regions.log 2>&1
tail -5 gpurun_out/pytest_regions.log
