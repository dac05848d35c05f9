set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_reduce_gpu.py -q -p no:cacheprovider --maxfail=20 > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
