set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_axpy_dot_gpu.py tests/test_offload_gpu.py -q -p no:cacheprovider -x > gpurun_out/pytest_axpy_dot.log 2>&1
timeout 900 python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
