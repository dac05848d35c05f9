set -x
mkdir -p gpurun_out
timeout 300 python tools/ordered_probe.py > gpurun_out/ordered_probe.jsonl 2> gpurun_out/ordered_probe.err
timeout 900 python -m pytest tests/test_reduce_gpu.py tests/test_axpy_dot_gpu.py tests/test_offload_gpu.py -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_ord.log 2>&1
timeout 600 python tools/ordered_sweep.py > gpurun_out/ordered_sweep.jsonl 2>&1
