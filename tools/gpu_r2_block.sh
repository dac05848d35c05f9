# CTA-size decoupling of the SPMD kernels: the GPU tests, then the sweep.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_reduce_gpu.py tests/test_axpy_dot_gpu.py tests/test_fuzz_gpu.py tests/test_parallel_gpu.py tests/test_trace_gpu.py tests/test_offload_gpu.py -m gpu -q -p no:cacheprovider --maxfail=10 > gpurun_out/r2g_pytest.log 2>&1
timeout 900 python tools/block_sweep.py > gpurun_out/r2g_block_sweep.jsonl 2> gpurun_out/r2g_block_sweep.err
