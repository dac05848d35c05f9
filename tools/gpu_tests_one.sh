mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_c_abi.py tests/test_generic_arena_gpu.py -q -p no:cacheprovider > gpurun_out/pytest_one.log 2>&1
