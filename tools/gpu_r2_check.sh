# Round-2 kernel changes on one B200: the GPU tests that cover them, the A/B
# of the new default policies, the config table for C3/C4.
# Usage: gpurun -- 'bash tools/gpu_r2_check.sh [tag]'
set -x
T=${1:-r2b}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_axpy_dot_gpu.py tests/test_reduce_gpu.py tests/test_ordered_gpu.py tests/test_generic_arena_gpu.py tests/test_fuzz_gpu.py -m gpu -q -p no:cacheprovider --maxfail=10 > gpurun_out/${T}_pytest.log 2>&1
timeout 600 python tools/r2_ab.py > gpurun_out/${T}_ab.jsonl 2> gpurun_out/${T}_ab.err
timeout 600 python tools/bench_configs.py --sections c3,c4 > gpurun_out/${T}_configs.jsonl 2> gpurun_out/${T}_configs.err
