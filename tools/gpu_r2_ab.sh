# A/B of the round-2 policies (tools/r2_ab.py) plus the generic-mode tests.
# Usage: gpurun -- 'bash tools/gpu_r2_ab.sh [tag] [sections]'
set -x
T=${1:-r2ab}
S=${2:-c3,c4}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_generic_arena_gpu.py tests/test_fuzz_gpu.py -m gpu -q -p no:cacheprovider --maxfail=10 > gpurun_out/${T}_pytest.log 2>&1
timeout 600 python tools/r2_ab.py --sections $S > gpurun_out/${T}_ab.jsonl 2> gpurun_out/${T}_ab.err
