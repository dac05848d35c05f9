# The round-end sequence on one B200: smoke, the GPU suite, both bench arms,
# and the multi-rank bench (2 ranks sharing the one GPU over gloo).
# Usage (from the repo root):  gpurun -- 'bash tools/gpu_round.sh [tag]'
set -x
T=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --maxfail=20 --durations=15 > gpurun_out/${T}_pytest_gpu.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${T}_bench_ref.log 2>&1
timeout 900 python bench.py --gpus 2 --steps 20 --warmup 5 --backend gloo > gpurun_out/${T}_bench_g2_gloo.log 2>&1
