set -x
mkdir -p gpurun_out
timeout 600 python tools/sweep.py --b2b > gpurun_out/sweep_b2b.jsonl 2> gpurun_out/sweep_b2b.err
timeout 900 python tools/sweep.py --quick > gpurun_out/sweep2.jsonl 2> gpurun_out/sweep2.err
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py --steps 1000 --warmup 10 > gpurun_out/bench.log 2>&1
