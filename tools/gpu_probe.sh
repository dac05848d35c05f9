set -x
mkdir -p gpurun_out
timeout 1200 python tools/steady_probe.py 500 bulk > gpurun_out/steady_bulk.jsonl 2>&1
