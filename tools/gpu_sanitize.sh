set -x
mkdir -p gpurun_out
timeout 600 python tools/fence_probe.py > gpurun_out/fence_probe.jsonl 2>&1
for tool in synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_driver.py > gpurun_out/sanitize_$tool.log 2>&1
done
