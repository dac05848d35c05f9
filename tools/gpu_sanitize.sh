set -x
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_driver.py > gpurun_out/sanitize_$tool.log 2>&1
done
