# ncu evidence for the bench's dominant kernel (one GPU, never multi-rank):
# the launch list of the bench command, one --set full capture of the bench
# kernel, and the capture's provenance (UTC time, sha of the library that ran)
# so bench.py can tell whether the committed capture is of the current build.
set -x
mkdir -p gpurun_out
B="python bench.py --e2e-steps 0 --no-cpu-baseline --ordered-steps 5"
printf '{"captured_at": "%s", "lib_sha16": "%s", "src_sha16": "%s"}\n' "$(date -u +%Y-%m-%dT%H:%M:%SZ)" \
  "$(sha256sum paper_2106_03219_b200/libomprt_b200.so | cut -c1-16)" \
  "$(python -c 'from paper_2106_03219_b200 import _build; print(_build.source_sha16())')" > gpurun_out/prof_bench.meta.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $B --steps 20 --warmup 3 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_reduce_bulk -s 3 -c 1 -o gpurun_out/prof_bench $B --steps 5 --warmup 1 > gpurun_out/ncu_full.log 2>&1
