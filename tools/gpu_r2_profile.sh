# ncu evidence, round 2: the bench kernel (launch list + --set full, with the
# capture's provenance) and the secondary construct kernels (--set full).
# Usage: gpurun -- 'bash tools/gpu_r2_profile.sh'
set -x
mkdir -p gpurun_out
bash tools/gpu_profile.sh
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:'k_axpy_minmax_bulk|k_axpy_minmax_ext|k_reduce_ext|k_dot_bulk|k_generic' -s 0 -c 14 \
  -o gpurun_out/prof_secondary python tools/profile_kernels.py > gpurun_out/ncu_secondary.log 2>&1
# summarise on the box (the reports themselves can exceed gpurun's 64 MiB merge)
python tools/ncu_summary.py launches gpurun_out/launches.csv gpurun_out/launches_bench.json > /dev/null
python tools/ncu_summary.py report gpurun_out/prof_bench.ncu-rep gpurun_out/ncu_bench_kernel.json \
  --algorithmic-bytes 8589934592 --meta gpurun_out/prof_bench.meta.json > /dev/null
python tools/ncu_summary.py report gpurun_out/prof_secondary.ncu-rep gpurun_out/ncu_secondary.json > /dev/null
ncu -i gpurun_out/prof_secondary.ncu-rep --page details --csv > gpurun_out/ncu_secondary_details.csv 2>/dev/null
rm -f gpurun_out/launches.csv
for f in gpurun_out/*.ncu-rep; do gzip -f "$f"; s=$(stat -c %s "$f.gz"); [ "$s" -gt 20000000 ] && rm -f "$f.gz"; done
ls -la gpurun_out
