mkdir -p gpurun_out
for cfg in "0 256" "0 1024"; do
  set -- $cfg
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:ordered_rows -c 1 -o gpurun_out/prof_rows_v$1_t$2 python tools/profile_ordered.py $1 $2 > gpurun_out/ncu_rows_v$1_t$2.log 2>&1
  gzip -f gpurun_out/prof_rows_v$1_t$2.ncu-rep
done
