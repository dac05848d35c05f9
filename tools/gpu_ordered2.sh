mkdir -p gpurun_out
timeout 300 python tools/ordered_probe.py > gpurun_out/ordered_probe.jsonl 2> gpurun_out/ordered_probe.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ordered_rows -c 1 -o gpurun_out/prof_rows_v0_t256 python tools/profile_ordered.py 0 256 > gpurun_out/ncu_rows.log 2>&1
gzip -f gpurun_out/prof_rows_v0_t256.ncu-rep
