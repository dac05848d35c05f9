mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_reduce_ordered_bulk -c 2 -o gpurun_out/prof_ordered python tools/profile_ordered.py > gpurun_out/ncu_ordered.log 2>&1
