set -x
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_(axpy_minmax_bulk|dot_bulk|generic|reduce_bulk)' -c 8 -o gpurun_out/prof_secondary python tools/profile_kernels.py > gpurun_out/ncu_secondary.log 2>&1
gzip -f gpurun_out/prof_secondary.ncu-rep
