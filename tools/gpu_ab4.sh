mkdir -p gpurun_out
: > gpurun_out/ab4.txt
for lib in build/ab/libN.so paper_2106_03219_b200/libomprt_b200.so build/ab/libN.so paper_2106_03219_b200/libomprt_b200.so; do
  OMPRT_B200_LIB=$lib timeout 300 python tools/c4_probe.py 2>/dev/null | sed "s#^#$(basename $lib) #" >> gpurun_out/ab4.txt
done
