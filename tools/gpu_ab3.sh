mkdir -p gpurun_out
: > gpurun_out/ab3.txt
for lib in build/ab/libH.so paper_2106_03219_b200/libomprt_b200.so build/ab/libH.so paper_2106_03219_b200/libomprt_b200.so; do
  OMPRT_B200_LIB=$lib timeout 300 python tools/c3_probe.py 2>/dev/null | sed "s#^#$(basename $lib) #" >> gpurun_out/ab3.txt
done
