# A/B of fold_row_in_order L2 prefetch variants on config 4 (generic ORDERED) and the literal ORDERED walk
mkdir -p gpurun_out
: > gpurun_out/ab_fold.txt
for rep in 1 2; do
for lib in paper_2106_03219_b200/libomprt_b200.so build/ab/libP256.so build/ab/libP512.so build/ab/libP1024.so build/ab/libB512.so build/ab/libB1024.so; do
  OMPRT_B200_LIB=$lib timeout 300 python tools/c4_probe.py 2>&1 | grep '"f64"' | sed "s#^#$(basename $lib) #" >> gpurun_out/ab_fold.txt
done
done
