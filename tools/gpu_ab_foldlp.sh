# A/B of the literal in-order fold's load policy (256-byte L2 promotion vs none vs evict_first) on config 4 ORDERED and the literal ORDERED walk
mkdir -p gpurun_out
: > gpurun_out/ab_foldlp.txt
for rep in 1 2; do
for lib in paper_2106_03219_b200/libomprt_b200.so build/ab/libNC.so build/ab/libEF.so; do
  OMPRT_B200_LIB=$lib timeout 300 python tools/c4_probe.py 2>&1 | grep '"f64", "ordered": true' | sed "s#^#$(basename $lib) #" >> gpurun_out/ab_foldlp.txt
  OMPRT_B200_LIB=$lib timeout 300 python tools/ordered_sweep.py vars=20 distribute:1:148:384 2>&1 | sed "s#^#$(basename $lib) #" >> gpurun_out/ab_foldlp.txt
done
done
