# A/B: generic SPMD fp64 workers with one vs two accumulator sets
mkdir -p gpurun_out
: > gpurun_out/ab_generic_na.txt
for rep in 1 2 3; do
for lib in paper_2106_03219_b200/libomprt_b200.so build/ab/libNA2.so; do
  OMPRT_B200_LIB=$lib timeout 300 python tools/c4_probe.py 2>&1 | grep '"f64", "ordered": false' | sed "s#^#$(basename $lib) #" >> gpurun_out/ab_generic_na.txt
done
done
OMPRT_B200_LIB=build/ab/libNA2.so timeout 600 python -m pytest tests -m gpu -q -k "generic" -p no:cacheprovider > gpurun_out/ab_generic_na_tests.txt 2>&1
