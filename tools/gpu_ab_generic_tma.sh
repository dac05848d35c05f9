# A/B: generic ORDERED worker fold, literal 32-byte walk vs TMA-fed 64-byte row windows
mkdir -p gpurun_out
: > gpurun_out/ab_generic_tma.txt
for rep in 1 2; do
for lib in paper_2106_03219_b200/libomprt_b200.so build/ab/libT.so; do
  OMPRT_B200_LIB=$lib timeout 300 python tools/c4_probe.py 2>&1 | grep f64 | sed "s#^#$(basename $lib) #" >> gpurun_out/ab_generic_tma.txt
done
done
OMPRT_B200_LIB=build/ab/libT.so timeout 600 python -m pytest tests -m gpu -q -k "generic" -p no:cacheprovider > gpurun_out/ab_generic_tma_tests.txt 2>&1
