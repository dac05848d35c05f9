mkdir -p gpurun_out
: > gpurun_out/ab5.txt
for lib in build/ab/libN.so paper_2106_03219_b200/libomprt_b200.so build/ab/libN.so paper_2106_03219_b200/libomprt_b200.so; do
  OMPRT_B200_LIB=$lib timeout 300 python bench.py --steps 1000 --e2e-steps 0 --no-cpu-baseline --ordered-steps 0 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $lib)', d['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'])" >> gpurun_out/ab5.txt
  OMPRT_B200_LIB=$lib timeout 300 python tools/c4_probe.py 2>/dev/null | sed "s#^#$(basename $lib) #" >> gpurun_out/ab5.txt
done
