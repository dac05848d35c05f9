mkdir -p gpurun_out
: > gpurun_out/ab2.txt
for lib in build/ab/libH.so paper_2106_03219_b200/libomprt_b200.so; do
  OMPRT_B200_LIB=$lib timeout 300 python tools/c3_ordered_probe.py 2>/dev/null | sed "s#^#$(basename $lib) #" >> gpurun_out/ab2.txt
  OMPRT_B200_LIB=$lib timeout 300 python tools/ordered_probe.py 2>/dev/null | grep dot | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$(basename $lib)', d['kernel'], d['threads'], 'literal', d['literal']['gbs'])" >> gpurun_out/ab2.txt
done
