mkdir -p gpurun_out
: > gpurun_out/ab6.txt
for lib in build/ab/libN.so paper_2106_03219_b200/libomprt_b200.so build/ab/libN.so paper_2106_03219_b200/libomprt_b200.so; do
  OMPRT_B200_LIB=$lib timeout 300 python tools/ordered_probe.py 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$(basename $lib)', d['kernel'], d['sched'], d['teams'], d['threads'], d['staged']['gbs'])" >> gpurun_out/ab6.txt
  OMPRT_B200_LIB=$lib timeout 300 python tools/c3_ordered_probe.py 2>/dev/null | sed "s#^#$(basename $lib) #" >> gpurun_out/ab6.txt
done
