mkdir -p gpurun_out
: > gpurun_out/ab.txt
for rep in 1 2; do
for lib in build/ab/libH.so build/ab/libA.so paper_2106_03219_b200/libomprt_b200.so; do
  OMPRT_B200_LIB=$lib timeout 300 python tools/ordered_probe.py 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$lib'.split('/')[-1], d['kernel'], d['sched'], d['teams'], d['threads'], d['staged']['gbs'])" >> gpurun_out/ab.txt
done
done
