mkdir -p gpurun_out
for t in 256 128 64 256; do
  timeout 300 python bench.py --threads $t --steps 1000 --warmup 10 --e2e-steps 0 --no-cpu-baseline --ordered-steps 0 > gpurun_out/bench_t$t.log 2>&1
  grep '^{' gpurun_out/bench_t$t.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($t, d['value'], d['roofline']['achieved'], d['clocks'])" >> gpurun_out/threads_sweep.txt
done
