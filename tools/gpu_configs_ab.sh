mkdir -p gpurun_out
for t in 256 384 256 384; do
  OMPRT_DEFAULT_THREADS=$t timeout 900 python tools/bench_configs.py --reps 100 > gpurun_out/configs_t$t.jsonl 2>&1
  cp gpurun_out/configs_t$t.jsonl gpurun_out/configs_t${t}_$(date +%s%N).jsonl
done
