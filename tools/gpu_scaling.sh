# Multi-GPU scaling of the bench on one node (needs >= 8 GPUs): NCCL combine
# overlapped with the next step (default) vs the exchange fused into the
# reduction kernel over NVLink peer memory (--exchange p2p).  One JSON line per
# run in gpurun_out/scaling.jsonl.
set -x
mkdir -p gpurun_out
: > gpurun_out/scaling.jsonl
PORT=29600
for n in 1 2 4 8; do
  for ex in nccl p2p; do
    [ "$n" = 1 ] && [ "$ex" = p2p ] && continue
    PORT=$((PORT + 1))
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $PORT bench.py --gpus $n --steps 500 --warmup 5 --e2e-steps 1 --exchange $ex \
      --no-cpu-baseline 2> gpurun_out/scaling_${n}_${ex}.err | grep '^{' >> gpurun_out/scaling.jsonl
  done
done
