#!/bin/bash
# Multi-GPU round: dist parity tests, then bench lines at N=2 and N=4 (run under gpurun --gpus 4).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dist.py -m gpu -x -q > gpurun_out/mg_dist.log 2>&1
echo "dist rc=$?"; tail -3 gpurun_out/mg_dist.log
for wl in gpt_block gpt24_train; do
  for n in 2 4; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29700 + n)) bench.py --gpus $n --steps 10 --warmup 3 --workload $wl \
      > gpurun_out/mg_${wl}_n$n.json 2> gpurun_out/mg_${wl}_n$n.err
    echo "$wl n=$n rc=$?"
  done
done
