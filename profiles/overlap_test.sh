#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/overlap; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dist.py -m gpu -x -q > $O/dist.log 2>&1; echo "dist rc=$?"; tail -3 $O/dist.log
for n in 2 4; do
  for ov in "" "--no-overlap"; do
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29900 + n)) \
      bench.py --gpus $n --steps 10 --warmup 3 --workload gpt24_train --no-cpu-baseline $ov > $O/c5_n$n$ov.json 2> $O/c5_n$n$ov.err
    echo "c5 n=$n $ov rc=$?"
  done
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29910 + n)) \
      bench.py --gpus $n --steps 10 --warmup 3 > $O/c3_n$n.json 2> $O/c3_n$n.err; echo "c3 n=$n rc=$?"
done
