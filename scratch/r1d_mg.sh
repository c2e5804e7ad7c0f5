#!/bin/bash
# r1d: dist parity (pipelined host path with scattered replicated inputs) + C3/C5 bench at N=2/4,
# RH_E2E_SCATTER A/B for the e2e line.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -m gpu -x -q > gpurun_out/d_mg_dist.log 2>&1
echo "dist rc=$?"; tail -3 gpurun_out/d_mg_dist.log
for n in 2 4; do
  for sc in 1 0; do
    RH_E2E_SCATTER=$sc timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29700 + n + 10*sc)) bench.py --gpus $n --steps 10 --warmup 3 --workload gpt_block \
      > gpurun_out/d_mg_gpt_block_n${n}_sc$sc.json 2> gpurun_out/d_mg_gpt_block_n${n}_sc$sc.err
    echo "n=$n sc=$sc rc=$?"
  done
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29750 + n)) bench.py --gpus $n --steps 10 --warmup 3 --workload gpt24_train \
      > gpurun_out/d_mg_gpt24_train_n$n.json 2> gpurun_out/d_mg_gpt24_train_n$n.err
  echo "c5 n=$n rc=$?"
done
