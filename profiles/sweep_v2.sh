#!/bin/bash
# C4 resharding sweep (graph captured before the timed region) + C5 bench at N=2/4; gpurun --gpus 4
cd "$(dirname "$0")/.."
O=gpurun_out/sweep_v2; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "reduce_outputs or fusion" > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
run() { n=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29800 + RANDOM % 100)) "$@"; }
for n in 2 4; do
  run $n bench_reshard.py --pairs all --sizes 1M,16M,256M --iters 20 > $O/sweep_all_n$n.jsonl 2> $O/sweep_all_n$n.err; echo "all n=$n rc=$?"
  run $n bench_reshard.py --pairs quick --sizes 1G,4G --iters 5 > $O/sweep_big_n$n.jsonl 2> $O/sweep_big_n$n.err; echo "big n=$n rc=$?"
  run $n bench_reshard.py --pairs quick --sizes 1M,16M,256M,1G --iters 10 --transport nccl > $O/sweep_nccl_n$n.jsonl 2> $O/sweep_nccl_n$n.err; echo "nccl n=$n rc=$?"
  run $n bench.py --gpus $n --steps 10 --warmup 3 --workload gpt24_train > $O/c5_n$n.json 2> $O/c5_n$n.err; echo "c5 n=$n rc=$?"
done
