#!/bin/bash
# Final-build C4 sweep (bf16 + f32 at N=2/4, NCCL baseline) and the bench lines at N=2/4 (gpurun --gpus 4)
cd "$(dirname "$0")/.."
O=gpurun_out/sweep_v3; mkdir -p $O
run() { n=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29800 + RANDOM % 100)) "$@"; }
for n in 2 4; do
  run $n bench_reshard.py --pairs all --sizes 1M,16M,256M --iters 20 > $O/sweep_all_n$n.jsonl 2> $O/sweep_all_n$n.err; echo "all n=$n rc=$?"
  run $n bench_reshard.py --pairs all --sizes 16M,256M --iters 20 --dtype f32 > $O/sweep_f32_n$n.jsonl 2> $O/sweep_f32_n$n.err; echo "f32 n=$n rc=$?"
  run $n bench_reshard.py --pairs quick --sizes 1G,4G --iters 5 > $O/sweep_big_n$n.jsonl 2> $O/sweep_big_n$n.err; echo "big n=$n rc=$?"
  run $n bench_reshard.py --pairs quick --sizes 1M,16M,256M,1G --iters 10 --transport nccl > $O/sweep_nccl_n$n.jsonl 2> $O/sweep_nccl_n$n.err; echo "nccl n=$n rc=$?"
  for wl in gpt_block gpt24_train; do
    run $n bench.py --gpus $n --steps 10 --warmup 3 --workload $wl > $O/bench_${wl}_n$n.json 2> $O/bench_${wl}_n$n.err; echo "$wl n=$n rc=$?"
  done
done
python bench_reshard.py --emulate 8 --pairs all --sizes 16M,256M --iters 10 > $O/sweep_emu8.jsonl 2> $O/sweep_emu8.err; echo "emu8 rc=$?"
