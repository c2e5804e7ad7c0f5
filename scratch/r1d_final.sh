#!/bin/bash
# r1d: full GPU suite (single-GPU + dist at N=2/4) with rematerialization on by default, smoke,
# C5 N=1 bench.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1100 python -m pytest tests -m gpu -x -q > gpurun_out/f_gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/f_gpu_tests.log
timeout 400 python bench.py --workload gpt24_train --steps 5 --warmup 3 > gpurun_out/f_c5_n1.json 2> gpurun_out/f_c5_n1.err; echo "c5 rc=$?"
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29811 \
  bench.py --gpus 4 --steps 10 --warmup 3 --workload gpt24_train > gpurun_out/f_c5_n4.json 2> gpurun_out/f_c5_n4.err; echo "c5 n4 rc=$?"
