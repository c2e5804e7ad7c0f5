#!/bin/bash
# r1d: the rematerializing chain kernel under ncu --set full (after a plain run exits 0).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python bench.py --workload gpt24_train --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1d_c5_plain2.json 2>&1
echo "plain rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"EwProgKernel<1, 1>|EwProgKernelILb1ELb1" -s 20 -c 1 \
  -o gpurun_out/r1d_c5_remat_kernel python bench.py --workload gpt24_train --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/r1d_ncu_remat.log 2>&1
echo "ncu rc=$?"
