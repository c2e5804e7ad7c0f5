#!/bin/bash
# r1d: C5 elementwise chain kernels under ncu --set full (DRAM traffic vs algorithmic bytes of
# the forward tanh ladder and the backward chain program), after a plain run exits 0.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --workload gpt24_train --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1d_c5_plain.json 2> gpurun_out/r1d_c5_plain.err
echo "plain rc=$?"
for k in EwLadderKernel EwProgKernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 40 -c 1 \
    -o gpurun_out/r1d_c5_$k python bench.py --workload gpt24_train --steps 3 --warmup 3 --no-cpu-baseline \
    > gpurun_out/r1d_ncu_$k.log 2>&1
  echo "ncu $k rc=$?"
done
