#!/bin/bash
# r1d: rematerialized tanh values (RH_REMAT=1): bit-exact parity, then the C5 step A/B at N=1.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "remat or fusion_bit_exact or ladder" > gpurun_out/r1d_remat_tests.log 2>&1
echo "tests rc=$?"; tail -15 gpurun_out/r1d_remat_tests.log
for r in 1 0; do
  RH_REMAT=$r timeout 400 python bench.py --workload gpt24_train --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r1d_c5_remat$r.json 2> gpurun_out/r1d_c5_remat$r.err
  echo "c5 remat=$r rc=$?"
done
