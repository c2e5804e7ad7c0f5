cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/d_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/d_gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/d_gpu_tests.log
timeout 300 python bench.py > gpurun_out/d_bench_n1.json 2> gpurun_out/d_bench_n1.err; echo "bench rc=$?"
