# re-timing through the round protocol: evaluator GPU tests, then the bench (default flags)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest -q tests/test_targets_gpu.py tests/test_hwsearch_gpu.py -m gpu > gpurun_out/rt_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/rt_tests.log
timeout 1200 python bench.py > gpurun_out/rt_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/rt_bench.log
