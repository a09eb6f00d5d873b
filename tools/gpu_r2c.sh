cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest -q tests/test_difftest_gpu.py tests/test_target_parity.py tests/test_api_gpu.py tests/test_acceptance_gpu.py -m gpu > gpurun_out/r2c_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2c_tests.log
timeout 900 python tools/upper_bound.py gpurun_out/upper_bound.json > gpurun_out/r2c_ub.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2c_ref.log 2>&1
echo "ref rc=$?" >> gpurun_out/r2c_ref.log
