# hardware-phase chain refill: new GPU tests, then bench hw phase with refill 32 vs 0 (same box)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest -q tests/test_hwsearch_gpu.py tests/test_targets_gpu.py -m gpu > gpurun_out/rf_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/rf_tests.log
for r in 1 2; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-attn --verify-samples 100000 --cpu-seconds 0.5 --refill 32 > gpurun_out/rf_on_$r.log 2>&1
  timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-attn --verify-samples 100000 --cpu-seconds 0.5 --refill 0 > gpurun_out/rf_off_$r.log 2>&1
done
