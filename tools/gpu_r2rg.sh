# step-mode propose with warp-per-chain candidate rows: engine/hwsearch/targets GPU tests,
# the load/propose probe, and the bench hw phase with refill 0 / 32 / 64 (same box)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest -q tests/test_hwsearch_gpu.py tests/test_engine_gpu.py tests/test_targets_gpu.py tests/test_api_gpu.py -m gpu > gpurun_out/rg_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/rg_tests.log
timeout 600 python tools/hw_load_probe.py > gpurun_out/rg_probe.log 2>&1
for r in 1 2; do
  for f in 0 32 64; do
    timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-attn --verify-samples 100000 --cpu-seconds 0.5 --refill $f > gpurun_out/rg_${f}_${r}.log 2>&1
    tail -1 gpurun_out/rg_${f}_${r}.log | python -c "import json,sys; d=json.loads(sys.stdin.read())['hw']; print('refill', $f, 'round', $r, round(d['candidates_per_s'],1), round(d['device_busy_frac'],3), d['priced'])" >> gpurun_out/rg_summary.log 2>&1
  done
done
