# run_search with range seeds: API tests + e2e A/B against HEAD's driver (array seeds)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -x tests/test_api_gpu.py tests/test_acceptance_gpu.py tests/test_engine_gpu.py -m gpu > gpurun_out/r2ae_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2ae_tests.log
for r in 1 2; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-attn --hw-steps 1 --chains 2 --verify-samples 1024 --cpu-seconds 0.1 2>/dev/null | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('range seeds', round(d['value']/1e6,1), 'M value', round(d['e2e']['value']/1e6,1), 'M e2e')" >> gpurun_out/r2ae_ab.log
done
