# persistent fused blocks A/B (SIP_FUSED_BLOCKS_PER_BATCH=1 = one block per 128 chains)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -x tests/test_engine_gpu.py tests/test_target_parity.py tests/test_api_gpu.py -m gpu > gpurun_out/r2ag_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2ag_tests.log
for r in 1 2; do for M in persistent per_batch; do
  if [ $M = per_batch ]; then export SIP_FUSED_BLOCKS_PER_BATCH=1; else unset SIP_FUSED_BLOCKS_PER_BATCH; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-attn --hw-steps 1 --chains 2 --verify-samples 1024 --cpu-seconds 0.1 2>/dev/null | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); e=d['engine']; print('$M', round(d['value']/1e6,1), 'M value', round(d['e2e']['value']/1e6,1), 'M e2e', 'realistic', {k: round(v['candidates_per_s']/1e6) for k,v in e['realistic_k'].items()})" >> gpurun_out/r2ag_ab.log
done; done
