# streamed evaluator rounds: tests, then hw-rate A/B against the captured-graph round
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -x tests/test_targets_gpu.py tests/test_api_gpu.py tests/test_acceptance_gpu.py -m gpu > gpurun_out/r2u_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2u_tests.log
for r in 1 2; do for M in graph streamed; do
  if [ $M = graph ]; then export SIP_ROUND_GRAPH=1; else unset SIP_ROUND_GRAPH; fi
  SIP_EVAL_TIMING=1 timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --verify-samples 100000 --cpu-seconds 0.1 2>gpurun_out/r2u_timing_${M}_$r.log | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); g=d['hw']; a=d['attn']['hw']; print('$M', 'gemm', round(g['candidates_per_s'],1), 'busy', round(g['device_busy_frac'],3), 'attn', round(a['candidates_per_s'],1), 'busy', round(a['device_busy_frac'],3), 'tuned', round(d['tuned']['speedup'],4), d['tuned']['speedup_iqr'])" >> gpurun_out/r2u_ab.log
done; done
