# chunk size of a 128-chain round: 64 (two references) vs 256 (one)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2; do for CK in 64 256; do
  SIP_ROUND_CHUNK=$CK timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --verify-samples 100000 --cpu-seconds 0.1 2>/dev/null | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); g=d['hw']; a=d['attn']['hw']; print('chunk $CK', 'gemm', round(g['candidates_per_s'],1), 'busy', round(g['device_busy_frac'],3), 'attn', round(a['candidates_per_s'],1), 'busy', round(a['device_busy_frac'],3), 'tuned', round(d['tuned']['speedup'],4), [round(x,4) for x in d['tuned']['speedup_iqr']], round(d['attn']['tuned']['speedup'],4))" >> gpurun_out/r2au.log
done; done
