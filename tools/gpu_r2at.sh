# hardware-phase chains per GPU: 16 (current default) vs 64 vs 128
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for CH in 16 64 128; do
  timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --verify-samples 100000 --cpu-seconds 0.1 --chains $CH 2>/dev/null | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); g=d['hw']; a=d['attn']['hw']; print('chains $CH', 'gemm', round(g['candidates_per_s'],1), 'busy', round(g['device_busy_frac'],3), 'priced', g['priced'], 'attn', round(a['candidates_per_s'],1), 'busy', round(a['device_busy_frac'],3), 'priced', a['priced'], 'tuned', round(d['tuned']['speedup'],4), round(d['attn']['tuned']['speedup'],4))" >> gpurun_out/r2at.log
done
