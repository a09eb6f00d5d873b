# same-box A/B of two libsip builds on the engine headline (alternating, 2 rounds)
for r in 1 2; do for L in "$@"; do SIP_LIB=$L timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-attn --hw-steps 1 --chains 2 --verify-samples 1024 --cpu-seconds 0.1 2>/dev/null | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$L'[-24:], round(d['value']/1e6,1), 'M cand/s', round(d['ms_per_step'],2), 'ms/step')"; done; done
