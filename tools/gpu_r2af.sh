cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2; do for C in 530432 795648 1061376; do
  timeout 300 python bench.py --sim-chains $C --steps 10 --warmup 3 --no-attn --hw-steps 1 --chains 2 --verify-samples 1024 --cpu-seconds 0.1 2>/dev/null | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print($C, round(d['value']/1e6,1), 'M value', round(d['e2e']['value']/1e6,1), 'M e2e', round(d['ms_per_step'],2), 'ms/step')" >> gpurun_out/r2af_c.log
done; done
