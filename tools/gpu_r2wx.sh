# 16-wave engine default: default bench line, engine ncu at the new chain count, and the
# chain-count sweep continued to 24 / 32 waves (two alternating rounds)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/wx_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/wx_bench.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:anneal_fused -s 1 -c 1 \
  -o gpurun_out/engine_wx python tools/profile_kernels.py engine > gpurun_out/wx_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/wx_ncu.log
for r in 1 2; do for C in 2121728 3182592 4243456; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-attn --hw-steps 1 --chains 2 --verify-samples 1024 --cpu-seconds 0.1 --sim-chains $C 2>/dev/null | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print($C, round(d['value']/1e6,1), 'M cand/s e2e', round(d['e2e']['value']/1e6,1), round(d['ms_per_step'],2), 'ms/step')" >> gpurun_out/wx.log
done; done
