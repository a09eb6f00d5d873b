# SlotRow iteration: fused parity, same-box A/B against dense rows, ncu
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r2g}
timeout 900 python -m pytest -q -x tests/test_engine_gpu.py tests/test_target_parity.py -m gpu > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
for r in 1 2; do for M in dense slots; do
  if [ $M = dense ]; then export SIP_NO_SLOTS=1; else unset SIP_NO_SLOTS; fi
  timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-attn --hw-steps 1 --chains 2 --verify-samples 1024 --cpu-seconds 0.1 2>/dev/null | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); e=d['engine']; print('$M', round(d['value']/1e6,1), 'M cand/s', round(d['ms_per_step'],2), 'ms/step chains', e['chains_per_gpu'])" >> gpurun_out/${TAG}_ab.log
done; done
unset SIP_NO_SLOTS
timeout 600 ncu --set full --import-source on --clock-control none -k regex:anneal_fused -s 1 -c 1 \
  -o gpurun_out/engine_${TAG} python tools/profile_kernels.py engine 265216 > gpurun_out/${TAG}_ncu.log 2>&1
