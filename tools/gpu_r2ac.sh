# MT row in pairs A/B: libsip.so (pairs) vs _obj/libsip_mtscalar.so
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r2ac}
timeout 1200 python -m pytest -q -x tests/test_engine_gpu.py tests/test_target_parity.py tests/test_api_gpu.py -m gpu > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
for r in 1 2; do for L in paper_2403_16863_b200/libsip.so paper_2403_16863_b200/_obj/libsip_mtscalar.so; do
  SIP_LIB=$L timeout 300 python bench.py --steps 10 --warmup 3 --no-attn --hw-steps 1 --chains 2 --verify-samples 1024 --cpu-seconds 0.1 2>/dev/null | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); e=d['engine']; print('$L'[-24:], round(d['value']/1e6,1), 'M value', round(d['e2e']['value']/1e6,1), 'M e2e', 'realistic', {k: round(v['candidates_per_s']/1e6) for k,v in e['realistic_k'].items()})" >> gpurun_out/${TAG}_ab.log
done; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:anneal_fused -s 1 -c 1 \
  -o gpurun_out/engine_${TAG} python tools/profile_kernels.py engine > gpurun_out/${TAG}_ncu.log 2>&1
