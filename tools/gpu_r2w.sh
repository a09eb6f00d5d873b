# A/B: current libsip.so vs _obj/libsip_base.so (HEAD) on value/e2e; engine + API parity tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r2w}
timeout 1200 python -m pytest -q -x tests/test_engine_gpu.py tests/test_target_parity.py tests/test_api_gpu.py tests/test_acceptance_gpu.py -m gpu > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
for r in 1 2; do for L in paper_2403_16863_b200/libsip.so paper_2403_16863_b200/_obj/libsip_base.so; do
  SIP_LIB=$L timeout 300 python bench.py --steps 10 --warmup 3 --no-attn --hw-steps 1 --chains 2 --verify-samples 1024 --cpu-seconds 0.1 2>/dev/null | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); e=d['engine']; print('$L'[-22:], round(d['value']/1e6,1), 'M value', round(d['e2e']['value']/1e6,1), 'M e2e', round(d['ms_per_step'],3), 'ms')" >> gpurun_out/${TAG}_ab.log
done; done
