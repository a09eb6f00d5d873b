# engine chains per GPU beyond eight waves (8 / 12 / 16 waves of 7 x 148 blocks of 128),
# two alternating rounds, plus the hwsearch GPU tests with the cohort release
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest -q tests/test_hwsearch_gpu.py -m gpu > gpurun_out/wv_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/wv_tests.log
for r in 1 2; do for C in 1060864 1591296 2121728; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-attn --hw-steps 1 --chains 2 --verify-samples 1024 --cpu-seconds 0.1 --sim-chains $C 2>/dev/null | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print($C, round(d['value']/1e6,1), 'M cand/s e2e', round(d['e2e']['value']/1e6,1), round(d['ms_per_step'],2), 'ms/step')" >> gpurun_out/wv.log
done; done
