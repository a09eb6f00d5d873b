# deferred module eviction A/B: bench hw rates (16 chains) and a 1024-chain GEMM search (60 s)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_targets_gpu.py -k "measure or cache" -m gpu > gpurun_out/r2ak_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2ak_tests.log
for r in 1 2; do for L in paper_2403_16863_b200/libsip.so paper_2403_16863_b200/_obj/libsip_base.so; do
  SIP_LIB=$L timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --verify-samples 100000 --cpu-seconds 0.1 2>/dev/null | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); g=d['hw']; a=d['attn']['hw']; print('$L'[-22:], 'gemm', round(g['candidates_per_s'],1), 'busy', round(g['device_busy_frac'],3), 'attn', round(a['candidates_per_s'],1), 'busy', round(a['device_busy_frac'],3))" >> gpurun_out/r2ak_ab.log
done; done
for L in paper_2403_16863_b200/libsip.so paper_2403_16863_b200/_obj/libsip_base.so; do
  SIP_LIB=$L timeout 600 python tools/long_search.py --target gemm --classes extended --chains 1024 --max-seconds 60 --verify-samples 100000 --out gpurun_out/r2ak_long_$(basename $L).json > gpurun_out/r2ak_long_$(basename $L).log 2>&1
done
