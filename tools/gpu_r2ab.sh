# checkpoint spacing A/B with SlotRow chains (parity of each variant first)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for V in ck16 ck64; do
  SIP_LIB=paper_2403_16863_b200/_obj/libsip_$V.so timeout 900 python -m pytest -q -x tests/test_engine_gpu.py -m gpu > gpurun_out/r2ab_tests_$V.log 2>&1
  echo "tests rc=$?" >> gpurun_out/r2ab_tests_$V.log
done
for r in 1 2; do for L in paper_2403_16863_b200/libsip.so paper_2403_16863_b200/_obj/libsip_ck16.so paper_2403_16863_b200/_obj/libsip_ck64.so; do
  SIP_LIB=$L timeout 300 python bench.py --steps 10 --warmup 3 --no-attn --hw-steps 1 --chains 2 --verify-samples 1024 --cpu-seconds 0.1 2>/dev/null | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); e=d['engine']; print('$L'[-22:], round(d['value']/1e6,1), 'M value', round(d['e2e']['value']/1e6,1), 'M e2e', round(e['avg_replay_steps_per_candidate'],1), 'steps/cand')" >> gpurun_out/r2ab_ab.log
done; done
