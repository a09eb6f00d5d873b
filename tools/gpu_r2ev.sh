# evaluator A/B: images gathered on the load workers (new) vs built serially before the
# workers start (old, paper_2403_16863_b200/_obj/libsip_old.so); two alternating rounds
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest -q tests/test_targets_gpu.py tests/test_api_gpu.py -m gpu > gpurun_out/ev_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/ev_tests.log
for r in 1 2; do
  SIP_LIB=paper_2403_16863_b200/_obj/libsip_old.so timeout 300 python tools/hw_round_probe.py gemm 128 >> gpurun_out/ev_old.log 2>&1
  SIP_EVAL_TIMING=1 timeout 300 python tools/hw_round_probe.py gemm 128 >> gpurun_out/ev_new.log 2>> gpurun_out/ev_new.err
done
