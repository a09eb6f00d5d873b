# attention rescale fix: the large-score probe that hung, the attention GPU tests, timing vs the old cubin
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for sg in 1.0 2.0 3.0 8.0; do
  timeout 90 python tools/attn_sigma_probe.py paper_2403_16863_b200/targets/attn_fwd.cubin 1 8 1024 $sg >> gpurun_out/fix_sig.log 2>&1; echo "fixed sigma $sg rc=$?" >> gpurun_out/fix_sig.log
done
timeout 900 python -m pytest -q tests/test_targets_gpu.py -m gpu -k "attention" > gpurun_out/fix_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/fix_tests.log
AB_ROUNDS=9 timeout 900 python tools/attn_ab.py paper_2403_16863_b200/_obj/attn_old.cubin > gpurun_out/fix_ab.log 2>&1
AB_ROUNDS=9 AB_S=1024 timeout 900 python tools/attn_ab.py paper_2403_16863_b200/_obj/attn_old.cubin > gpurun_out/fix_ab1k.log 2>&1
