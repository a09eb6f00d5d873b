cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for sg in 1.0 2.0 3.0 8.0; do
  timeout 90 python tools/attn_sigma_probe.py paper_2403_16863_b200/targets/attn_fwd.cubin 1 8 1024 $sg >> gpurun_out/sig.log 2>&1; echo "base sigma $sg rc=$?" >> gpurun_out/sig.log
done
timeout 90 python tools/attn_sigma_probe.py paper_2403_16863_b200/_obj/attn_spec.cubin 1 8 1024 3.0 >> gpurun_out/sig.log 2>&1; echo "spec sigma 3 rc=$?" >> gpurun_out/sig.log
