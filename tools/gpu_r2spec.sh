# attention: speculative first-half exponentials, bitwise check + timing A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/attn_spec_check.py paper_2403_16863_b200/_obj/attn_spec.cubin > gpurun_out/spec_check.log 2>&1
echo "check rc=$?" >> gpurun_out/spec_check.log
AB_ROUNDS=9 timeout 900 python tools/attn_ab.py paper_2403_16863_b200/_obj/attn_spec.cubin > gpurun_out/spec_ab.log 2>&1
AB_ROUNDS=9 AB_S=1024 timeout 900 python tools/attn_ab.py paper_2403_16863_b200/_obj/attn_spec.cubin > gpurun_out/spec_ab1k.log 2>&1
