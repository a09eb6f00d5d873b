cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
AB_ROUNDS=10 timeout 900 python tools/attn_ab.py paper_2403_16863_b200/_obj/attn/poly0.cubin paper_2403_16863_b200/_obj/attn/poly1.cubin paper_2403_16863_b200/_obj/attn/poly2.cubin > gpurun_out/r2z_attn_ab.log 2>&1
AB_S=1024 AB_ROUNDS=10 timeout 900 python tools/attn_ab.py paper_2403_16863_b200/_obj/attn/poly0.cubin paper_2403_16863_b200/_obj/attn/poly1.cubin paper_2403_16863_b200/_obj/attn/poly2.cubin > gpurun_out/r2z_attn_ab_1k.log 2>&1
