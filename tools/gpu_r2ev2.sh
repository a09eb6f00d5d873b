# engine A/B: checkpoint loads/stores with an L2 evict_last policy (-DSIP_CK_EVICT_LAST) vs default
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash tools/engine_ab.sh paper_2403_16863_b200/libsip.so paper_2403_16863_b200/_obj/libsip_evl.so > gpurun_out/evl_ab.log 2>&1
SIP_LIB=paper_2403_16863_b200/_obj/libsip_evl.so timeout 900 python -m pytest -q tests/test_target_parity.py -m gpu -k "byte_identical or vs_oracle_on_target" > gpurun_out/evl_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/evl_tests.log
