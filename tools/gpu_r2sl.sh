# SlotRow gather8 slot blocks branch-free: engine parity GPU tests, then engine A/B vs the
# previous build (paper_2403_16863_b200/_obj/libsip_base.so), same box
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest -q tests/test_engine_gpu.py tests/test_target_parity.py tests/test_acceptance_gpu.py tests/test_api_gpu.py -m gpu > gpurun_out/sl_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/sl_tests.log
bash tools/engine_ab.sh paper_2403_16863_b200/_obj/libsip_base.so paper_2403_16863_b200/libsip.so > gpurun_out/sl_ab.log 2>&1
