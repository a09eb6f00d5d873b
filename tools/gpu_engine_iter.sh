# engine iteration: parity tests (current lib + each variant), same-box A/B, ncu of the current kernel
#   bash tools/gpu_engine_iter.sh TAG [variant.so ...]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-it}; shift
timeout 900 python -m pytest -q -x tests/test_engine_gpu.py tests/test_target_parity.py tests/test_api_gpu.py -m gpu > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
for V in "$@"; do
  SIP_LIB=$V timeout 600 python -m pytest -q -x tests/test_target_parity.py tests/test_engine_gpu.py -m gpu > gpurun_out/${TAG}_tests_$(basename $V).log 2>&1
  echo "tests rc=$?" >> gpurun_out/${TAG}_tests_$(basename $V).log
done
timeout 900 bash tools/engine_ab.sh paper_2403_16863_b200/_obj/libsip_base.so paper_2403_16863_b200/libsip.so "$@" > gpurun_out/${TAG}_ab.log 2>&1
timeout 300 python tools/engine_history_probe.py >> gpurun_out/${TAG}_ab.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:anneal_fused -s 1 -c 1 \
  -o gpurun_out/engine_$TAG python tools/profile_kernels.py engine 303104 > gpurun_out/${TAG}_ncu.log 2>&1
