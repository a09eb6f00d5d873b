cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt
timeout 2400 python -m pytest -q tests -m gpu -x > gpurun_out/r2a_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2a_tests.log
timeout 900 python bench.py > gpurun_out/r2a_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r2a_bench.log
