# evaluator rounds + engine ncu at the bench's chain count + short bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_targets_gpu.py -m gpu -k "measure" > gpurun_out/r2b_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2b_tests.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:anneal_fused -s 1 -c 1 \
  -o gpurun_out/engine_r2b python tools/profile_kernels.py engine > gpurun_out/r2b_ncu.log 2>&1
timeout 1200 python bench.py --steps 5 --warmup 3 --hw-steps 8 --attn-steps 4 --verify-samples 200000 > gpurun_out/r2b_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r2b_bench.log
