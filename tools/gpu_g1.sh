cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
timeout 1500 python -m pytest -q tests/test_target_parity.py tests/test_distributed.py tests/test_targets_gpu.py -m gpu -k "target or nccl or attention" > gpurun_out/g1_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/g1_tests.log
for tool in memcheck racecheck synccheck; do timeout 600 compute-sanitizer --tool $tool python tools/sanitize_run.py attn_multi > gpurun_out/g1_san_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/g1_san_$tool.log; done
timeout 900 python bench.py --steps 3 --warmup 3 --no-attn --hw-steps 4 --verify-samples 100000 > gpurun_out/g1_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/g1_bench.log
