# full GPU tier + smoke + default bench + bench launch list (round-2 checkpoint)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash tools/gpu_full.sh r2n
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/r2n_launches.csv python bench.py --steps 2 --warmup 3 --hw-steps 4 --attn-steps 2 --verify-samples 100000 --cpu-seconds 1 --no-e2e > gpurun_out/r2n_ncu_bench.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2n_ncu_bench.log
