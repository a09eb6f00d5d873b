# final evidence: full GPU tier, smoke, default bench, reference arm, launch list, engine ncu
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-fin}
bash tools/gpu_full.sh $TAG
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_ref.log 2>&1
echo "ref rc=$?" >> gpurun_out/${TAG}_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --hw-steps 4 --attn-steps 2 --verify-samples 100000 --cpu-seconds 1 --no-e2e > gpurun_out/${TAG}_ncu_bench.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${TAG}_ncu_bench.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:anneal_fused -s 1 -c 1 \
  -o gpurun_out/engine_${TAG} python tools/profile_kernels.py engine > gpurun_out/${TAG}_ncu.log 2>&1
