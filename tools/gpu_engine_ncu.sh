# ncu --set full of one fused engine launch at the bench's chain count (source-level)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r2}
C=${2:-303104}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:anneal_fused -s 1 -c 1 \
  -o gpurun_out/engine_$TAG python tools/profile_kernels.py engine $C > gpurun_out/engine_ncu_$TAG.log 2>&1
echo "ncu rc=$?" >> gpurun_out/engine_ncu_$TAG.log
