# final-code multi-rank paths on one B200 (ranks share cuda:0) + the realistic-k lines at 16 waves
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SIP_SHARE_DEVICE=1 timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --hw-steps 4 --attn-steps 2 --verify-samples 200000 --cpu-seconds 1 > gpurun_out/mr_spawn2.log 2>&1
echo "spawn rc=$?" >> gpurun_out/mr_spawn2.log
SIP_SHARE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-attn --hw-steps 4 --refill 32 --verify-samples 200000 --cpu-seconds 1 > gpurun_out/mr_torchrun2.log 2>&1
echo "torchrun rc=$?" >> gpurun_out/mr_torchrun2.log
