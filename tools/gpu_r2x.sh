# multi-rank paths on one B200 (ranks share cuda:0): the bench spawning its own ranks, torchrun, reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SIP_SHARE_DEVICE=1 timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --hw-steps 4 --attn-steps 2 --verify-samples 200000 --cpu-seconds 1 > gpurun_out/r2x_spawn2.log 2>&1
echo "spawn rc=$?" >> gpurun_out/r2x_spawn2.log
SIP_SHARE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-attn --hw-steps 4 --verify-samples 200000 --cpu-seconds 1 > gpurun_out/r2x_torchrun2.log 2>&1
echo "torchrun rc=$?" >> gpurun_out/r2x_torchrun2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 --no-unmodified > gpurun_out/r2x_ref2.log 2>&1
echo "ref rc=$?" >> gpurun_out/r2x_ref2.log
