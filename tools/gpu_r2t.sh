cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SIP_EVAL_TIMING=1 timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --verify-samples 100000 --cpu-seconds 0.1 > gpurun_out/r2t_bench.log 2> gpurun_out/r2t_timing.log
