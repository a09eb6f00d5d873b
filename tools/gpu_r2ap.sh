# module load cost: load image as is vs merc sections renamed (SIP_MERC_MODE=1)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for M in 0 1; do
  SIP_MERC_MODE=$M SIP_EVAL_TIMING=1 timeout 600 python tools/long_search.py --target gemm --classes extended --chains 64 --max-seconds 20 --verify-samples 100000 --out gpurun_out/r2ap_merc$M.json > gpurun_out/r2ap_merc$M.log 2> gpurun_out/r2ap_timing$M.log
  SIP_MERC_MODE=$M timeout 300 python -m pytest -q tests/test_targets_gpu.py -k canary -m gpu > gpurun_out/r2ap_canary$M.log 2>&1
done
