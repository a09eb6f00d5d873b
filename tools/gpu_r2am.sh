# module cache kept small after each round vs grown to the round size (SIP_MODULE_KEEP=100000)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for K in 64; do
  SIP_MODULE_KEEP=$K timeout 900 python tools/long_search.py --target gemm --classes sm100 --chains 4096 --max-seconds 150 --verify-samples 100000 --out gpurun_out/r2an_keep$K.json > gpurun_out/r2an_keep$K.log 2>&1
done
