# hardware-priced searches at the bench shapes after chunked rounds
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python tools/long_search.py --target gemm --classes sm100 --chains 16384 --max-seconds 600 --out gpurun_out/r02_long_gemm_4096_sm100.json > gpurun_out/r2ao_gemm.log 2>&1
timeout 1200 python tools/long_search.py --target attn --classes sm100 --chains 2048 --max-seconds 600 --out gpurun_out/r02_long_attn_4096_sm100.json > gpurun_out/r2ao_attn.log 2>&1
