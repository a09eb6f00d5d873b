# sm100-class hardware searches at the bench shapes (GEMM 4096^3, attention B4 H32 S4096)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python tools/long_search.py --target gemm --classes sm100 --chains 4096 --max-seconds 900 --out gpurun_out/r02_long_gemm_4096_sm100.json > gpurun_out/r2aj_gemm.log 2>&1
timeout 1500 python tools/long_search.py --target attn --classes sm100 --chains 1024 --max-seconds 900 --out gpurun_out/r02_long_attn_4096_sm100.json > gpurun_out/r2aj_attn.log 2>&1
