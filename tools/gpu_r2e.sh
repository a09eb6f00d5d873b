# sm100 classes: device-vs-model legality, hardware audit of every admitted swap, searches
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest -q tests/test_targets_gpu.py -k "legality_matches_model or single_swap" -x > gpurun_out/r2e_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2e_tests.log
timeout 900 python tools/long_search.py --target gemm --shape M=512,N=512,K=2048 --classes sm100 --chains 256 --max-seconds 300 --out gpurun_out/long_gemm_512_sm100.json > gpurun_out/r2e_gemm.log 2>&1
timeout 900 python tools/long_search.py --target attn --shape B=4,H=32,S=1024 --classes sm100 --chains 256 --max-seconds 300 --out gpurun_out/long_attn_1k_sm100.json > gpurun_out/r2e_attn.log 2>&1
