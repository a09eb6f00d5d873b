# hardware-priced sm100-class searches on the attention listing after the rescale fix (new SASS)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/long_search.py --target attn --classes sm100 --chains 1024 --max-seconds 300 --out gpurun_out/r02_long_attn_4096_sm100_fix.json > gpurun_out/ls_attn.log 2>&1
echo "rc=$?" >> gpurun_out/ls_attn.log
timeout 900 python tools/long_search.py --target attn --classes sm100 --chains 512 --max-seconds 200 --shape B=4,H=32,S=1024 --out gpurun_out/r02_long_attn_1k_sm100_fix.json > gpurun_out/ls_attn1k.log 2>&1
echo "rc=$?" >> gpurun_out/ls_attn1k.log
