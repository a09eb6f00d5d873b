# hardware-priced searches at the paper's shapes + ncu of the nvcc schedules
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python tools/long_search.py --target gemm --shape M=512,N=512,K=2048 --chains 256 --max-seconds 600 --out gpurun_out/long_gemm_512.json > gpurun_out/ps_gemm.log 2>&1
timeout 1200 python tools/long_search.py --target attn --shape B=4,H=32,S=1024 --chains 256 --max-seconds 600 --out gpurun_out/long_attn_1k.json > gpurun_out/ps_attn1k.log 2>&1
timeout 1200 python tools/long_search.py --target attn --shape B=1,H=4,S=16384 --chains 128 --max-seconds 600 --out gpurun_out/long_attn_16k.json > gpurun_out/ps_attn16k.log 2>&1
cat > /tmp/ps_prof.py <<'PY'
import sys; sys.path.insert(0, '.')
from paper_2403_16863_b200.evaluator import B200Backend
from paper_2403_16863_b200.targets import make_target
kind, shape = sys.argv[1], dict(kv.split("=") for kv in sys.argv[2].split(","))
tgt = make_target(kind, **{k: int(v) for k, v in shape.items()}).allocate()
be = B200Backend(tgt, rounds=False)
for _ in range(3): be.run_perm(None)
PY
for spec in "gemm M=512,N=512,K=2048" "attn B=4,H=32,S=1024" "attn B=1,H=4,S=16384"; do
  set -- $spec
  tag=$(echo $2 | tr ',=' '__')
  timeout 600 ncu --set full --clock-control none -k regex:"gemm_lrelu|attn_fwd" -s 2 -c 1 -o gpurun_out/ps_${1}_${tag} python /tmp/ps_prof.py $1 $2 > gpurun_out/ps_ncu_${1}_${tag}.log 2>&1
done
