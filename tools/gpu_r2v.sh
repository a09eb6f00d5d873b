cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for T in 4 8 16 32; do
  SIP_LOAD_THREADS=$T SIP_EVAL_TIMING=1 timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-attn --verify-samples 100000 --cpu-seconds 0.1 2>gpurun_out/r2v_timing_$T.log | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); g=d['hw']; print('threads $T', 'gemm', round(g['candidates_per_s'],1), 'busy', round(g['device_busy_frac'],3))" >> gpurun_out/r2v_ab.log
done
nproc >> gpurun_out/r2v_ab.log
