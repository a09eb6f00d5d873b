"""Config 5: fused attention S sweep (B=4 H=32 D=128, S = 1K..16K), on 1..8 B200s.

Per S: the nvcc schedule's TFLOP/s, a hardware-priced search (extended classes),
the accepted schedule re-timed against nvcc (paired), and its 10M-sample
verification -- the same flow as bench.py's hardware phase.  torch SDPA is timed
beside it for context.  Writes one JSON document (argv[1], default stdout).

Multi-GPU (one process per GPU, ``--gpus N`` spawns the ranks itself or run it under
torchrun): every rank runs its own chains (seeds sharded), the ranks all-gather
(energy, seed) each epoch over libsip's NCCL communicator and adopt the global best, and
the 10 M verification samples of the accepted schedule are sharded by batch (rank,
rank + N, ...); rank 0 writes the document.
"""
import argparse
import json
import sys
import time

sys.path.insert(0, '.')
import torch
import torch.nn.functional as F

import bench

ap = argparse.ArgumentParser()
ap.add_argument("out", nargs="?")
ap.add_argument("--seqs", default="1024,2048,4096,8192,16384")
ap.add_argument("--rounds", type=int, default=8)
ap.add_argument("--gpus", type=int, default=1)
a = ap.parse_args()
import os
import subprocess

if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    sys.exit(subprocess.call([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                              f"--nproc-per-node={a.gpus}", "--master-addr", "127.0.0.1",
                              "--master-port", str(port), __file__, *sys.argv[1:]]))
world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
os.environ["SIP_DEVICE"] = str(local)
dist = None
if world > 1:
    import torch.distributed as td

    from paper_2403_16863_b200.engine import get_context
    from paper_2403_16863_b200.parallel import NcclGroup

    td.init_process_group("gloo")  # rendezvous only; the exchanges run over NCCL (libsip)
    dist = NcclGroup(get_context(local), rank, world, rendezvous=td)
args = argparse.Namespace(chains=16, epoch=8, verify_samples=10_000_000, classes="extended")
rows = []
for S in [int(x) for x in a.seqs.split(",")]:
    t0 = time.time()
    r = bench.hardware_phase("attn", None, local, rank, world, dist, args, a.rounds,
                             shape=dict(B=4, H=32, S=S, D=128))
    if rank != 0:
        continue
    from paper_2403_16863_b200.attention import AttnTarget
    tgt = AttnTarget(B=4, H=32, S=S, device=local).allocate()
    q, k, v = tgt.inputs
    for _ in range(3):
        F.scaled_dot_product_attention(q, k, v)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10):
        F.scaled_dot_product_attention(q, k, v)
    e1.record()
    torch.cuda.synchronize()
    sdpa = tgt.flops / (e0.elapsed_time(e1) / 10) / 1e9
    del tgt, q, k, v
    torch.cuda.empty_cache()
    row = {"S": S, "flop_per_launch": 4 * 4 * 32 * S * S * 128,
           "roofline": {k2: r["roofline"][k2] for k2 in ("achieved", "peak", "frac", "avg_launch_ms",
                                                          "clocks_during")},
           "tuned": r["tuned"], "verify": r["verify"], "hw": r["hw"],
           "torch_sdpa_tflops": sdpa, "seconds": time.time() - t0}
    rows.append(row)
    print(f"S={S}: nvcc {r['tuned']['nvcc_tflops']:.0f} TFLOP/s, tuned x{r['tuned']['speedup']:.4f}, "
          f"verify {r['verify']['passed']}/{r['verify']['samples']}, sdpa {sdpa:.0f}", flush=True)
if dist:
    dist.barrier()
    dist.close()
if rank != 0:
    sys.exit(0)
doc = {"config": f"fused attention S sweep, B=4 H=32 D=128 fp16, non-causal, {world} x B200",
       "ranks": world, "peaks": bench.peaks(), "rows": rows}
if a.out:
    json.dump(doc, open(a.out, "w"), indent=1)
else:
    print(json.dumps(doc))
