"""Benchmark: SIP search-and-evaluate on B200 over the shipped sm_100a targets.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one process per GPU)

Headline (``value``): candidates evaluated per second by the batched search
engine.  Workload: the reference's default search (95 iterations, simulator
energy, AnnealConfig defaults) over the decoded listing of the hand-written
tcgen05 GEMM+LeakyReLU cubin (the M=N=K=4096 target of configs[1]);
``--sim-chains`` chains per GPU (default: two full waves of the fused kernel); one *step* = one epoch: every chain runs its
95 iterations in one kernel launch, then the ranks all-gather (energy, seed)
over NCCL and restart from the global champion.  Device time (CUDA events,
barrier + synchronize on both sides, max over ranks).  ``e2e``: the same
metric through the public API (``run_search`` with Kernel objects, host
buffers, device->host histories and schedules).

Hardware phases (same run): candidates of the GEMM (and the attention
target, B=4 H=32 S=4096 D=128) are re-encoded, loaded with cuModuleLoadData
and timed on the B200 inside CUDA graphs (L2 flushed before every timed
launch): ``hw`` rate and its device-busy fraction, ``roofline`` (the GEMM's
TFLOP/s over the measured peak, from the evaluator's CUDA events), ``tuned``
(nvcc schedule vs best schedule found) and ``verify`` (the best schedule vs the
baseline on independent random samples).  ``cpu_baseline``: the reference
algorithm (oracle C port) on one core over the same listing.

``--impl reference``: the reference's CPU search (oracle port -- the
reference is pure Python and absent on the GPU box) on all host cores over
the same listing; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "tuned attn/GEMM TFLOP/s vs nvcc schedule; candidates evaluated/sec at 1-8 GPU"
UNIT = "candidates/s"
SHAPE = dict(M=4096, N=4096, K=4096)
ATTN_SHAPE = dict(B=4, H=32, S=4096, D=128)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--sim-chains", type=int, default=0,
                    help="engine chains per GPU (0: 16 full waves of SlotRow chains, 112 blocks of "
                         "128 per SM; 2 121 728 on a 148-SM B200)")
    ap.add_argument("--chains", type=int, default=128,
                    help="hardware-priced chains per GPU (more candidates per round amortise its nvcc reference)")
    ap.add_argument("--refill", type=int, default=0,
                    help="hardware phase: start a cohort of this many fresh chains whenever that many "
                         "chain slots are idle (finished chains), so every round prices a full set "
                         "of candidates (0: one cohort, run until its chains finish)")
    ap.add_argument("--hw-steps", type=int, default=24, help="hardware search rounds")
    ap.add_argument("--classes", default="extended", choices=["global", "extended", "sm100"],
                    help="hardware-phase candidate classes: the reference's (global) or the "
                         "sm_100 extension (DESIGN.md s5b); the simulator headline always uses global")
    ap.add_argument("--epoch", type=int, default=8, help="rounds between global-best exchanges")
    ap.add_argument("--verify-samples", type=int, default=10_000_000,
                    help="samples per accepted (champion) schedule, sharded over ranks")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-attn", action="store_true")
    ap.add_argument("--attn-steps", type=int, default=8, help="attention hardware search rounds")
    ap.add_argument("--no-unmodified", action="store_true",
                    help="reference arm: skip the unmodified-package lines (baseline/_ref)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
class ClockSampler:
    """SM clock and throttle reasons sampled every 20 ms during the timed region.

    NVML (nvidia-ml-py) from a background thread; `nvidia-smi -lms 200` is the
    fallback.  The bench's timed regions are often shorter than nvidia-smi's start-up,
    so NVML is what gives them samples at all."""

    REASONS = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int, period_s: float = 0.02):
        self.index = index
        self.period = period_s
        self.rows = []  # (sm_mhz, max_mhz, {reason names})
        self.proc = None
        self.stop = threading.Event()
        self.thread = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def poll():
                while not self.stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.rows.append((float(sm), float(mx), {k for k, v in bits.items() if rs & v}))
                    except pynvml.NVMLError:
                        pass
                    self.stop.wait(self.period)

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return self
        except Exception:  # no NVML: nvidia-smi
            pass
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                  "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                  "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={fields}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6 and parts[0].replace(".", "").isdigit():
                rs = {self.REASONS[i] for i in range(4) if parts[2 + i].lower() == "active"}
                self.rows.append((float(parts[0]), float(parts[1]), rs))

    def __exit__(self, *exc):
        self.stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [r[0] for r in self.rows]
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(r[1] for r in self.rows),
                "sm_mhz_min": min(sm), "reasons": sorted(set().union(*(r[2] for r in self.rows))),
                "samples": len(self.rows), "source": "nvml" if self.proc is None else "nvidia-smi"}


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"tflops": float(d["bf16_tflops"]), "hbm": float(d["hbm_gbs"]), "src": "measured",
                "tflops_sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"]))}
    return {"tflops": 1590.0, "hbm": 6650.0, "src": "fallback", "tflops_sustained": 1400.0}


def engine_roofline(cand_per_s: float, chains: int, state_bytes: int, sm_mhz) -> dict | None:
    """Issue and DRAM rooflines of the fused engine kernel.

    The kernel is a serial integer recurrence per chain (no tensor or FP work): its bound is
    warp-instruction issue, one per scheduler per cycle = 148 SMs x 4 x the SM clock measured
    during the timed region.  Instructions per priced candidate and DRAM bytes per chain come
    from the committed ncu capture of the same kernel at the bench's chain count
    (profiles/engine_ncu_summary.json); the rate is this run's."""
    p = ROOT / "profiles" / "engine_ncu_summary.json"
    if not p.exists() or not sm_mhz:
        return None
    d = json.loads(p.read_text())
    inst = d["warp_inst_per_launch"] / d["priced_per_launch"]
    achieved = inst * cand_per_s
    peak = 148 * 4 * sm_mhz * 1e6
    dram_per_chain = (d["dram_read_bytes"] + d["dram_write_bytes"]) / d["chains"]
    return {"bound": "issue", "achieved": achieved, "peak": peak, "unit": "warp-inst/s",
            "frac": achieved / peak, "warp_inst_per_candidate": inst,
            "issue_active_ncu": d.get("issue_active_pct"),
            "traffic": dram_per_chain * chains, "chain_state_bytes": state_bytes * chains,
            "traffic_over_state": dram_per_chain / state_bytes,
            "source": f"profiles/engine_ncu_summary.json ({d.get('source')}); rate and clock from this run"}


def engine_at_realistic_k(ctx, gemm_listing, temps, dist, world, steps: int = 3) -> dict:
    """The same engine and metric with the sm_100 extension classes, where the
    listings have hundreds of candidates instead of the reference classes' five: the GEMM
    listing and the attention listing, sixteen full waves of chains each, histories recorded."""
    import torch

    from paper_2403_16863_b200.cubin import render_listing
    from paper_2403_16863_b200.machine import MachineConfig
    from paper_2403_16863_b200.parallel import RED_MAX, RED_SUM
    from paper_2403_16863_b200.tables import KernelTables
    from paper_2403_16863_b200.targets import TARGET_DIR

    out = {}
    attn = render_listing((TARGET_DIR / "attn_fwd.cubin").read_bytes(), "attn_fwd_f16")
    for name, lst in (("gemm_lrelu_f16", gemm_listing), ("attn_fwd_f16", attn)):
        dk = ctx.kernel(KernelTables.build(lst.kernel, MachineConfig(), classes="extended"))
        C = 16 * dk.wave_chains()  # sixteen full waves, as the headline (chain-count sweep, DESIGN s4)
        for w in range(2):
            dk.anneal_epoch_reduced(10_000_000 + w * C, C, temps)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        priced = 0
        for k in range(steps):
            res, _ = dk.anneal_epoch_reduced(20_000_000 + k * C, C, temps)
            priced += int(res["priced"])
        torch.cuda.synchronize()
        sec = allreduce(dist, [time.perf_counter() - t0], RED_MAX)[0]
        priced = allreduce(dist, [priced], RED_SUM)[0]
        out[name] = {"candidates_per_s": priced / sec, "n": lst.n, "k": int(dk.k), "chains_per_gpu": C,
                     "classes": "extended", "priced_per_chain": priced / (world * C * steps)}
    return out


def ncu_traffic(kind: str) -> float | None:
    """dram bytes per launch of a target from its committed ncu --set full summary."""
    p = ROOT / "profiles" / f"{kind}_ncu_summary.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["dram_bytes_per_launch"])
        except (KeyError, ValueError):
            return None
    return None


# ---------------------------------------------------------------------------
def decoded_listing():
    from paper_2403_16863_b200.cubin import render_listing
    from paper_2403_16863_b200.targets import TARGET_DIR

    return render_listing((TARGET_DIR / "gemm_lrelu.cubin").read_bytes(), "gemm_lrelu_f16")


# the reference's default search (anneal.py:28-60): T 1.0 -> 0.01, cooling 1.05 = 95 iterations
REF_TEMPS = None


def ref_temperatures() -> list:
    """AnnealConfig() defaults restated (anneal.py:47-60), so the CPU arm imports no product code."""
    global REF_TEMPS
    if REF_TEMPS is None:
        import math

        t_max, t_min, cooling = 1.0, 0.01, 1.05
        budget = math.ceil(math.log(t_max / t_min) / math.log(cooling))
        from oracle import oracle

        REF_TEMPS = oracle.temperatures(t_max, cooling, budget)
    return REF_TEMPS


def cpu_reference_rate(seconds: float, workers: int = 1, name: str = "gemm_lrelu_f16") -> dict:
    """Reference search (oracle C port, simulator energy) on the committed decoded listing
    (tests/golden/listings), with tables packed from the reference's own per-instruction
    facts (oracle/golden_tables.py): the CPU arm touches no product code."""
    from oracle import oracle
    from oracle.golden_tables import load_targets, tables_from_facts

    rec = load_targets()[name]
    temps = ref_temperatures()
    if workers <= 1:
        ol = oracle.OracleListing(tables_from_facts(rec))
        t0 = time.perf_counter()
        priced = chains = 0
        while time.perf_counter() - t0 < seconds:
            hist, *_ = ol.anneal(chains, temps)
            priced += int((hist["status"] <= 1).sum())
            chains += 1
        dt = time.perf_counter() - t0
    else:
        from concurrent.futures import ProcessPoolExecutor

        t0 = time.perf_counter()
        with ProcessPoolExecutor(workers) as ex:
            futs = [ex.submit(_cpu_worker, name, w, seconds) for w in range(workers)]
            res = [f.result() for f in futs]
        dt = time.perf_counter() - t0
        priced = sum(r[0] for r in res)
        chains = sum(r[1] for r in res)
    return {"value": priced / dt, "unit": UNIT, "cores": workers, "kind": "port",
            "sample": f"{chains} chains x {len(temps)} iterations of the reference search "
                      f"(oracle C port, simulator energy) on the decoded {name} listing "
                      f"(n={rec['n']}), {dt:.1f} s"}


def _cpu_worker(name, wid, seconds):
    sys.path.insert(0, str(ROOT))
    from oracle import oracle
    from oracle.golden_tables import load_targets, tables_from_facts

    ol = oracle.OracleListing(tables_from_facts(load_targets()[name]))
    temps = ref_temperatures()
    t0 = time.perf_counter()
    priced = chains = 0
    seed = wid * 1_000_000
    while time.perf_counter() - t0 < seconds:
        hist, *_ = ol.anneal(seed + chains, temps)
        priced += int((hist["status"] <= 1).sum())
        chains += 1
    return priced, chains


def run_reference(args, rank: int) -> None:
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    per_step = max(1.0, 60.0 / max(1, args.steps + args.warmup))
    for _ in range(args.warmup):
        cpu_reference_rate(min(per_step, 2.0), workers=cores)
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        vals.append(cpu_reference_rate(per_step, workers=cores))
    wall = time.perf_counter() - t0
    value = sum(v["value"] for v in vals) / len(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (decoded sm_100a listing of the shipped GEMM+LeakyReLU cubin)",
        "config": {"workload": "reference SIP search (simulator energy) over the gemm_lrelu_f16 "
                               "listing, M=N=K=4096 target", "chains_per_step": "bounded by time"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": vals[0]["sample"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    ref = ROOT / "baseline" / "_ref"
    if (ref / "sasstune").exists() and not args.no_unmodified:
        # the unmodified reference package itself (pip-installed into baseline/_ref), beside
        # the port: its simulator search on all cores, and its hardware loop through its
        # own ExternalCommandBackend driving the B200 adapter
        line["unmodified_reference"] = {"simulator": unmodified_sim_rate(20.0, cores)}
        line["unmodified_reference"]["hw"] = unmodified_hw_rate(90.0)
    print(json.dumps(line), flush=True)


REF_LISTING = ROOT / "tests" / "golden" / "listings" / "gemm_lrelu_f16.sass"


def _unmodified_worker(wid: int, seconds: float):
    sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
    from sasstune import AnnealConfig as RC, MachineConfig as RM, SimulatorBackend as RS
    from sasstune.driver import run_search as rrun
    from sasstune.sasstext import parse_kernel as rparse

    kernel = rparse(REF_LISTING.read_text())
    t0 = time.perf_counter()
    priced = chains = 0
    while time.perf_counter() - t0 < seconds:
        rep = rrun(kernel, RS(RM()), RC(seed=100_000 * wid + chains), chains=1)
        priced += sum(1 for h in rep.chains[0].state.history if h.energy is not None)
        chains += 1
    return priced, chains, time.perf_counter() - t0


def unmodified_sim_rate(seconds: float, workers: int) -> dict:
    """sasstune.run_search (SimulatorBackend, AnnealConfig defaults) on the committed decoded
    listing, one chain per call, `workers` processes with disjoint seeds (the reference runs
    its chains sequentially, driver.py:73-79)."""
    from concurrent.futures import ProcessPoolExecutor

    t0 = time.perf_counter()
    with ProcessPoolExecutor(workers) as ex:
        res = list(ex.map(_unmodified_worker, range(workers), [seconds] * workers))
    wall = time.perf_counter() - t0
    priced, chains = sum(r[0] for r in res), sum(r[1] for r in res)
    return {"value": priced / wall, "unit": UNIT, "cores": workers, "chains": chains,
            "sample": f"{chains} chains of sasstune.run_search on the decoded gemm_lrelu_f16 listing "
                      f"(n=1184), {workers} processes, {wall:.1f} s wall (includes imports)"}


def unmodified_hw_rate(seconds: float) -> dict | None:
    """sasstune.anneal through its ExternalCommandBackend with the B200 adapter
    (`python -m paper_2403_16863_b200 measure --target gemm {schedule_file}`, a subprocess per
    rep as backends.py:66-116 does): the reference's hardware loop on this box.  Bounded by
    time: once `seconds` have passed every further measurement fails fast (the reference then
    discards the candidate, anneal.py:186-189) and the rate counts the priced ones."""
    try:
        import torch

        if not torch.cuda.is_available():
            return None
    except ImportError:
        return None
    sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
    from sasstune import AnnealConfig as RC, ExternalCommandBackend, MeasurementFailed as RMF
    from sasstune.anneal import anneal as ranneal
    from sasstune.sasstext import parse_kernel as rparse

    inner = ExternalCommandBackend(f"{sys.executable} -m paper_2403_16863_b200 measure --target gemm "
                                   "{schedule_file}", timeout_s=300.0, workdir=str(ROOT))

    class Bounded:
        unit = inner.unit

        def __init__(self):
            self.t0 = time.perf_counter()
            self.priced = 0
            self.busy = 0.0

        def measure(self, kernel, reps=1):
            if time.perf_counter() - self.t0 > seconds:
                raise RMF("bench time budget spent")
            t = time.perf_counter()
            out = inner.measure(kernel, reps)
            self.busy += time.perf_counter() - t
            self.priced += 1
            return out

    be = Bounded()
    try:
        ranneal(rparse(REF_LISTING.read_text()), be, RC(seed=0, t_max=0.02, t_min=0.0005, cooling=1.02,
                                                         measure_reps=5))
    except RMF as exc:  # the baseline measurement itself failed
        return {"error": str(exc)}
    cands = max(0, be.priced - 1)  # the first measure is the baseline t0
    return {"candidates_per_s": cands / be.busy if be.busy and cands else 0.0, "priced": cands,
            "seconds_measuring": be.busy,
            "what": "unmodified sasstune.anneal + ExternalCommandBackend (5 subprocess reps per "
                    "candidate) + the B200 adapter; one chain, reference classes"}


# ---------------------------------------------------------------------------
def allreduce(group, vals, op):
    """Element-wise reduction over ranks (op: parallel.RED_SUM / RED_MAX / RED_MIN)."""
    if group is None:
        return [float(v) for v in vals]
    return group.allreduce(vals, op)


def time_flush(device: int, reps: int = 10) -> float:
    """Device time (ms) of the evaluator's L2 flush: a 256 MB memset."""
    import torch

    buf = torch.empty(256 << 20, dtype=torch.uint8, device=torch.device("cuda", device))
    buf.fill_(0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for r in range(reps):
        buf.fill_(r & 0xFF)
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def warm_launch_ms(be, n: int, reps: int = 10) -> float:
    """Median device time (ms) of the nvcc schedule launched back to back without an L2
    flush, as the evaluator's warm-up launches run (not added to the roofline's samples)."""
    import ctypes

    from paper_2403_16863_b200.engine import c_dblp, c_u16p

    import numpy as np

    ident = np.arange(n, dtype=np.uint16)
    med = ctypes.c_double()
    raw = np.zeros(reps, dtype=np.float64)
    be.ctx.check(be.ctx.lib.sip_measure(be.module.handle, ident.ctypes.data_as(c_u16p), ctypes.byref(be.launch),
                                        2, reps, 0, ctypes.byref(med), raw.ctypes.data_as(c_dblp)))
    return med.value


def library_tflops(kind, tgt, be, n: int, rounds: int = 6, reps: int = 5) -> dict:
    """Context only: the same operation through the vendor library on the same inputs
    (torch.matmul -> cuBLAS; scaled_dot_product_attention -> cuDNN/flash), timed like for
    like with the nvcc schedule of our kernel: `rounds` alternating rounds of `reps` launches
    each, a 256 MB L2 flush before every launch on both sides, so both see the same power
    state and clocks; medians over all launches."""
    import numpy as np
    import torch

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=tgt.inputs[0].device)
    if kind == "gemm":
        A, B = tgt.inputs
        fn = lambda: torch.matmul(A, B.transpose(1, 2))  # noqa: E731
        name = "torch.matmul (cuBLAS), fp16, no activation"
    else:
        import torch.nn.functional as F

        q, k, v = tgt.inputs
        fn = lambda: F.scaled_dot_product_attention(q, k, v)  # noqa: E731
        name = "torch scaled_dot_product_attention, fp16, non-causal"
    for _ in range(3):
        fn()
    ident = np.arange(n, dtype=np.uint16)
    lib_ms, ours_ms = [], []
    for _ in range(rounds):
        for _ in range(reps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            lib_ms.append(e0.elapsed_time(e1))
        ours_ms.extend(be._measure_single(ident, reps).raw)
    ms, ours = statistics.median(lib_ms), statistics.median(ours_ms)
    return {"tflops": tgt.flops / ms / 1e9, "ms": ms, "what": name,
            "ours_nvcc_ms": ours, "ours_nvcc_tflops": tgt.flops / ours / 1e9, "library_over_ours": ours / ms,
            "method": f"{rounds} alternating rounds of {reps} flushed launches each (library, then the nvcc "
                      "schedule of our kernel through sip_measure); medians"}


FULL_SHAPE_INPUTS = 16  # independent Philox input sets compared at the tuned shape


def hardware_phase(kind, listing, local, rank, world, dist, args, rounds, shape=None):
    """Hardware-priced search on one tuning target: rate, roofline, tuned vs nvcc, verification."""
    import numpy as np
    import torch

    from paper_2403_16863_b200 import AnnealConfig
    from paper_2403_16863_b200.evaluator import B200Backend
    from paper_2403_16863_b200.hwsearch import HardwareSearch
    from paper_2403_16863_b200.targets import make_target
    from paper_2403_16863_b200.verify import Verifier

    from paper_2403_16863_b200.parallel import RED_MAX as MAX, RED_MIN as MIN, RED_SUM as SUM

    shape = shape or (SHAPE if kind == "gemm" else ATTN_SHAPE)
    tgt = make_target(kind, device=local, **shape).allocate()
    be = B200Backend(tgt, listing, device=local, warmup=2, flush_l2=True)
    n = be.listing.n
    hcfg = AnnealConfig(seed=0, t_max=0.02, t_min=0.0005, cooling=1.02, measure_reps=5,
                        candidate_classes=args.classes)
    # clocks are sampled over the whole phase (nvidia-smi needs ~0.5 s to deliver its
    # first sample; the timed rounds alone can be shorter than that)
    hclk = ClockSampler(local).__enter__()
    hs = HardwareSearch(be, hcfg, args.chains, epoch=args.epoch, dist=dist, refill=args.refill)
    hs.step()
    be.kernel_ms.clear()
    launches0, evald0 = hs.launches, hs.evaluated
    torch.cuda.synchronize()
    h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0.record()
    for _ in range(rounds):
        hs.step()
    torch.cuda.synchronize()
    h1.record()
    h1.synchronize()
    h_ms = allreduce(dist, [h0.elapsed_time(h1)], MAX)[0]
    h_eval, h_launch = allreduce(dist, [hs.evaluated - evald0, hs.launches - launches0], SUM)
    # the nvcc schedule timed on its own as well, so the roofline never depends on how
    # many candidates the search happened to price
    be._measure_single(np.arange(n, dtype=np.uint16), 15)
    hclk.__exit__(None, None, None)
    clocks = hclk.summary()
    kern = list(be.kernel_ms)
    pk = peaks()
    avg_ms = sum(kern) / len(kern)
    achieved = tgt.flops / (avg_ms / 1e3) / 1e12
    # kernels timed back to back for seconds run power-capped: the sustained peak applies
    # when the SM clock under load sat well below its maximum (B200_PROFILING.md)
    sustained = (clocks.get("sm_mhz") and clocks.get("sm_max_mhz")
                 and clocks["sm_mhz"] < 0.9 * clocks["sm_max_mhz"] and pk.get("tflops_sustained"))
    peak = pk["tflops_sustained"] if sustained else pk["tflops"]
    # the burst peak scaled to the SM clock this kernel actually ran at (power cap): how
    # busy the tensor pipe was per cycle, independent of how the cap set the clock
    scaled = (pk["tflops"] * clocks["sm_mhz"] / clocks["sm_max_mhz"]
              if clocks.get("sm_mhz") and clocks.get("sm_max_mhz") else None)
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "frac_of_burst_peak": achieved / pk["tflops"],
                "clock_scaled_peak": scaled,
                "frac_at_observed_clock": achieved / scaled if scaled else None,
                "clocks_during": clocks,
                "traffic": ncu_traffic(kind),
                "kernel": be.listing.func, "flop_per_launch": tgt.flops, "launches_timed": len(kern),
                "avg_launch_ms": avg_ms,
                "peak_source": ("MEASURED_PEAKS.json bf16_tflops_sustained (power-capped clocks during "
                                "the timed region)" if sustained else
                                "MEASURED_PEAKS.json bf16_tflops (burst)") if pk["src"] == "measured"
                else "fallback 1590 TFLOP/s"}
    # the evaluator roofline of SURVEY s8d config 4: (warmup + reps) launches of the kernel per
    # candidate, nothing else -- 1 / ((warmup + reps) * T_kernel) candidates/s per GPU
    warm_ms = warm_launch_ms(be, n)
    floor_ms = (be.warmup + hcfg.measure_reps) * avg_ms
    rate = h_eval / (h_ms / 1e3)
    hw = {"candidates_per_s": rate, "rounds": rounds, "chains_per_gpu": args.chains,
          "refill": args.refill, "chains_started": len(hs.seeds),
          "candidate_classes": args.classes, "candidates_in_listing": int(hs.dk.k),
          "chain_rounds": rounds * args.chains * world, "priced": int(h_eval),
          "evaluator_roofline_candidates_per_s": world * 1e3 / floor_ms,
          "device_busy_frac": rate / (world * 1e3 / floor_ms),
          "t_kernel_ms": avg_ms, "warm_launch_ms": warm_ms,
          "cold_input_sets": be.nsets,
          "note": ("one round = the live chains' candidates re-encoded and loaded with cuModuleLoadData "
                   "on 8 host threads while the device already runs the warm-ups of the modules loaded so "
                   "far (streamed round, chunks of <= 64 candidates): every candidate and one nvcc reference "
                   "warmed up (2 launches each), then launched 5 times in rotated order with an event pair each; "
                   "energy = median over reps of t_cand / t_ref in the same rep. Launches rotate over "
                   f"{be.nsets} input sets so no launch finds its inputs in L2 (no flush). Roofline = "
                   "1 / ((warmup + reps) * T_kernel), T_kernel = average timed launch")}
    if not be.nsets:
        hw["note"] += "; this target needs a 256 MB L2 flush before every timed launch instead"
        hw["flush_ms"] = time_flush(local)
    res = hs.result()
    if dist:
        hs.exchange()
        res = hs.result()
    # acceptance: the best schedule that survives a fail-fast verification screen (SIP
    # rejects candidates whose outputs differ); the survivor then gets the full run below
    ver = Verifier(kind, device=local)
    acc_e, acc_perm, rejected = hs.verified_best(ver)
    if dist:  # every rank screened the same exchanged ranking; rank 0's choice wins
        acc_perm = dist.broadcast_perm(acc_perm, 0)
    tuned = verify = None
    if rank == 0:
        ident = np.arange(n, dtype=np.uint16)
        best = acc_perm
        # re-timed with the protocol that priced it: nvcc and best schedules alternate over 45
        # reps, launches rotated over cold input sets (a 256 MB flush where a target needs it)
        ratio, raw = be.ratio_round(best, 45)
        t_nvcc = be._measure_single(ident, 15).value
        t_best = t_nvcc * ratio
        q1, q3 = np.percentile(raw, [25, 75])
        # the spread of single pairs (IQR) vs the uncertainty of their median: a seeded
        # bootstrap of the median over the 45 pair ratios
        boot = np.median(np.random.default_rng(0).choice(np.asarray(raw), (2000, len(raw))), axis=1)
        b_lo, b_hi = np.percentile(boot, [2.5, 97.5])
        # what a user is handed: the accepted schedule only when its re-timed median is not
        # slower than nvcc's (a search energy below 1 can be noise); else the nvcc schedule
        emit_nvcc = ratio > 1.0
        tuned = {"nvcc_ms": t_nvcc, "best_ms": t_best, "speedup": 1.0 / ratio,
                 "emitted": "nvcc schedule (the accepted one re-timed slower)" if emit_nvcc else "accepted schedule",
                 "emitted_speedup": 1.0 if emit_nvcc else 1.0 / ratio,
                 "speedup_iqr": [1.0 / q3, 1.0 / q1], "speedup_ci95": [1.0 / b_hi, 1.0 / b_lo], "pairs": 45,
                 "nvcc_tflops": tgt.flops / t_nvcc / 1e9, "best_tflops": tgt.flops / t_best / 1e9,
                 "instructions_moved": int((best != ident).sum()),
                 "search_best_energy": res["best_energy"], "accepted_energy": acc_e,
                 "rejected_by_verification": [{"energy": e, "first_failing_sample": v.first_fail_sample,
                                               "max_abs_err": v.max_abs_err} for e, v in rejected],
                 "paper_speedup": 1.1227 if kind == "gemm" else 1.062,
                 "library_tflops": library_tflops(kind, tgt, be, n)}
    # every rank verifies its share of the samples (batches rank, rank+world, ...) of the
    # same champion; (passed, failed) sum and the first failing sample is the min over ranks
    best = acc_perm
    per_rank = -(-args.verify_samples // (world * ver.batch)) * ver.batch
    vr = ver.run(best, per_rank, first_batch=rank, batch_stride=world)
    tot = allreduce(dist, [vr.samples, vr.passed, vr.failed, vr.bitdiff_elems, vr.compared_bytes], SUM)
    vsec = allreduce(dist, [vr.seconds], MAX)[0]
    ff = allreduce(dist, [vr.first_fail_sample if vr.first_fail_sample >= 0 else 2.0 ** 62], MIN)[0]
    if rank == 0:
        verify = {"samples": int(tot[0]), "passed": int(tot[1]), "failed": int(tot[2]),
                  "bit_identical": tot[3] == 0, "first_failing_sample": None if ff >= 2.0 ** 62 else int(ff),
                  "seconds": vsec, "samples_per_s": tot[0] / vsec,
                  "compare_gb_per_s": tot[4] / vsec / 1e9, "ranks": world,
                  "sample": ("one independent 256x256x1024 GEMM+LeakyReLU problem" if kind == "gemm"
                             else "one independent head, S=512 D=128, input scale cycling 0.5/1/2/4 over batches") + ", Philox inputs; baseline "
                            "and champion launched on it, outputs compared (sip_compare)",
                  "tolerance": {"atol": ver.atol, "rtol": ver.rtol}}
        # the same comparison at the tuned shape itself (one sample = one full problem of the
        # benchmarked size), so the accepted schedule is checked where it was timed too
        full = Verifier(kind, device=local, batch=1, shape=dict(shape))
        vf = full.run(best, FULL_SHAPE_INPUTS, check_every=FULL_SHAPE_INPUTS)
        verify["tuned_shape"] = {"inputs": vf.samples, "passed": vf.passed, "failed": vf.failed,
                                 "bit_identical": vf.bitdiff_elems == 0, "shape": dict(shape),
                                 "seconds": vf.seconds}
        del full
    return {"roofline": roofline, "hw": hw, "tuned": tuned, "verify": verify, "launches": h_launch}


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` without a launcher: start N ranks (one process per GPU) with
    torch.distributed.run on 127.0.0.1 and pass rank 0's output through."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"), *sys.argv[1:]]
    return subprocess.call(cmd)


def main() -> None:
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but the launcher started {world} ranks")
    # test hook: SIP_SHARE_DEVICE=1 runs every rank on cuda:0 (collectives over gloo: NCCL
    # refuses two ranks on one device) so the multi-rank path can be exercised on a
    # one-GPU box; never used for reported numbers
    share = os.environ.get("SIP_SHARE_DEVICE") == "1"
    if share:
        local = 0
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import numpy as np
    import torch

    torch.cuda.set_device(local)
    os.environ["SIP_DEVICE"] = str(local)
    from paper_2403_16863_b200.engine import get_context
    from paper_2403_16863_b200.parallel import RED_MAX as MAX, RED_SUM as SUM, NcclGroup, TorchGroup

    ctx = get_context(local)
    dist = None
    if world > 1:
        import torch.distributed as td

        # torch.distributed only for the rendezvous (gloo, CPU); the epoch exchange, the
        # max-over-ranks timings and the verdict merges run over libsip's NCCL communicator
        td.init_process_group("gloo")
        dist = TorchGroup(td) if share else NcclGroup(ctx, rank, world, rendezvous=td)

    from paper_2403_16863_b200 import AnnealConfig, SimulatorBackend, run_search
    from paper_2403_16863_b200.machine import MachineConfig
    from paper_2403_16863_b200.tables import KernelTables

    listing = decoded_listing()
    n = listing.n

    # ================= phase A: batched search engine (headline) =================
    tables = KernelTables.build(listing.kernel, MachineConfig())
    dk = ctx.kernel(tables)
    acfg = AnnealConfig()  # reference defaults: T 1.0 -> 0.01, cooling 1.05, 95 iterations
    temps = acfg.temperatures()
    # 112 blocks of 128 chains per SM = 16 full waves of SlotRow chains (7 resident blocks):
    # the last wave's tail (chains differ in length) shrinks with more waves.  Same box,
    # engine / e2e x 1e9: 227 328 chains 3.88 / 3.81, 265 216 3.97 / 3.92, 397 824 4.10 /
    # 4.07, 530 432 4.19 / 4.18, 795 648 4.30 / 4.29, 1 060 864 4.38 / 4.38, 1 591 296
    # 4.46 / 4.47, 2 121 728 4.50 / 4.51
    C = args.sim_chains or 112 * 128 * ctx.sm_count
    best = {"e": 1.0, "perm": None}

    def epoch(ep: int):
        # chains seeded (ep*world + rank)*C + c on the device; the champion (best energy,
        # then seed) and the counters are reduced there too, so a step moves ~2 KB
        res, champ = dk.anneal_epoch_reduced((ep * world + rank) * C, C, temps, start=best["perm"])
        e_mine = float(res["best_energy"])
        if dist:  # NCCL allgather of (energy, seed, rank); owner broadcasts its champion
            e_mine, _, _, champ = dist.exchange_best(e_mine, int(res["best_seed"]), champ)
        if e_mine < best["e"]:
            best["e"], best["perm"] = e_mine, champ
        return int(res["priced"]), int(res["replayed"]), int(res["ambiguous"])

    for w in range(args.warmup):
        epoch(w)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    priced = replayed = amb = 0
    with ClockSampler(local) as clk:
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record()
        for k in range(args.steps):
            p, r, a = epoch(args.warmup + k)
            priced, replayed, amb = priced + p, replayed + r, amb + a
        torch.cuda.synchronize()
        ev1.record()
        ev1.synchronize()
    ms = ev0.elapsed_time(ev1)
    ms_all = allreduce(dist, [ms], MAX)[0]
    priced_all, replayed_all, props_all = allreduce(
        dist, [priced, replayed, C * len(temps) * args.steps], SUM)
    value = priced_all / (ms_all / 1e3)
    engine = {"kernel": "anneal_fused_kernel", "chains_per_gpu": C, "iterations": len(temps),
              "history": "recorded for every chain (stays in HBM)",
              "proposals_per_s": props_all / (ms_all / 1e3),
              "scoreboard_steps_per_s": replayed_all / (ms_all / 1e3),
              "avg_replay_steps_per_candidate": replayed_all / max(1.0, priced_all),
              "listing_instructions": n, "candidates_in_listing": int(dk.k),
              "global_best_energy": best["e"], "ambiguous_metropolis": amb}

    engine["realistic_k"] = engine_at_realistic_k(ctx, listing, temps, dist, world)
    engine["roofline"] = engine_roofline(priced_all / world / (ms_all / 1e3), C, dk.state_bytes(len(temps)),
                                         clk.summary().get("sm_mhz"))

    # e2e: the same metric through the public API (Kernel object in, AnnealStates out)
    e2e = None
    if not args.no_e2e:
        # untimed, and shaped like the timed loop (the previous step's report alive while
        # the next runs): the first calls build the device tables, both result workspaces
        # and both page-locked summary blocks
        rep = None
        for w in range(max(2, args.warmup)):
            rep = run_search(listing.kernel, SimulatorBackend(MachineConfig()),
                             AnnealConfig(seed=(2_000_000 + w * world + rank) * C), chains=C)
            rep.best.state.best_perm
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ep_priced = 0
        for k in range(args.steps):
            rep = run_search(listing.kernel, SimulatorBackend(MachineConfig()),
                             AnnealConfig(seed=(1_000_000 + k * world + rank) * C), chains=C)
            ep_priced += rep.candidates_evaluated
            champion = rep.best.state.best_perm  # the step's result: the winning schedule (D2H)
            assert len(champion) == n
        torch.cuda.synchronize()
        e1.record()
        e1.synchronize()
        e_ms = allreduce(dist, [e0.elapsed_time(e1)], MAX)[0]
        e_priced = allreduce(dist, [ep_priced], SUM)[0]
        # per step: the temperature schedule goes down (consecutive seeds are generated on the
        # device; the listing's tables are cached per table set, anneal.device_kernel); the
        # device-reduced champion record, the champion's summary and its best schedule come up
        e2e = {"value": e_priced / (e_ms / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(len(temps) * 8),
               "d2h_bytes_per_step": int(48 + 48 + 2 * n),
               "api": "run_search(kernel, SimulatorBackend(), AnnealConfig(seed), chains=C) per step; "
                      "the champion (driver.py:81-85 ranking) is reduced on the device; per-chain "
                      "summaries, histories and schedules stay in HBM until accessed (the champion's "
                      "summary and best schedule are fetched every step)"}

    # ================= phase B: hardware evaluator on the tuning targets =================
    gemm = hardware_phase("gemm", listing, local, rank, world, dist, args, rounds=args.hw_steps)
    attn = None
    if not args.no_attn:
        attn = hardware_phase("attn", None, local, rank, world, dist, args, rounds=args.attn_steps)
    cpu = None
    if rank == 0 and world == 1:
        cpu = cpu_reference_rate(args.cpu_seconds, workers=1)
    roofline = gemm["roofline"]
    h_launch = gemm["launches"] + (attn["launches"] if attn else 0)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_all / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic: decoded listing of the shipped gemm_lrelu_f16 cubin; "
                    "Philox N(0,1) fp16 GEMM inputs for the hardware phase",
            "config": {"workload": "SIP search (reference defaults: 95 iterations, simulator energy) "
                                   "over the sm_100a gemm_lrelu_f16 listing (M=N=K=4096 target), "
                                   "chains sharded over GPUs; hardware phase times candidates of "
                                   "the same kernel on the B200",
                       "chains_per_gpu": C, "step": "one epoch = 95 iterations of every chain + "
                                                    "NCCL allgather of (energy, seed) + champion broadcast",
                       "l2": f"engine chain state ({dk.state_bytes(len(temps)) / 1e3:.1f} KB per chain, "
                             f"{dk.state_bytes(len(temps)) * C / 1e9:.1f} GB per GPU) is far larger than "
                             "L2, so every step streams it from HBM; the hardware phase rotates its "
                             "launches over input sets whose combined size exceeds L2 (or flushes a "
                             "256 MB buffer where that would take more than 64 sets)",
                       "parallelism": f"{world} GPU(s), independent chains, allgather per epoch"},
            "roofline": roofline, "engine": engine,
            "hw": gemm["hw"], "tuned": gemm["tuned"], "verify": gemm["verify"],
            "attn": None if attn is None else {k: attn[k] for k in ("roofline", "hw", "tuned", "verify")},
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary(),
            "gpu_launches": int(args.steps * world * 1 + h_launch),
            "candidates_evaluated": int(priced_all),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.close()
        import torch.distributed as td

        td.destroy_process_group()


if __name__ == "__main__":
    main()
