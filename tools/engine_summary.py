"""profiles/engine_ncu_summary.json from an ncu --set full capture of the fused engine
kernel (tools/profile_kernels.py engine) and its log (the captured launch's priced count).

    python tools/engine_summary.py gpurun_out/engine_TAG.ncu-rep gpurun_out/TAG_ncu.log SOURCE_NAME
"""
import json
import re
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from ncu_summary import summarize  # noqa: E402

rep, log, source = sys.argv[1], sys.argv[2], sys.argv[3]
k = [r for r in summarize(rep) if "anneal_fused" in r["kernel"]][0]
lines = [m for m in re.finditer(r"launch (\d+) chains (\d+) priced (\d+) replayed (\d+)", Path(log).read_text())]
m = lines[-1]  # ncu captures the second launch (-s 1 -c 1)
v = lambda key: float(k[key]["value"])  # noqa: E731
scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
out = {
    "kernel": k["kernel"], "source": source, "chains": int(m.group(2)), "priced_per_launch": int(m.group(3)),
    "replayed_per_launch": int(m.group(4)),
    "warp_inst_per_launch": v("smsp__inst_executed.sum"),
    "dram_read_bytes": v("dram__bytes_read.sum") * scale[k["dram__bytes_read.sum"]["unit"]],
    "dram_write_bytes": v("dram__bytes_write.sum") * scale[k["dram__bytes_write.sum"]["unit"]],
    "duration_ms": v("gpu__time_duration.sum"),
    "issue_active_pct": v("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "warps_active_pct": v("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "registers": v("launch__registers_per_thread"),
    "l2_hit_pct": v("lts__t_sector_hit_rate.pct"),
}
Path("profiles/engine_ncu_summary.json").write_text(json.dumps(out, indent=1) + "\n")
print(json.dumps(out, indent=1))
