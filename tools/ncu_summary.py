"""Summarise ncu reports into profiles/*.json (run here, on the CPU container).

    python tools/ncu_summary.py gpurun_out/prof_gemm.ncu-rep profiles/r01_gemm.json [traffic.json]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg", "lts__t_bytes.sum",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def summarize(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[head.index("Kernel Name")]}
        for k in KEYS:
            if k in head:
                i = head.index(k)
                d[k] = {"value": r[i], "unit": units[i]}
        res.append(d)
    return res


if __name__ == "__main__":
    data = summarize(sys.argv[1])
    json.dump(data, open(sys.argv[2], "w"), indent=1)
    if len(sys.argv) > 3:
        d = data[0]
        rd = float(d["dram__bytes_read.sum"]["value"]) * SCALE[d["dram__bytes_read.sum"]["unit"]]
        wr = float(d["dram__bytes_write.sum"]["value"]) * SCALE[d["dram__bytes_write.sum"]["unit"]]
        json.dump({"kernel": d["kernel"], "dram_bytes_per_launch": rd + wr, "dram_read": rd,
                   "dram_write": wr, "source": "ncu --set full (" + sys.argv[1].split("/")[-1] + ")"},
                  open(sys.argv[3], "w"), indent=1)
