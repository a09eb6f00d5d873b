"""Per-source-line stall hotspots of an ncu report (run here on the CPU container).

    python tools/ncu_lines.py gpurun_out/engine_it1.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))

    def I(x):
        try:
            return int(x)
        except ValueError:
            return 0
    lines = [r for r in rows[3:] if len(r) > 9 and r[0].isdigit()]
    tot = sum(I(r[4]) for r in lines)
    print("samples", tot)
    for r in sorted(lines, key=lambda r: -I(r[4]))[:top]:
        ex = I(r[7])
        print(r[0].rjust(5), f"{100 * I(r[4]) / tot:5.1f}%", str(ex).rjust(11),
              f"thr={I(r[8]) / max(1, ex):4.1f}", r[1].strip()[:84])


if __name__ == "__main__":
    main()
