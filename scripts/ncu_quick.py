"""Summarise an ncu report here (no GPU): key raw metrics and the top stall lines.

    python scripts/ncu_quick.py REPORT.ncu-rep [--top N] [--grep TEXT]
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__cycles_elapsed.avg.per_second",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]


def main():
    rep = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 25
    grep = sys.argv[sys.argv.index("--grep") + 1] if "--grep" in sys.argv else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, v = r[0], r[2]
    for k in KEYS:
        if k in h:
            print(f"{k:70s} {v[h.index(k)]}")
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hh = rows[1]
    data = rows[2:]
    i_s, i_src, i_ex = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Source"), hh.index(
        "Instructions Executed")
    tot = sum(float(x[i_s]) for x in data) or 1.0
    print("--- top stall lines (% of samples, executed, source)")
    for x in sorted(data, key=lambda x: -float(x[i_s]))[:top]:
        print(f"{100 * float(x[i_s]) / tot:5.1f} {x[i_ex]:>10s} {x[0][-5:]} {x[i_src][:110]}")
    if grep:
        print(f"--- lines matching {grep}")
        for x in data:
            if grep in x[i_src]:
                print(f"{100 * float(x[i_s]) / tot:5.1f} {x[i_ex]:>10s} {x[0][-5:]} {x[i_src][:110]}")


if __name__ == "__main__":
    main()
