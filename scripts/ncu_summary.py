"""Summarise ncu reports (.ncu-rep from `ncu --set full`) or a launch list (.csv from
`ncu --metrics gpu__time_duration.sum --csv`) into small JSON files under profiles/.

    python scripts/ncu_summary.py gpurun_out/ncu_*.ncu-rep --out profiles/r01_ncu_full.json
    python scripts/ncu_summary.py --launches gpurun_out/launches.csv --out profiles/r01_launches.json
"""
import argparse
import collections
import csv
import io
import json
import subprocess

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
           "launch__shared_mem_per_block_dynamic", "lts__t_bytes.sum", "sm__cycles_elapsed.avg.per_second"]


def summarize_rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:160]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                d[m] = f"{r[i]} {units[i]}".strip()
        res.append(d)
    return res


def summarize_launches(path):
    rows = list(csv.reader(open(path)))
    i0 = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[i0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[i0 + 1:]:
        if len(r) <= vi or not r[vi]:
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        v = float(r[vi].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        tot[name][0] += 1
        tot[name][1] += v * scale
    all_us = sum(t for _, t in tot.values())
    return [{"kernel": k, "launches": n, "total_us": round(t, 1), "share": round(t / all_us, 4)}
            for k, (n, t) in sorted(tot.items(), key=lambda kv: -kv[1][1])]


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("reps", nargs="*")
    ap.add_argument("--launches", default=None)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    res = {}
    for p in a.reps:
        res[p.split("/")[-1]] = summarize_rep(p)
    if a.launches:
        res["launches"] = summarize_launches(a.launches)
    json.dump(res, open(a.out, "w"), indent=1)
    print(json.dumps(res, indent=1)[:3000])
