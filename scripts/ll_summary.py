"""Summarise an ncu launch list (gpu__time_duration.sum [+ launch__grid_size, dram__bytes_read.sum])
by kernel: launches, us per launch, MB read per launch, GB/s.

    python scripts/ll_summary.py gpurun_out/ll.csv [...]
"""
import collections
import csv
import sys

for path in sys.argv[1:]:
    rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
    h = rows[0]
    ik, iid, im, iv = (h.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Value"))
    K = collections.OrderedDict()
    for r in rows[1:]:
        K.setdefault(r[iid], {"k": r[ik]})[r[im]] = r[iv]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    tot = 0.0
    for v in K.values():
        t = float(v["gpu__time_duration.sum"].replace(",", "")) / 1e3
        b = float(v.get("dram__bytes_read.sum", "0").replace(",", ""))
        a = agg[v["k"][:60] + " g" + v.get("launch__grid_size", "?")]
        a[0] += 1
        a[1] += t
        a[2] += b
        tot += t
    print(path, "total us", round(tot, 1), "launches", len(K))
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {k:72s} n={a[0]:3d} us={a[1] / a[0]:7.2f} MB={a[2] / a[0] / 1e6:7.2f} GB/s={a[2] / a[1] / 1e3:7.1f}")
