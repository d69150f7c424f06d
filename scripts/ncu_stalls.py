"""Stall-reason totals of an ncu report over an address range (or the whole kernel).

    python scripts/ncu_stalls.py REPORT.ncu-rep [LO_HEX HI_HEX]   (addresses: low 20 bits)
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
lo = int(sys.argv[2], 16) if len(sys.argv) > 3 else 0
hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else 1 << 40
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
tot = {h[i]: 0.0 for i in cols}
for r in rows[2:]:
    a = int(r[0], 16) & 0xFFFFF
    if lo <= a <= hi:
        for i in cols:
            try:
                tot[h[i]] += float(r[i])
            except ValueError:
                pass
s = sum(tot.values()) or 1
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    if v:
        print(f"{k:28s} {100 * v / s:5.1f}%")
