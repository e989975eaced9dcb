"""Summarise an ncu --metrics gpu__time_duration.sum CSV (kernel -> total us, count)."""
import csv
import sys
from collections import defaultdict

tot = defaultdict(float)
cnt = defaultdict(int)
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            k = d["Kernel Name"].split("(")[0][:70]
            v = float(d["Metric Value"].replace(",", ""))
            if d["Metric Unit"] == "nsecond":
                v /= 1000
            elif d["Metric Unit"] == "msecond":
                v *= 1000
            tot[k] += v
            cnt[k] += 1
s = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v:10.1f} us {100 * v / s:5.1f}%  x{cnt[k]:<3d} {k}")
