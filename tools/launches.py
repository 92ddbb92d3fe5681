"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.OrderedDict()
for d in data:
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    n = d["Kernel Name"].split("(")[0][:70]
    v = float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] == "ns" else 1.0)
    agg.setdefault(n, []).append(v)
for n, v in agg.items():
    print(f"{n:70s} n={len(v):3d} mean={sum(v)/len(v):8.2f}us min={min(v):8.2f}us")
