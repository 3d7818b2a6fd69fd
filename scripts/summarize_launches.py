"""Aggregate an ncu --csv launch list by kernel name: count, total us, share."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[hi]
ix = {h: i for i, h in enumerate(hdr)}
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for r in rows[hi + 1:]:
    if len(r) < len(hdr):
        continue
    name = r[ix["Kernel Name"]][:90]
    m, v = r[ix["Metric Name"]], float(r[ix["Metric Value"]].replace(",", ""))
    if m == "gpu__time_duration.sum":
        agg[name][0] += 1
        agg[name][1] += v / 1e3
    elif m.startswith("dram__bytes"):
        agg[name][2] += v
tot = sum(v[1] for v in agg.values())
print(f"total {tot:.1f} us over {sum(v[0] for v in agg.values())} launches")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{v[0]:6d} {v[1]:10.1f} us {100 * v[1] / tot:5.1f}%  {v[2] / 1e6:9.1f} MB  {k}")
