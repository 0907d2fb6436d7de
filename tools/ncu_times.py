"""Sum gpu__time_duration per kernel from an ncu --csv launch list: us total and us/frame."""
import collections
import csv
import sys

fn, frames = sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
lines = [l for l in open(fn).read().splitlines() if l.startswith('"')]
r = list(csv.reader(lines))
h = r[0]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
agg, cnt = collections.Counter(), collections.Counter()
for row in r[1:]:
    if row[mi] != "gpu__time_duration.sum":
        continue
    name = row[ki].split("(")[0].replace("void ", "")[:44]
    agg[name] += float(row[vi].replace(",", "")) / 1e3
    cnt[name] += 1
tot = 0
for k, v in agg.items():
    tot += v
    print(f"{k:46s} n={cnt[k]:4d} {v:10.1f} us {v / frames:8.4f} us/frame")
print(f"{'total':46s}        {tot:10.1f} us {tot / frames:8.4f} us/frame")
